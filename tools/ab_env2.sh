#!/bin/bash
# A/B of planner environment switches: bash tools/ab_env2.sh <config> "<ENV=V ...>" ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cfg=$1; shift
for rep in 1 2; do
  for e in "" "$@"; do
    env $e python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/abe.log 2>&1
    echo "$rep $cfg [$e] $(tail -1 gpurun_out/abe.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["plan"]["passes"], d["plan"]["octet_sweeps"])' 2>&1 | tail -1)"
  done
done
