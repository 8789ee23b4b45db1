#!/bin/bash
# GPU tests, then an interleaved A/B of library variants (run under gpurun).
#   bash tools/r2_ab.sh "<configs>" <variant>...   e.g. bash tools/r2_ab.sh "deep21 rand28" base
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ -z "$NO_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -3 gpurun_out/pytest_gpu.log
fi
CFGS=$1; shift
for rep in 1 2; do
for cfg in $CFGS; do
  for lib in default $@; do
    env $( [ $lib = default ] || echo NSB_LIB_VARIANT=$lib ) timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/ab_${cfg}_$lib.log 2>&1
    echo "$rep $cfg $lib $(tail -1 gpurun_out/ab_${cfg}_$lib.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["e2e"]["value"])' 2>&1 | tail -1)"
  done
done
done
