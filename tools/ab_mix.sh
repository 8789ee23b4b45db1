#!/bin/bash
# A/B: default vs env switches vs lib variants on deep21 (2 interleaved reps)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
  for v in "default" "lib:hot2"; do
    case $v in default) E="";; env:*) E="${v#env:}";; lib:*) E="NSB_LIB_VARIANT=${v#lib:}";; esac
    env $E python bench.py --config ${CFG:-deep21} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/abm.log 2>&1
    echo "$rep $v $(tail -1 gpurun_out/abm.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["plan"]["passes"], d["plan"]["octet_sweeps"], d["plan"]["device_gate_ops"])' 2>&1 | tail -1)"
  done
done
