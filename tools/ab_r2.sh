#!/bin/bash
# A/B of kernel build variants on deep21 and rand28 (3 runs each, interleaved)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for rep in 1 2; do
for cfg in deep21 rand28; do
  for lib in default $@; do
    env $( [ $lib = default ] || echo NSB_LIB_VARIANT=$lib ) python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/ab_${cfg}_$lib.log 2>&1
    echo "$rep $cfg $lib $(tail -1 gpurun_out/ab_${cfg}_$lib.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"])' 2>&1 | tail -1)"
  done
done
done
