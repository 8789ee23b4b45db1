#!/bin/bash
# 12-qubit tiles, 256 threads, one CTA per SM (build variant t12) vs the default
mkdir -p gpurun_out
NSB_LIB_VARIANT=t12 timeout 600 python -m pytest tests/test_engine_gpu.py -m gpu -x -q > gpurun_out/t12_tests.log 2>&1
echo "t12 engine tests rc=$?"; tail -1 gpurun_out/t12_tests.log
NSB_LIB_VARIANT=t12 timeout 600 python -m pytest tests/test_fullsize_parity_gpu.py -m gpu -x -q -k "deep21 or forced" > gpurun_out/t12_tests2.log 2>&1
echo "t12 parity rc=$?"; tail -1 gpurun_out/t12_tests2.log
for rep in 1 2; do
for lib in default t12; do
  for cfg in ${CFGS:-deep21 mcm16 rand28}; do
    env $( [ $lib = default ] || echo NSB_LIB_VARIANT=$lib ) timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/t12_$cfg.log 2>&1
    tail -1 gpurun_out/t12_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib $cfg', d['value'], d['ms_per_step'], 'passes', d['plan']['passes'], 'e2e', d['e2e']['value'])" 2>/dev/null || tail -3 gpurun_out/t12_$cfg.log
  done
done
done
