#!/bin/bash
# TMA tiles: GPU parity of the HBM-policy paths, then rand28 / deep21 with and
# without TMA (NSB_TMA=0: per-thread cp.async under the usual layout).
mkdir -p gpurun_out
timeout 120 python tools/tma_debug.py 1 2>&1 | grep -v "^   at"
timeout 900 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q \
  > gpurun_out/tma_tests.log 2>&1
tail -3 gpurun_out/tma_tests.log
for v in 1 0; do
  for cfg in rand28 ${CFGS}; do
    NSB_TMA=$v timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 \
      > gpurun_out/tma_${cfg}_$v.log 2>&1
    tail -1 gpurun_out/tma_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$v $cfg', d['value'], d['ms_per_step'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['value'])" 2>/dev/null || tail -5 gpurun_out/tma_${cfg}_$v.log
  done
done
