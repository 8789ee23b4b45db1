#!/bin/bash
NSB_TMA_STORE=0 timeout 120 python tools/tma_debug.py 1 2>&1 | grep -v "^   at" | grep -v " 0 wrong" ; echo "debug cases done"
NSB_TMA_STORE=0 timeout 600 python -m pytest tests/test_fullsize_parity_gpu.py -m gpu -x -q -k "rand28 or hbm" 2>&1 | tail -1
for rep in 1 2; do
for spec in "1 1" "1 0" "0 1"; do
  set -- $spec
  NSB_TMA=$1 NSB_TMA_STORE=$2 timeout 300 python bench.py --config ${CFG:-rand28} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 5 --warmup 2 > gpurun_out/ab3.log 2>&1
  tail -1 gpurun_out/ab3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$1 store=$2', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/ab3.log
done
done
