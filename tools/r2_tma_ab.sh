#!/bin/bash
# rand28 timing decomposition, TMA vs per-thread cp.async (NSB_DEBUG_BLOCKED:
# 1 skip sweeps, 16 request the next tile at the tile start)
for spec in "1 0" "1 1" "1 16" "1 17" "0 0" "0 1" ${EXTRA}; do
  set -- $spec
  NSB_TMA=$1 NSB_DEBUG_BLOCKED=$2 timeout 300 python bench.py --config ${CFG:-rand28} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 2 \
    > gpurun_out/ab_$1_$2.log 2>&1
  tail -1 gpurun_out/ab_$1_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$1 debug=$2', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/ab_$1_$2.log
done
