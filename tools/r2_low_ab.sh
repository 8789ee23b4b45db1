#!/bin/bash
# deep21 tile-policy A/B at HEAD: always-tiled low qubits (1, 2 = default, 3 with / without TMA)
for spec in "2 1" "1 1" "3 1" "3 0" "2 1"; do
  set -- $spec
  NSB_LOW_QUBITS=$1 NSB_TMA=$2 timeout 300 python bench.py --config ${CFG:-deep21} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/low.log 2>&1
  tail -1 gpurun_out/low.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('low=$1 tma=$2', d['ms_per_step'], 'passes', d['plan']['passes'], 'sweeps', d['plan']['octet_sweeps'])" 2>/dev/null || tail -3 gpurun_out/low.log
done
