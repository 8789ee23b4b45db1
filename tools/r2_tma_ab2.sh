#!/bin/bash
for spec in "1 0" "1 16" "0 0" "1 0" "1 16" "0 0"; do
  set -- $spec
  NSB_TMA=$1 NSB_DEBUG_BLOCKED=$2 timeout 300 python bench.py --config ${CFG:-rand28} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 5 --warmup 2 > gpurun_out/ab2.log 2>&1
  tail -1 gpurun_out/ab2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA=$1 debug=$2', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/ab2.log
done
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
NSB_TMA=1 timeout 600 ncu --metrics $M --clock-control none -k regex:k_blocked -s 2 -c 1 --csv \
    python bench.py --config rand28 --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 1 --warmup 1 > gpurun_out/ncu_bk2.csv 2>/dev/null
grep -E "k_blocked" gpurun_out/ncu_bk2.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"'
