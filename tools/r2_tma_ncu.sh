#!/bin/bash
# shared-memory bank conflicts / wavefronts / barrier stalls of k_blocked on rand28, TMA plan vs not
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,gpu__time_duration.sum
for spec in "0 2" "1 0" "1 2"; do
  set -- $spec
  NSB_TMA=$1 NSB_TMA_MAX_COPIES=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:k_blocked -s 2 -c 1 --csv \
    python bench.py --config rand28 --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 1 --warmup 1 > gpurun_out/ncu_tma_$1_$2.csv 2>/dev/null
  echo "== TMA=$1 copies<=$2"; grep -E "k_blocked" gpurun_out/ncu_tma_$1_$2.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"'
done
