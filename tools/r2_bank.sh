#!/bin/bash
# bank-conflict fix: rand28 / deep21 times and conflicts, TMA plan vs not
M=l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
for cfg in rand28 deep21; do
  for t in 1 0; do
    NSB_TMA=$t timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/bk_${cfg}_$t.log 2>&1
    tail -1 gpurun_out/bk_${cfg}_$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg TMA=$t', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/bk_${cfg}_$t.log
  done
done
for t in 1 0; do
  NSB_TMA=$t timeout 600 ncu --metrics $M --clock-control none -k regex:k_blocked -s 2 -c 1 --csv \
    python bench.py --config rand28 --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 1 --warmup 1 > gpurun_out/ncu_bk_$t.csv 2>/dev/null
  echo "== rand28 TMA=$t"; grep -E "k_blocked" gpurun_out/ncu_bk_$t.csv | awk -F'","' '{print $(NF-2), $(NF)}' | tr -d '"'
done
