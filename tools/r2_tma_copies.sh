#!/bin/bash
# rand28 vs NSB_TMA_MAX_COPIES (0: TMA plan layout, every pass on cp.async)
for c in 0 1 2 4 8; do
  NSB_TMA_MAX_COPIES=$c timeout 300 python bench.py --config ${CFG:-rand28} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 2 > gpurun_out/cp_$c.log 2>&1
  tail -1 gpurun_out/cp_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('copies<=$c', d['ms_per_step'])" 2>/dev/null || tail -3 gpurun_out/cp_$c.log
done
NSB_TMA=0 timeout 300 python bench.py --config ${CFG:-rand28} --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 2 > gpurun_out/cp_off.log 2>&1
tail -1 gpurun_out/cp_off.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TMA off', d['ms_per_step'])"
