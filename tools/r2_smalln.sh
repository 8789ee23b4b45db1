#!/bin/bash
# small states: the full grid (default) vs one CTA per tile (NSB_TILE_GRID=1)
for cfg in ucc8 mcm16; do
  for v in 0 1; do
    env $( [ $v = 1 ] && echo NSB_TILE_GRID=1 ) timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 5 --warmup 3 > gpurun_out/sn.log 2>&1
    tail -1 gpurun_out/sn.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg tile_grid=$v', d['ms_per_step'], d['value'])" 2>/dev/null || tail -3 gpurun_out/sn.log
  done
done
