#!/bin/bash
# Quick GPU check used while tuning: GPU tests (optional) + deep21 + rand28 values.
# usage: bash tools/quick_bench.sh [tests]
mkdir -p gpurun_out
if [ "$1" = "tests" ]; then python -m pytest tests -m gpu -x -q 2>&1 | tail -2; fi
for cfg in deep21 rand28; do
  python bench.py --config $cfg --no-cpu-baseline --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/q_$cfg.log 2>&1
  tail -1 gpurun_out/q_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['config']; print('$cfg', d['value'], d['ms_per_step'], 'passes', c['passes'], 'sweeps', c.get('octet_sweeps'), 'hbm_frac', d['roofline']['frac'])" 2>/dev/null || tail -5 gpurun_out/q_$cfg.log
done
