#!/bin/bash
# per-plan thread layout: GPU suite, then small states with the one-octet layout (default for n <= 17) vs two
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/oct_tests.log 2>&1
echo "gpu tests rc=$?"; tail -1 gpurun_out/oct_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in ucc8 mcm16 deep21; do
  for o in default 2; do
    env $( [ $o = default ] || echo NSB_PLAN_OCTETS=$o ) timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 5 --warmup 3 > gpurun_out/oct.log 2>&1
    tail -1 gpurun_out/oct.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg octets=$o', d['ms_per_step'], d['value'], 'e2e', d['e2e']['value'])" 2>/dev/null || tail -3 gpurun_out/oct.log
  done
done
