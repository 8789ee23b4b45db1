#!/bin/bash
# dataflow passes: parity first (bounded), then deep21 / mcm16 A/B against grid barriers
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_fullsize_gpu.py -m gpu -x -q > gpurun_out/flow_tests.log 2>&1
echo "tests rc=$?"; tail -2 gpurun_out/flow_tests.log
timeout 900 python -m pytest tests/test_fullsize_parity_gpu.py tests/test_deep21_golden.py -m gpu -x -q -k "deep21" > gpurun_out/flow_tests2.log 2>&1
echo "deep21 parity rc=$?"; tail -2 gpurun_out/flow_tests2.log
for rep in 1 2; do
for v in 1 0; do
  for cfg in ${CFGS:-deep21 mcm16}; do
    NSB_FLOW=$v timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-sharded --e2e-steps 1 --steps 3 --warmup 3 > gpurun_out/flow_$cfg.log 2>&1
    tail -1 gpurun_out/flow_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FLOW=$v $cfg', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'])" 2>/dev/null || tail -3 gpurun_out/flow_$cfg.log
  done
done
done
