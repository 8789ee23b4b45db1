#!/bin/bash
# full GPU test suite + smoke + default bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/full_gpu_tests.log 2>&1
tail -3 gpurun_out/full_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/full_bench.log 2>&1
tail -1 gpurun_out/full_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'], 'e2e', d['e2e']['value'], 'launches', d['gpu_launches'])" 2>/dev/null || tail -5 gpurun_out/full_bench.log
