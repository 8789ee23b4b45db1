#!/bin/bash
# GPU tests + bench (run under gpurun).  Usage: bash tools/r2_gpu_quick.sh [pytest -k expr]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -n "$1" ]; then K="-k $1"; fi
timeout 1500 python -m pytest tests -m gpu -q $K > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/pytest_gpu.log
tail -2 gpurun_out/bench.log | cut -c1-600
