#!/bin/bash
# Round-2 GPU check: tests, bench, sanitizers (run under gpurun).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
for tool in memcheck racecheck synccheck; do
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 \
     python tools/sanitize_blocked.py 3 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
done
tail -3 gpurun_out/pytest_gpu.log gpurun_out/bench.log gpurun_out/sanitize_*.log
