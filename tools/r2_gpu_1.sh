#!/bin/bash
# GPU tests (1 GPU) + A/B against a variant build (run under gpurun).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
if [ -n "$AB" ]; then NO_TESTS=1 bash tools/r2_ab.sh "$AB_CFGS" $AB | grep -v "^$"; fi
