#!/bin/bash
# Multi-GPU checks (run under gpurun --gpus N): default bench line with the
# sharded sub-object, the NCCL sharded GPU tests.
N=${1:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
  --master-port 29511 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/n${N}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/n${N}_bench.log
timeout 900 python -m pytest tests -m gpu -q -k "sharded or nccl" > gpurun_out/n${N}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/n${N}_pytest.log
tail -2 gpurun_out/n${N}_pytest.log
grep '^{' gpurun_out/n${N}_bench.log | tail -1 | cut -c1-300
