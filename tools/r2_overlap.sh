#!/bin/bash
# Overlapped qubit swaps on N GPUs (run under gpurun --gpus N): the NCCL /
# peer-memory sharded tests, then shard32 / shard34 bench lines (swap_overlap
# object: overlapped vs sequential run), optionally with several swap CTA counts.
N=${1:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -q -k "sharded or nccl or chunked" > gpurun_out/ov${N}_pytest.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/ov${N}_pytest.log
  tail -3 gpurun_out/ov${N}_pytest.log
fi
for q in ${QUBITS:-32 34}; do
  for ctas in ${CTAS:-0}; do
    NSB_SWAP_CTAS=$ctas timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
      --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --config shard --qubits $q \
      --steps 2 --warmup 1 > gpurun_out/ov${N}_shard${q}_c${ctas}.log 2>&1
    echo "shard$q ctas=$ctas rc=$? $(grep '^{' gpurun_out/ov${N}_shard${q}_c${ctas}.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read())["sharded"]; print(d["ms_per_run"], d["breakdown_ms"], d["swap_overlap"])' 2>&1 | tail -1)"
  done
done
