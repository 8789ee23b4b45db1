#!/bin/bash
# copy-engine swap overlap on N GPUs: NCCL/peer parity job, then shard34 / shard32 A/B of the swap modes
N=${1:-2}
mkdir -p gpurun_out
[ -z "$NO_TESTS" ] && timeout 900 python -m pytest tests/test_sharded.py -m gpu -q -k "nccl" > gpurun_out/ce_pytest.log 2>&1
tail -3 gpurun_out/ce_pytest.log
for q in ${QS:-32 34}; do
for mode in ${MODES:-ce 0 1}; do
  NSB_SWAP_OVERLAP=$mode timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29521 bench.py --config shard --qubits $q --gpus $N --steps 2 --warmup 1 > gpurun_out/ce_${q}_$mode.log 2>&1
  grep '^{' gpurun_out/ce_${q}_$mode.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d.get('sharded', d)
print('shard$q mode=$mode', d.get('ms_per_step'), {k: s.get(k) for k in ('qubit_swaps','breakdown_ms')}, s.get('swap_overlap', {}).get('hidden_frac'), s.get('swap_overlap', {}).get('breakdown_ms'))" 2>/dev/null || tail -5 gpurun_out/ce_${q}_$mode.log
done
done
