#!/bin/bash
# copy-engine swap overlap variants (chunk bits, staging slot bytes) on shard34, 2 GPUs
for spec in ${SPECS:-"3 4294967296" "3 1073741824" "2 4294967296" "2 1073741824" "1 1073741824"}; do
  set -- $spec
  NSB_SWAP_CHUNK_BITS=$1 NSB_SWAP_STAGE_BYTES=$2 NSB_SWAP_OVERLAP=ce timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29521 bench.py --config shard --qubits ${Q:-34} --gpus 2 --steps 2 --warmup 1 > gpurun_out/cevar.log 2>&1
  grep '^{' gpurun_out/cevar.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d.get('sharded', d); o=s.get('swap_overlap', {})
print('bits $1 stage $2', d.get('ms_per_step'), o.get('breakdown_ms'), o.get('hidden_frac'), o.get('overlapped_passes'))" 2>/dev/null || tail -3 gpurun_out/cevar.log
done
