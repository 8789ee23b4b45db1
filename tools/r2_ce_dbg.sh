#!/bin/bash
# copy-engine swap timing decomposition (NSB_OVERLAP_DEBUG bits, wrong states)
for d in ${DBG:-2 6 10 18 22 26 30}; do
  NSB_OVERLAP_DEBUG=$d NSB_SWAP_OVERLAP=ce timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29521 bench.py --config shard --qubits ${Q:-34} --gpus 2 --steps 1 --warmup 1 > gpurun_out/cedbg_$d.log 2>&1
  grep '^{' gpurun_out/cedbg_$d.log | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); s=d.get('sharded', d)
print('debug $d', d.get('ms_per_step'), s.get('swap_overlap', {}).get('breakdown_ms'))" 2>/dev/null || tail -3 gpurun_out/cedbg_$d.log
done
