#!/bin/bash
# Sharded-state bench (BASELINE config 5) on N GPUs of one box.
# usage: bash tools/shard_bench.sh N Q [Q ...]
N=$1; shift
mkdir -p gpurun_out
for Q in "$@"; do
  if [ "$N" = 1 ]; then
    timeout 900 python bench.py --config shard --qubits $Q --steps 3 --warmup 3 > gpurun_out/shard_n${N}_q$Q.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29400 + Q)) bench.py --config shard --qubits $Q --steps 3 --warmup 3 \
      > gpurun_out/shard_n${N}_q$Q.log 2>&1
  fi
  tail -1 gpurun_out/shard_n${N}_q$Q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$N Q=$Q', d['value'], d['ms_per_step'], d['breakdown_ms'], 'nvlink', d['nvlink']['achieved_gbs'], 'hbm_frac', d['roofline']['frac'], 'swaps', d['config']['qubit_swaps'])" 2>/dev/null || tail -3 gpurun_out/shard_n${N}_q$Q.log
done
