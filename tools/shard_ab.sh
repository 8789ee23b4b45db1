# peer-memory vs NCCL qubit swaps on N GPUs: bash tools/shard_ab.sh N Q
N=$1; Q=$2
mkdir -p gpurun_out
for mode in p2p nccl; do
  env $( [ $mode = nccl ] && echo NSB_SWAP_NCCL=1 ) timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29400 + Q)) bench.py --config shard --qubits $Q --steps 3 --warmup 3 > gpurun_out/shard_${mode}_n${N}_q$Q.log 2>&1
  tail -1 gpurun_out/shard_${mode}_n${N}_q$Q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode N=$N Q=$Q', d['value'], d['ms_per_step'], d['breakdown_ms'], 'nvlink', d['nvlink']['achieved_gbs'], d['config']['qubit_swap_path'])" 2>/dev/null || tail -3 gpurun_out/shard_${mode}_n${N}_q$Q.log
done
