#!/bin/bash
# Overlapped-swap timing experiments on N GPUs (run under gpurun --gpus N).
N=${1:-2}; Q=${2:-34}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() {  # tag env...
  tag=$1; shift
  env "$@" timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config shard --qubits $Q \
    --steps 1 --warmup 1 > gpurun_out/ovx_${tag}.log 2>&1
  echo "$tag rc=$? $(grep '^{' gpurun_out/ovx_${tag}.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read())["sharded"]; o=d["swap_overlap"]; print(d["ms_per_run"], d["breakdown_ms"], o["run_ms_overlapped"], o["run_ms_sequential"], o["swap_ms_sequential"], o["overlapped_passes"])' 2>&1 | tail -1)"
}
run default X=1
run noswap NSB_OVERLAP_DEBUG=1
run nogates NSB_OVERLAP_DEBUG=2
run ctas128 NSB_SWAP_CTAS=128
run ctas8 NSB_SWAP_CTAS=8
run bits1 NSB_SWAP_CHUNK_BITS=1
