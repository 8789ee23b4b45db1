"""torchrun job for tests/test_sharded.py::test_nccl_sharded_matches_oracle:
every rank runs the sharded NCCL executor on its GPU, rank 0 gathers the
shards and stores them next to the full-state oracle run."""

import os
import sys
from pathlib import Path

import numpy as np
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    sys.path.insert(0, str(p))

import shard_exec as SE  # noqa: E402
from paper_2310_17739_b200 import sharded as S  # noqa: E402
from paper_2310_17739_b200 import workloads as W  # noqa: E402


def cases():
    wl = W.filter_workload(11, 1, n_steps=3, seed=5, hop_range=8)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    yield "filter12", wl.executable(fops), wl.params, pool, wl.n_qubits
    wl = W.layered_workload(14, 6, 14)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    yield "layered14", fops, wl.params, pool, 14
    # big enough for chunked overlap of swaps with the gate group after them
    wl = W.layered_workload(18, 6, 18)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    yield "layered18", fops, wl.params, pool, 18


def main(out):
    # the copy-engine exchange on every geometry (the library otherwise keeps
    # short-run regions on the SM swap kernel)
    os.environ["NSB_CE_MIN_RUN"] = "0"
    # peer-memory swaps overlapped with the gate group after them: on the copy
    # engines (the default, "_p2p") and with the SM swap kernel ("_p2psm");
    # NCCL pack/send/unpack swaps ("_nccl")
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    res = {}
    cs = list(cases())
    modes = [(True, "ce", "_p2p"), (True, "1", "_p2psm"), (False, "0", "_nccl")]
    for (tag, ops, params, pool, n), (peer, mode, suffix) in (
            (c, m) for m in modes for c in cs):
        os.environ["NSB_SWAP_OVERLAP"] = mode
        tag = tag + suffix
        st = S.ShardedState.from_torch_distributed(n, device=int(os.environ["LOCAL_RANK"]),
                                                   peer_swaps=peer)
        probs, steps = st.run_mma(ops, params, pool)
        shard = st.download()
        norm = st.norm()
        samples = {clog: st.sample(1024, 2310, chunk_log2=clog) for clog in (4, 13)}
        rej = st.run_rejection(ops, params, pool, 200, 91) if S.replayable(ops) else None
        st.close()
        shards = [None] * dist.get_world_size()
        dist.all_gather_object(shards, shard)
        if rank == 0:
            want_p, want = SE.full_mma(ops, params, pool, n)
            res["got_" + tag] = np.concatenate(shards)
            res["want_" + tag] = want
            res["gotp_" + tag] = np.asarray(probs)
            res["overlap_" + tag] = np.asarray([st.last_overlapped_passes])
            res["wantp_" + tag] = np.asarray(want_p)
            ref = SE.O.sample(res["got_" + tag], n, 1024, 2310)
            res["samples_ok_" + tag] = np.asarray([samples[c] == ref for c in sorted(samples)])
            if rej is not None:  # sharded rejection mode against the full-state oracle
                from test_sharded import _oracle_instrs
                want = SE.O.run_rejection(_oracle_instrs(ops, params, pool), n, 200, 91)
                acc, rcounts, rsteps = rej
                res["rejection_ok_" + tag] = np.asarray([(acc, rsteps, rcounts) == tuple(want)])
            print(tag, "swaps", S.swap_count(steps), "norm", norm, flush=True)
    if rank == 0:
        np.savez(out, **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
