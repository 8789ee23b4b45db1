"""Sharded state (paper_2310_17739_b200/sharded.py).

CPU: the schedule (qubit swaps, reordered local groups, collective
measurements, layout restore) is executed on numpy shards with the oracle's
primitives and must reproduce the full-state reference run; a world_size-2
gloo job runs the same steps with one shard per process and real
point-to-point exchanges.  GPU (>= 2 devices): the NCCL path against the
oracle."""

from __future__ import annotations

import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import shard_exec as SE
from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200 import sharded as S
from paper_2310_17739_b200 import workloads as W

ROOT = Path(__file__).resolve().parents[1]


def _filter(n_sys=7, trotter=1, n_steps=3, seed=5):
    wl = W.filter_workload(n_sys, trotter, n_steps=n_steps, seed=seed, hop_range=6)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    return wl.executable(fops), wl.params, pool, wl.n_qubits


def _layered(n, layers, seed):
    wl = W.layered_workload(n, layers, seed)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    return fops, wl.params, pool, n


def _close(got, want, tol=1e-10):
    assert np.linalg.norm(got - want) <= tol * max(np.linalg.norm(want), 1e-300)


@pytest.mark.parametrize("g", [1, 2, 3])
def test_schedule_filter_matches_full_state(g):
    ops, params, pool, n = _filter()
    want_p, want = SE.full_mma(ops, params, pool, n)
    steps = S.schedule(ops, n, g)
    assert S.swap_count(steps) > 0
    got_p, got = SE.run_steps_all(steps, params, pool, n, g)
    assert [got_p[k] for k in sorted(got_p)] == pytest.approx(want_p, rel=1e-10, abs=1e-14)
    _close(got, want)


@pytest.mark.parametrize("n,g,seed", [(7, 1, 1), (8, 2, 2), (9, 3, 3), (10, 1, 4)])
def test_schedule_layered_matches_full_state(n, g, seed):
    ops, params, pool, n = _layered(n, 4, seed)
    _, want = SE.full_mma(ops, params, pool, n)
    steps = S.schedule(ops, n, g)
    _, got = SE.run_steps_all(steps, params, pool, n, g)
    _close(got, want)


def test_schedule_small_window_and_order():
    ops, params, pool, n = _filter(seed=9)
    want_p, want = SE.full_mma(ops, params, pool, n)
    for window in (1, 3, 17):
        steps = S.schedule(ops, n, 2, window=window)
        got_p, got = SE.run_steps_all(steps, params, pool, n, 2)
        # measurements keep their reference order
        order = [s.step for s in steps if s.kind == "measure"]
        assert order == sorted(order) == list(range(len(want_p)))
        _close(got, want)


def test_schedule_lookahead_saves_swaps():
    ops, _, _, n = _layered(12, 6, 7)
    eager = S.swap_count(S.schedule(ops, n, 2, window=1))
    ahead = S.swap_count(S.schedule(ops, n, 2))
    assert ahead <= eager


def test_schedule_g0_is_one_group():
    ops, params, pool, n = _filter()
    steps = S.schedule(ops, n, 0)
    assert S.swap_count(steps) == 0
    assert all(s.kind in ("gates", "measure") for s in steps)


def test_schedule_rejects_bad_args():
    ops, _, _, n = _filter()
    with pytest.raises(ValueError):
        S.schedule(ops, n, n)


# ---------------------------------------------------------------------------
# sampling a sharded state (sample_shard) against the reference's sample


def _random_state(n, seed, concentrate=False):
    rng = np.random.default_rng(seed)
    a = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    if concentrate:  # all mass in the first quarter: ranks with zero mass
        a[1 << (n - 2):] = 0.0
    return a / np.linalg.norm(a)


@pytest.mark.parametrize("seed", [3, 11, 1234])
def test_sample_one_rank_one_chunk_is_reference(seed):
    n = 9
    a = _random_state(n, seed)
    assert SE.sample_all([a], n, 2048, seed, n) == SE.O.sample(a, n, 2048, seed)


@pytest.mark.parametrize("g,clog", [(0, 0), (0, 4), (1, 3), (2, 0), (2, 5), (3, 2)])
@pytest.mark.parametrize("concentrate", [False, True])
def test_sample_shards_match_reference(g, clog, concentrate):
    n = 10
    a = _random_state(n, 100 + g + clog, concentrate)
    nl = n - g
    shards = [a[r << nl:(r + 1) << nl].copy() for r in range(1 << g)]
    for seed in (7, 42):
        assert SE.sample_all(shards, nl, 1024, seed, clog) == SE.O.sample(a, n, 1024, seed)


def test_sample_shard_edge_draws():
    """Draws at 0, inside zero-mass chunks' boundaries and at the total."""
    from paper_2310_17739_b200.sharded import sample_shard
    nl = 4
    p = np.array([0, 0, .25, 0, 0, .25, 0, 0, 0, 0, .5, 0, 0, 0, 0, 0], np.float64)
    sums = p.reshape(-1, 4).sum(axis=1)
    starts = np.array([0.0, 1.0])

    def fetch(off, count, out):
        out[:] = p[off: off + count]

    draws = np.array([0.0, 0.2499, 0.25, 0.5, 0.75, 0.999, 1.0])
    got = sample_shard(0, nl, draws, starts, True, sums, 2, fetch)
    want = np.clip(np.searchsorted(np.cumsum(p), draws, side="right"), 0, 15)
    assert got.tolist() == want.tolist()


# ---------------------------------------------------------------------------
# world_size-2/4/8 gloo: one shard per process, real exchanges


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ops, params, pool, n = _filter()
        g = world.bit_length() - 1
        nl = n - g
        steps = S.schedule(ops, n, g)
        a = np.zeros(1 << nl, np.complex128)
        if rank == 0:
            a[0] = 1.0
        probs = {}
        for s in steps:
            if s.kind == "gates":
                a = SE.apply_ops(a, s.ops, params, pool)
            elif s.kind == "swap":
                b = (rank >> s.global_bit) & 1
                half = SE.half_index(nl, s.local_q, 1 - b)
                send = torch.from_numpy(a[half].view(np.float64).copy())
                recv = torch.empty_like(send)
                peer = rank ^ (1 << s.global_bit)
                reqs = [dist.isend(send, peer), dist.irecv(recv, peer)]
                for r in reqs:
                    r.wait()
                a[half] = recv.numpy().view(np.complex128)
            else:
                part = torch.tensor([SE.O.branch_probability(a, s.local_q, 0)], dtype=torch.float64)
                parts = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, part)
                p0 = 0.0
                for t in parts:
                    p0 += float(t[0])
                probs[s.step] = p0
                SE.O.project(a, s.local_q, 0, p0)
        # collective sampling (ShardedState.sample with gloo collectives)
        clog = 3
        sums = SE.chunk_sums(a, clog)
        tot = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(tot, torch.tensor([float(np.cumsum(sums)[-1])], dtype=torch.float64))
        starts = np.zeros(world + 1)
        for r in range(world):
            starts[r + 1] = starts[r] + float(tot[r][0])
        draws = SE.O.as_rng(99).random(512) * starts[-1]
        pr = a.real ** 2 + a.imag ** 2

        def fetch(off, count, out):
            out[:] = pr[off: off + count]

        mine = S.sample_shard(rank, nl, draws, starts, rank == world - 1, sums, clog, fetch)
        parts = [torch.zeros(512, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(mine))
        idx = torch.stack(parts).max(dim=0).values.numpy()
        values, counts = np.unique(idx, return_counts=True)
        samples = {SE.O.bitstring(int(v), n): int(c) for v, c in zip(values, counts)}
        shards = [None] * world
        dist.all_gather_object(shards, a)
        if rank == 0:
            q.put((probs, np.concatenate(shards), samples))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_world_matches_full_state(world):
    """g = 1, 2, 3 global qubits: one shard per process (8 ranks = the 8-GPU
    layout of BASELINE config 5), real point-to-point exchanges."""
    ops, params, pool, n = _filter()
    want_p, want = SE.full_mma(ops, params, pool, n)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    probs, got, samples = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [probs[k] for k in sorted(probs)] == pytest.approx(want_p, rel=1e-10, abs=1e-14)
    _close(got, want)
    assert samples == SE.O.sample(got, n, 512, 99)


# ---------------------------------------------------------------------------
# GPU: NCCL exchange on >= 2 devices (run under gpurun --gpus 2)


def _gpu_count():
    try:
        return N.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("ranks", [1, 2, 4])
def test_nccl_sharded_matches_oracle(tmp_path, ranks):
    """One rank per GPU over NCCL: sharded MMA runs, ShardedState.sample (device
    chunk masses + range probabilities, 2^4 and 2^13 chunks) and sharded
    rejection mode against the full-state oracle and the reference sampler.
    ranks = 1 runs the same executor, sampler and rejection path on one GPU
    (g = 0: no qubit swaps), so a one-GPU box covers their device half."""
    if _gpu_count() < ranks:
        pytest.skip(f"needs {ranks} GPUs")
    port = _free_port()
    out = tmp_path / "sharded.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           str(ROOT / "tests" / "sharded_gpu_job.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    d = np.load(out)
    for name in d.files:
        if name.startswith("want_"):
            tag = name[5:]
            _close(d["got_" + tag], d[name])
            assert np.allclose(d["gotp_" + tag], d["wantp_" + tag], rtol=1e-10, atol=1e-14)
            assert d["samples_ok_" + tag].all(), tag  # ShardedState.sample == reference sample
    rej = [k for k in d.files if k.startswith("rejection_ok_")]
    assert rej and all(d[k].all() for k in rej), rej  # sharded rejection mode == reference
    if ranks > 1:  # peer-memory swaps overlapped with the gate group after them (chunked passes)
        assert int(d["overlap_layered18_p2p"][0]) > 0    # copy engines
        assert int(d["overlap_layered18_p2psm"][0]) > 0  # SM swap kernel
        assert int(d["overlap_layered18_nccl"][0]) == 0


# ---------------------------------------------------------------------------
# sharded rejection mode: accepted path + host replay (numpy shards)


@pytest.mark.parametrize("g", [0, 1, 2])
def test_sharded_rejection_replay_matches_reference(g):
    """schedule(keep_resets) + run_path on shards + replay_rejection +
    sample_draws reproduce the reference's rejection-mode tallies and samples
    (engine.py:431-474) for the same seed."""
    ops, params, pool, n = _filter()
    assert S.replayable(ops)
    steps = S.schedule(ops, n, g, keep_resets=True)
    assert sum(1 for s in steps if s.kind == "reset") == 3
    path, shards = SE.run_path_all(steps, params, pool, n, g)
    assert [m for m, _, _ in path] == [True, False] * 3
    n_steps = int(np.count_nonzero(ops["kind"] == N.OP_MEASURE))
    rng = SE.O.as_rng(77)
    accepted, step_rej, units = S.replay_rejection(path, n_steps, 300, rng)
    counts = SE.sample_all(shards, n - g, 0, None, 3, units=units) if accepted else {}
    want_acc, want_steps, want_counts = SE.O.run_rejection(_oracle_instrs(ops, params, pool), n,
                                                           300, 77)
    assert (accepted, step_rej, counts) == (want_acc, want_steps, want_counts)


def _oracle_instrs(ops, params, pool):
    out = []
    for r in ops:
        k = int(r["kind"])
        qs = tuple(int(q) for q in r["q"][: int(r["nq"])])
        if k == N.OP_MEASURE:
            out.append(("measure", qs, (), None, int(r["cbit"]) if int(r["cbit"]) >= 0 else 0))
        elif k == N.OP_RESET:
            out.append(("reset", qs, (), None, None))
        elif k == N.OP_GATE:
            out.append(("c" + str(len(qs)) if len(qs) <= 2 else "dense", qs, (),
                        SE.op_matrix(r, params, pool), None))
    return out


def test_replayable_and_reset_draw_leaving_the_path():
    ops, params, pool, n = _filter()
    assert S.replayable(ops)
    assert not S.replayable(ops[ops["kind"] != N.OP_RESET])
    path = [(True, 0, 0.9), (False, -1, 0.0)]  # the reset is certain to draw 1
    with pytest.raises(NotImplementedError):
        S.replay_rejection(path, 1, 5, SE.O.as_rng(1))
