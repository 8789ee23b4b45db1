"""Host emulation of the sharded executor (test infrastructure).

Runs a `sharded.schedule` step list on numpy shards with the oracle's
primitives (oracle/nucsim_oracle.py: apply_dense, branch_probability,
project), following ShardedProgram.run and nsb_shard_swap's exchange rule:
rank r with bit b of `global_bit` swaps the half of its shard whose bit
`local_q` is 1-b, element for element in index order, with the partner
rank r ^ (1 << global_bit).  `exchange` is pluggable so the same code runs
all ranks in one process or one rank per gloo process.
"""

from __future__ import annotations

import numpy as np

from oracle import nucsim_oracle as O
from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200.gates import BY_CODE, gate_matrix


def op_matrix(rec, params, payloads) -> np.ndarray:
    nq = int(rec["nq"])
    off = int(rec["payload"])
    if off >= 0:
        d = 1 << nq
        return payloads[off: off + d * d].reshape(d, d)
    g = BY_CODE[int(rec["tag"])]
    p0 = int(rec["param"])
    pars = tuple(float(x) for x in params[p0: p0 + g.n_params]) if g.n_params else ()
    return gate_matrix(g, pars)


def apply_ops(a, ops, params, payloads):
    for rec in ops:
        if int(rec["kind"]) != N.OP_GATE:
            continue
        qs = tuple(int(q) for q in rec["q"][: int(rec["nq"])])
        a = O.apply_dense(a, op_matrix(rec, params, payloads), qs)
    return a


def full_mma(ops, params, payloads, n):
    """Reference semantics on the full state (engine.py:414-423)."""
    a = np.zeros(1 << n, np.complex128)
    a[0] = 1.0
    probs = []
    for rec in ops:
        k = int(rec["kind"])
        if k == N.OP_GATE:
            a = apply_ops(a, rec[None], params, payloads)
        elif k == N.OP_MEASURE:
            q = int(rec["q"][0])
            p0 = O.branch_probability(a, q, 0)
            O.project(a, q, 0, p0)
            probs.append(p0)
    return probs, a


def half_index(nl: int, bit: int, value: int) -> np.ndarray:
    idx = np.arange(1 << nl, dtype=np.int64)
    return idx[((idx >> bit) & 1) == value]


def local_swap_all(shards, global_bit, local_q, nl):
    """nsb_shard_swap for every rank at once (single-process emulation)."""
    for r in range(len(shards)):
        b = (r >> global_bit) & 1
        if b:
            continue
        p = r | (1 << global_bit)
        mine, theirs = half_index(nl, local_q, 1), half_index(nl, local_q, 0)
        x = shards[r][mine].copy()
        shards[r][mine] = shards[p][theirs]
        shards[p][theirs] = x


def run_steps_all(steps, params, payloads, n, g):
    """All ranks in one process; returns ({step: p0}, full state)."""
    nl = n - g
    shards = [np.zeros(1 << nl, np.complex128) for _ in range(1 << g)]
    shards[0][0] = 1.0
    probs = {}
    for s in steps:
        if s.kind == "gates":
            shards = [apply_ops(a, s.ops, params, payloads) for a in shards]
        elif s.kind == "swap":
            local_swap_all(shards, s.global_bit, s.local_q, nl)
        else:
            p0 = 0.0
            for a in shards:  # rank order
                p0 += O.branch_probability(a, s.local_q, 0)
            probs[s.step] = p0
            for a in shards:
                O.project(a, s.local_q, 0, p0)
    return probs, np.concatenate(shards)


def chunk_sums(a: np.ndarray, clog: int) -> np.ndarray:
    """Per-chunk sums of |a_i|^2 (the values only steer the search; any
    fixed order is valid -- the device uses a warp tree)."""
    p = a.real ** 2 + a.imag ** 2
    return p.reshape(-1, 1 << clog).sum(axis=1)


def sample_all(shards, nl, shots, seed, clog, units=None):
    """ShardedState.sample (or sample_draws with `units`) for every rank at
    once (single-process emulation)."""
    from paper_2310_17739_b200.sharded import sample_shard
    world = len(shards)
    sums = [chunk_sums(a, clog) for a in shards]
    starts = np.zeros(world + 1)
    for r in range(world):
        starts[r + 1] = starts[r] + float(np.cumsum(sums[r])[-1])
    if units is None:
        units = O.as_rng(seed).random(shots)
    shots = len(units)
    draws = np.asarray(units) * starts[-1]
    idx = np.full(shots, -1, np.int64)
    for r, a in enumerate(shards):
        p = a.real ** 2 + a.imag ** 2

        def fetch(off, count, out, p=p):
            out[:] = p[off: off + count]

        got = sample_shard(r, nl, draws, starts, r == world - 1, sums[r], clog, fetch)
        assert np.all((got < 0) | (idx < 0)), "a draw owned by two ranks"
        idx = np.maximum(idx, got)
    assert np.all(idx >= 0), "a draw owned by no rank"
    n = nl + world.bit_length() - 1
    np.clip(idx, 0, (1 << n) - 1, out=idx)
    values, counts = np.unique(idx, return_counts=True)
    return {O.bitstring(int(v), n): int(c) for v, c in zip(values, counts)}


def run_path_all(steps, params, payloads, n, g):
    """ShardedProgram.run_path for every rank at once: ([(is_measure, step, p)],
    shards) along the accepted rejection-mode path."""
    nl = n - g
    shards = [np.zeros(1 << nl, np.complex128) for _ in range(1 << g)]
    shards[0][0] = 1.0
    path = []
    for s in steps:
        if s.kind == "gates":
            shards = [apply_ops(a, s.ops, params, payloads) for a in shards]
        elif s.kind == "swap":
            local_swap_all(shards, s.global_bit, s.local_q, nl)
        else:
            p0 = 0.0
            for a in shards:  # rank order
                p0 += O.branch_probability(a, s.local_q, 0)
            path.append((s.kind == "measure", s.step, p0))
            if p0 <= 0.0:
                break
            for a in shards:
                O.project(a, s.local_q, 0, p0)
    return path, shards
