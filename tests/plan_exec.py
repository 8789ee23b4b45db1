"""Host executor of an exported device plan (test infrastructure).

Runs the PassDesc / GateDesc program that nsb_plan_create would upload
(exported by nsb_host_plan_view) with numpy, following the kernel's
semantics in csrc/device.cu line by line except the shared-memory swizzle,
which is a storage detail.  Lets the CPU suite verify the planner -- the
relabeling frame, pivots, dual rows, pass tiling, measurement epilogues --
against the oracle without a GPU.  Small qubit counts only.
"""

from __future__ import annotations

import ctypes

import numpy as np

from paper_2310_17739_b200 import _native as N

PASS_DT = np.dtype([("gate_begin", "<i4"), ("gate_end", "<i4"), ("mat_begin", "<i4"),
                    ("mat_count", "<i4"), ("k", "<i4"), ("measure_q", "<i4"),
                    ("measure_slot", "<i4"), ("collapse_q", "<i4"), ("collapse_slot", "<i4"),
                    ("pad", "<i4", (3,)), ("tq", "i1", (16,)), ("oq", "i1", (48,))])
GATE_DT = np.dtype([("mat", "<i4"), ("cls", "u1"), ("nq", "u1"), ("tla", "u1"), ("tlb", "u1"),
                    ("sa", "<u2"), ("sb", "<u2"), ("st1", "<u2"), ("st2", "<u2"), ("st3", "<u2"),
                    ("cols", "<u2"), ("spar", "u1"), ("pad0", "u1", (3,)), ("tcol", "<u2", (8,)),
                    ("rsa", "<u2"), ("rsb", "<u2"), ("rst1", "<u2"), ("rst2", "<u2"),
                    ("rst3", "<u2"), ("rtcol", "<u2", (8,)), ("pad1", "u1", (14,)),
                    ("ra_out", "<u8"), ("rb_out", "<u8")], align=True)
THREADS = 256  # kPassThreads
TILE_MAX = 11  # kTileQubitsMax
(DENSE1, DIAG1, DENSE2, SPARSE2, MONO2, DIAG2, CX01, CX10, PAIRQ, PAIRP, PAIRX, SWAP,
 PERMUTE) = range(13)


class HostPlan:
    def __init__(self, ops, params, payloads, n, workers=148):
        h = ctypes.c_void_p()
        st = N.Status()
        N.check(N.lib().nsb_host_plan_build(N.ptr(ops), len(ops), N.ptr(params),
                                            N.ptr(payloads.view(np.float64)), n, workers,
                                            ctypes.byref(h), ctypes.byref(st)), st)
        self.h = h
        v = N.PlanView()
        N.lib().nsb_host_plan_view(h, ctypes.byref(v))
        assert v.pass_desc_bytes == PASS_DT.itemsize and v.gate_desc_bytes == GATE_DT.itemsize
        self.n, self.k, self.mma_ok, self.n_measures = v.n_qubits, v.tile_qubits, v.mma_ok, v.n_measures

        def arr(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            raw = (ctypes.c_uint8 * (count * dt.itemsize)).from_address(p)
            return np.frombuffer(bytes(raw), dtype=dt)

        self.passes = arr(v.passes, v.n_passes, PASS_DT)
        self.mma_passes = arr(v.mma_passes, v.n_mma_passes, PASS_DT)
        self.gates = arr(v.gates, v.n_gate_descs, GATE_DT)
        self.mats = arr(v.matrices, v.n_matrices, np.dtype(np.complex128))
        self.items = arr(v.items, 4 * v.n_items, np.dtype(np.int32)).reshape(-1, 4)

    def __del__(self):
        if getattr(self, "h", None):
            N.lib().nsb_host_plan_free(self.h)
            self.h = None


def _scatter(values: np.ndarray, bits) -> np.ndarray:
    out = np.zeros_like(values)
    for j, b in enumerate(bits):
        out |= ((values >> j) & 1) << int(b)
    return out


def _ins0(j, pos):
    return ((j >> pos) << (pos + 1)) | (j & ((1 << pos) - 1))


def _parity(x):
    x = np.asarray(x, dtype=np.uint64)
    p = np.zeros(x.shape, np.uint64)
    while np.any(x):
        p ^= x & np.uint64(1)
        x = x >> np.uint64(1)
    return p.astype(np.int64)


def _mix2(x, y, m):
    return m[0] * x + m[1] * y, m[2] * x + m[3] * y


def _swz(l):
    return l ^ (((l >> 3) ^ (l >> 6) ^ (l >> 9)) & 7)


def _apply(B, g, mats, tbases, k, nvalid):
    """One gate sweep over a batch B (nvalid tiles of 2^k stored back to back),
    enumerated exactly as k_blocked's make_sweep / item_addr: swizzled
    shared-memory addresses, un-swizzled here (swz is an involution) to index B."""
    m = mats[int(g["mat"]):]
    nq = int(g["nq"])
    per_tile = 1 << (k - nq)
    items = per_tile * nvalid
    j = np.arange(items, dtype=np.int64)
    t, i = j % THREADS, j // THREADS
    a = np.zeros(items, np.int64)
    r = np.zeros(items, np.int64)  # load side, through the read map
    for b in range(8):
        a ^= np.where((t >> b) & 1, int(g["tcol"][b]), 0)
        r ^= np.where((t >> b) & 1, int(g["rtcol"][b]), 0)
    la = _parity(t & int(g["tla"]))
    lb = _parity(t & int(g["tlb"]))
    sp = int(g["spar"])
    for bit, (st, rst) in enumerate(((int(g["st1"]), int(g["rst1"])), (int(g["st2"]), int(g["rst2"])),
                                     (int(g["st3"]), int(g["rst3"])))):
        on = ((i >> bit) & 1).astype(bool)
        a = np.where(on, a ^ st, a)
        r = np.where(on, r ^ rst, r)
        la = np.where(on, la ^ ((sp >> (2 * bit)) & 1), la)
        lb = np.where(on, lb ^ ((sp >> (2 * bit + 1)) & 1), lb)
    tile = j >> (k - nq)
    ga = _parity(tbases[tile].astype(np.uint64) & np.uint64(g["ra_out"]))
    gb = _parity(tbases[tile].astype(np.uint64) & np.uint64(g["rb_out"]))
    la, lb = (la ^ ga) & 1, (lb ^ gb) & 1
    if nq == 1:
        lb = lb * 0
    sa, sb = int(g["sa"]), int(g["sb"])
    rsa, rsb = int(g["rsa"]), int(g["rsb"])
    a0 = a ^ (la * sa) ^ (lb * sb)
    r0 = r ^ (la * rsa) ^ (lb * rsb)
    U = _swz  # swizzled address -> batch index
    S = B.copy()  # the kernel sweeps out of place: loads see the pre-gate batch
    if nq == 1:
        i0, i1 = U(a0), U(a0 ^ sa)
        x, y = S[U(r0)], S[U(r0 ^ rsa)]
        if g["cls"] == PERMUTE:
            B[i0], B[i1] = x, y
            return
        if g["cls"] == DIAG1:
            x, y = m[0] * x, m[1] * y
        else:
            x, y = _mix2(x, y, m[:4])
        B[i0], B[i1] = x, y
        return
    idx = [U(a0), U(a0 ^ sa), U(a0 ^ sb), U(a0 ^ sa ^ sb)]
    ridx = [U(r0), U(r0 ^ rsa), U(r0 ^ rsb), U(r0 ^ rsa ^ rsb)]
    assert len(np.unique(np.concatenate(idx))) == 4 * items  # items partition the batch
    assert len(np.unique(np.concatenate(ridx))) == 4 * items
    x = [S[ix] for ix in ridx]
    c = int(g["cls"])
    out = list(x)
    if c in (CX01, CX10, SWAP):
        s, tt = {CX01: (1, 3), CX10: (2, 3), SWAP: (1, 2)}[c]
        out[s], out[tt] = x[tt], x[s]
    elif c in (PAIRQ, PAIRP, PAIRX):
        (u0, u1), (u2, u3) = {PAIRQ: ((0, 2), (1, 3)), PAIRP: ((0, 1), (2, 3)),
                              PAIRX: ((0, 3), (1, 2))}[c]
        out[u0], out[u1] = _mix2(x[u0], x[u1], m[:4])
        out[u2], out[u3] = _mix2(x[u2], x[u3], m[4:8])
    elif c == DIAG2:
        out = [m[s] * x[s] for s in range(4)]
    elif c == MONO2:
        cols = int(g["cols"])
        out = [m[s] * x[(cols >> (2 * s)) & 3] for s in range(4)]
    elif c == SPARSE2:
        cols = int(g["cols"])
        out = [m[2 * s] * x[(cols >> (4 * s)) & 3] + m[2 * s + 1] * x[(cols >> (4 * s + 2)) & 3]
               for s in range(4)]
    else:
        out = [sum(m[4 * s + u] * x[u] for u in range(4)) for s in range(4)]
    for ix, v in zip(idx, out):
        B[ix] = v


def run_passes(plan: HostPlan, passes, state, carry_p0=1.0, eps=1e-12, workers=148):
    """Execute a pass list on `state` in place, with k_blocked's per-CTA
    contiguous tile ranges and batches; returns {step: p0} and the carry."""
    n = plan.n
    rec = {}
    for P in passes:
        k = int(P["k"])
        lidx = _scatter(np.arange(1 << k, dtype=np.int64), P["tq"][:k])
        n_tiles = 1 << (n - k)
        tb_all = _scatter(np.arange(n_tiles, dtype=np.int64), P["oq"][:n - k])
        nb = 1 if k >= TILE_MAX else min(1 << (TILE_MAX - k), 4)
        block = plan.mats[int(P["mat_begin"]):int(P["mat_begin"]) + int(P["mat_count"])]
        gates = plan.gates[int(P["gate_begin"]):int(P["gate_end"])]
        assert len(gates) <= 48 and len(block) <= 512
        cq = int(P["collapse_q"])
        per, extra = divmod(n_tiles, workers)
        for cta in range(min(workers, n_tiles)):
            t_begin = cta * per + min(cta, extra)
            t_end = t_begin + per + (1 if cta < extra else 0)
            for t0 in range(t_begin, t_end, nb):
                nvalid = min(nb, t_end - t0)
                tbs = tb_all[t0:t0 + nvalid]
                idx = (tbs[:, None] | lidx[None, :]).reshape(-1)
                B = state[idx]
                if cq >= 0:
                    B = np.where((idx >> cq) & 1, 0.0, B * (1.0 / np.sqrt(carry_p0)))
                for g in gates:
                    _apply(B, g, block, tbs, k, nvalid)
                state[idx] = B
        mq = int(P["measure_q"])
        if mq >= 0:
            keep = ((np.arange(state.size) >> mq) & 1) == 0
            carry_p0 = float(np.sum(np.abs(state[keep]) ** 2))
            rec[int(P["measure_slot"])] = carry_p0
            if carry_p0 < eps:
                break
    return rec, carry_p0


def run_mma(plan: HostPlan, eps=1e-12, workers=148):
    assert plan.mma_ok
    state = np.zeros(1 << plan.n, np.complex128)
    state[0] = 1.0
    rec, _ = run_passes(plan, plan.mma_passes, state, eps=eps, workers=workers)
    return [rec[s] for s in sorted(rec)], state
