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
import os

import numpy as np

from paper_2310_17739_b200 import _native as N

PASS_DT = np.dtype([("group_begin", "<i4"), ("group_end", "<i4"), ("op_begin", "<i4"),
                    ("op_end", "<i4"), ("mat_begin", "<i4"), ("mat_count", "<i4"), ("k", "<i4"),
                    ("measure_q", "<i4"), ("measure_slot", "<i4"), ("collapse_q", "<i4"),
                    ("collapse_slot", "<i4"), ("tma", "<i4"), ("tq", "i1", (16,)),
                    ("oq", "i1", (32,)), ("tperm", "i1", (16,))])
_VARIANT = os.environ.get("NSB_LIB_VARIANT")  # build variants (csrc/Makefile DEFS)
OCTETS = 1 if _VARIANT == "o1" else 2  # kOctets
THREAD_BITS = 8 if OCTETS == 1 or _VARIANT == "t12" else 7  # kThreadBits
INDEX_BITS = THREAD_BITS + (1 if OCTETS == 2 else 0)  # kIndexBits
INDEX_SLOTS = 10 if INDEX_BITS > 8 else 8  # kIndexSlots
THREADS = 1 << THREAD_BITS  # kPassThreads
TILE_MAX = 12 if _VARIANT == "t12" else 11  # kTileQubitsMax
GROUP_DT = np.dtype([("am", "<u2", (3,)), ("ram", "<u2", (3,)), ("tcol", "<u2", (INDEX_SLOTS,)),
                     ("rtcol", "<u2", (INDEX_SLOTS,)), ("op_begin", "u1"), ("n_ops_sync", "u1"),
                     ("kmat", "<u2"), ("r_out", "<u8", (4,))], align=True)
OP_DT = np.dtype([("mat", "<i2"), ("cls", "u1"), ("pat", "u1"), ("cols", "<u2"), ("kind", "u1"), ("pad", "u1")])
(DENSE1, DIAG1, DENSE2, SPARSE2, MONO2, DIAG2, CX01, CX10, PAIRQ, PAIRP, PAIRX, SWAP,
 PERMUTE, PAIRQR, PAIRPR, PAIRXR) = range(16)
PATTERNS = {0: (0, 1), 1: (0, 2), 2: (1, 2), 3: (0,), 4: (1,), 5: (2,)}
PAT_T, PAT_ALL = (6, 7, 8), 9  # whole-octet ops (planner.h kPatT0..T2, kPatAll)
PAT_D = (10, 11, 12)  # two-axis whole-octet ops (planner.h kPatD01..D12)
PAT_Q = (13, 14, 15)  # register ops of four-axis groups (kind picks the op)
KIND_SWAP = {52 + p: p for p in range(3)}  # register position p <-> octet index (planner.h)
KIND_CX = {55 + j * 3 + (k if k < j else k - 1): (j, k) for j in range(4) for k in range(4)
           if j != k}  # registers c' = c with bit k ^= bit j (bit 3 = octet index)


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
        assert v.pass_desc_bytes == PASS_DT.itemsize
        assert v.group_desc_bytes == GROUP_DT.itemsize and v.gate_op_bytes == OP_DT.itemsize
        self.n, self.k, self.mma_ok, self.n_measures = v.n_qubits, v.tile_qubits, v.mma_ok, v.n_measures
        self.tma = bool(v.tma_edges)
        # the kernel thread layout the plan is laid out for (planner.cpp)
        self.octets, self.thread_bits = v.octets, v.thread_bits

        def arr(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            raw = (ctypes.c_uint8 * (count * dt.itemsize)).from_address(p)
            return np.frombuffer(bytes(raw), dtype=dt)

        self.passes = arr(v.passes, v.n_passes, PASS_DT)
        self.mma_passes = arr(v.mma_passes, v.n_mma_passes, PASS_DT)
        self.groups = arr(v.groups, v.n_groups, GROUP_DT)
        self.ops = arr(v.gate_ops, v.n_gate_ops, OP_DT)
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


def _swz_edge(l):
    """planner.h swz_tma: the 128-byte TMA swizzle a tile is loaded / stored
    under at the pass edges of a TMA plan (first group's loads, last group's
    stores)."""
    return l ^ ((l >> 3) & 7)


def _reg_cx(x, j, k):
    """reg_cx / swap_axis_q of csrc/device.cu on the 16 registers of a thread:
    register c (bit 3 = octet index = octet-index bit THREAD_BITS of the last
    array axis) -- registers c' = c with bit k ^= bit j."""
    n = x[0].shape[-1]
    t = np.arange(n)
    half = [t[((t >> THREAD_BITS) & 1) == q] for q in (0, 1)]
    get = lambda c: x[c & 7][..., half[c >> 3]]

    def put(c, v):
        x[c & 7][..., half[c >> 3]] = v
    for c in range(16):
        if (c >> j) & 1 and not (c >> k) & 1:
            e = c | (1 << k)
            a, b = get(c).copy(), get(e).copy()
            put(c, b)
            put(e, a)


def _swap_q(x, p):
    """swap_axis_q: exchange register position p with the octet index."""
    A = 1 << p
    n = x[0].shape[-1]
    t = np.arange(n)
    lo = t[((t >> THREAD_BITS) & 1) == 0]
    hi = lo | (1 << THREAD_BITS)
    for c in range(8):
        if c & A:
            continue
        a = x[c | A][..., lo].copy()
        x[c | A][..., lo] = x[c][..., hi]
        x[c][..., hi] = a


def _gate(x, op, m):
    """One GateOp on the octet registers x[0..7] (arrays over threads),
    as gate2 / gate1 in csrc/device.cu."""
    pat = int(op["pat"])
    c = int(op["cls"])
    if pat in PAT_Q:
        kind = int(op["kind"])
        if kind in KIND_SWAP:
            _swap_q(x, KIND_SWAP[kind])
        else:
            _reg_cx(x, *KIND_CX[kind])
        return
    if pat == PAT_ALL:  # whole-octet diagonal (planner group fusion)
        for r in range(8):
            x[r] = m[r] * x[r]
        return
    if pat in PAT_D:  # 4x4 on two axes, one block per value of the third
        a, b = PATTERNS[pat - PAT_D[0]]
        A, B = 1 << a, 1 << b
        H = 7 ^ A ^ B
        for hh in (0, 1):
            h = H if hh else 0
            idx = [h, h | A, h | B, h | A | B]
            v = [x[i] for i in idx]
            w = m[16 * hh: 16 * hh + 16]
            for r in range(4):
                x[idx[r]] = sum(w[4 * r + c] * v[c] for c in range(4))
        return
    if pat in PAT_T:  # 2x2 on axis t, one block per value of the other two axes
        t = pat - PAT_T[0]
        A = 1 << t
        L0, L1 = (2 if t == 0 else 1), (2 if t == 2 else 4)
        for b in range(4):
            h = (L0 if b & 1 else 0) | (L1 if b & 2 else 0)
            x[h], x[h | A] = _mix2(x[h], x[h | A], m[4 * b: 4 * b + 4])
        return
    axes = PATTERNS[pat]
    if len(axes) == 1:
        A = 1 << axes[0]
        for base in range(8):
            if base & A:
                continue
            if c == DIAG1:
                x[base], x[base | A] = m[0] * x[base], m[1] * x[base | A]
            else:
                x[base], x[base | A] = _mix2(x[base], x[base | A], m[:4])
        return
    P, Q = axes
    R = 3 - P - Q
    A, B, H = 1 << P, 1 << Q, 1 << R
    for h in (0, H):
        idx = [h, h | A, h | B, h | A | B]
        v = [x[i] for i in idx]
        out = list(v)
        if c in (CX01, CX10, SWAP):
            s, t = {CX01: (1, 3), CX10: (2, 3), SWAP: (1, 2)}[c]
            out[s], out[t] = v[t], v[s]
        elif c in (PAIRQ, PAIRP, PAIRX, PAIRQR, PAIRPR, PAIRXR):
            (u0, u1), (u2, u3) = {PAIRQ: ((0, 2), (1, 3)), PAIRP: ((0, 1), (2, 3)),
                                  PAIRX: ((0, 3), (1, 2)), PAIRQR: ((0, 2), (1, 3)),
                                  PAIRPR: ((0, 1), (2, 3)), PAIRXR: ((0, 3), (1, 2))}[c]
            out[u0], out[u1] = _mix2(v[u0], v[u1], m[:4])
            out[u2], out[u3] = _mix2(v[u2], v[u3], m[4:8])
        elif c == DIAG2:
            out = [m[s] * v[s] for s in range(4)]
        elif c == MONO2:
            cols = int(op["cols"])
            out = [m[s] * v[(cols >> (2 * s)) & 3] for s in range(4)]
        elif c == SPARSE2:
            cols = int(op["cols"])
            out = [m[2 * s] * v[(cols >> (4 * s)) & 3] + m[2 * s + 1] * v[(cols >> (4 * s + 2)) & 3]
                   for s in range(4)]
        else:
            out = [sum(m[4 * s + u] * v[u] for u in range(4)) for s in range(4)]
        for i, val in zip(idx, out):
            x[i] = val


def _check() -> bool:
    """Per-CTA emulation with the partition / warp-locality asserts (default);
    NSB_PLAN_EXEC_CHECK=0 executes every batch of a pass at once instead
    (same arithmetic, vectorised over batches: for the larger tests)."""
    return os.environ.get("NSB_PLAN_EXEC_CHECK", "1") != "0"


def _apply_group(B, G, ops, mats, tbases, k, nvalid, u_load=_swz, u_store=_swz, tb=THREAD_BITS,
                 octets=OCTETS):
    """One octet sweep over a batch B (nvalid tiles of 2^k stored back to
    back), enumerated exactly as k_blocked's apply_group: swizzled shared-
    memory addresses, un-swizzled here (swz is an involution) to index B."""
    cb = k - 3
    n_act = nvalid << cb
    t = np.arange(n_act, dtype=np.int64)
    a = np.zeros(n_act, np.int64)
    r = np.zeros(n_act, np.int64)
    ib = tb + (1 if octets == 2 else 0)
    for b in range(ib):
        a ^= np.where((t >> b) & 1, int(G["tcol"][b]), 0)
        r ^= np.where((t >> b) & 1, int(G["rtcol"][b]), 0)
    tile = t >> cb
    q_col = int(G["tcol"][tb]) if octets == 2 else 0  # one octet per thread: none
    q_rcol = int(G["rtcol"][tb]) if octets == 2 else 0
    am = [int(v) for v in G["am"]] + [q_col]
    ram = [int(v) for v in G["ram"]] + [q_rcol]
    kmat = int(G["kmat"])
    kl = [_parity(tbases[tile].astype(np.uint64) & np.uint64(G["r_out"][i])) for i in range(4)]
    for j in range(4):  # loads: load basis rows; stores: final row j = sum of kmat's load rows
        r ^= kl[j] * ram[j]
        ks = np.zeros_like(kl[0])
        for i in range(4):
            if (kmat >> (4 * j + i)) & 1:
                ks ^= kl[i]
        a ^= ks * am[j]
    am, ram = am[:3], ram[:3]
    st = [a ^ (am[0] if c & 1 else 0) ^ (am[1] if c & 2 else 0) ^ (am[2] if c & 4 else 0)
          for c in range(8)]
    ld = [r ^ (ram[0] if c & 1 else 0) ^ (ram[1] if c & 2 else 0) ^ (ram[2] if c & 4 else 0)
          for c in range(8)]
    S = B.copy()  # out of place: loads see the pre-sweep batch
    loads = stores = None
    if _check():
        assert len(np.unique(np.concatenate(st))) == 8 * n_act  # octets partition the batch
        assert len(np.unique(np.concatenate(ld))) == 8 * n_act
        n_warps = (1 << tb) // 32
        warp = (t >> 5) & (n_warps - 1)  # octet-index bits 5 .. kThreadBits-1
        # physical shared-memory slots per warp (the kernel's addresses)
        loads = [np.sort(np.concatenate([l[warp == w] for l in ld])) for w in range(n_warps)]
        stores = [np.sort(np.concatenate([s_[warp == w] for s_ in st])) for w in range(n_warps)]
    x = [S[u_load(l)] for l in ld]
    o0 = int(G["op_begin"])
    for op in ops[o0:o0 + (int(G["n_ops_sync"]) & 127)]:
        _gate(x, op, mats[int(op["mat"]):])
    for s, v in zip(st, x):
        B[u_store(s)] = v
    return loads, stores


def _apply_group_batches(Bs, G, ops, mats, tbs, k, nvalid, u_load=_swz, u_store=_swz,
                         tb=THREAD_BITS, octets=OCTETS):
    """_apply_group on every batch at once: Bs (n_batches, nvalid << k),
    tbs (n_batches, nvalid) tile bases."""
    cb = k - 3
    n_act = nvalid << cb
    t = np.arange(n_act, dtype=np.int64)
    a0 = np.zeros(n_act, np.int64)
    r0 = np.zeros(n_act, np.int64)
    ib = tb + (1 if octets == 2 else 0)
    for b in range(ib):
        a0 ^= np.where((t >> b) & 1, int(G["tcol"][b]), 0)
        r0 ^= np.where((t >> b) & 1, int(G["rtcol"][b]), 0)
    tile = t >> cb
    q_col = int(G["tcol"][tb]) if octets == 2 else 0  # one octet per thread: none
    q_rcol = int(G["rtcol"][tb]) if octets == 2 else 0
    am = [int(v) for v in G["am"]] + [q_col]
    ram = [int(v) for v in G["ram"]] + [q_rcol]
    kmat = int(G["kmat"])
    a = np.broadcast_to(a0, (Bs.shape[0], n_act)).copy()
    r = np.broadcast_to(r0, (Bs.shape[0], n_act)).copy()
    kl = [_parity(tbs[:, tile].astype(np.uint64) & np.uint64(G["r_out"][i])) for i in range(4)]
    for j in range(4):
        r ^= kl[j] * ram[j]
        ks = np.zeros_like(kl[0])
        for i in range(4):
            if (kmat >> (4 * j + i)) & 1:
                ks ^= kl[i]
        a ^= ks * am[j]
    am, ram = am[:3], ram[:3]
    x = [np.take_along_axis(Bs, u_load(r ^ (ram[0] if c & 1 else 0) ^ (ram[1] if c & 2 else 0)
                                    ^ (ram[2] if c & 4 else 0)), axis=1) for c in range(8)]
    o0 = int(G["op_begin"])
    for op in ops[o0:o0 + (int(G["n_ops_sync"]) & 127)]:
        _gate(x, op, mats[int(op["mat"]):])
    for c in range(8):
        st = a ^ (am[0] if c & 1 else 0) ^ (am[1] if c & 2 else 0) ^ (am[2] if c & 4 else 0)
        np.put_along_axis(Bs, u_store(st), x[c], axis=1)


def run_passes(plan: HostPlan, passes, state, carry_p0=1.0, eps=1e-12, workers=148,
               chunk=None):
    """Execute a pass list on `state` in place, with k_blocked's per-CTA
    contiguous tile ranges and batches; returns {step: p0} and the carry.
    chunk = (cmask, cval): only the tiles whose bits at cmask equal cval
    (k_blocked's chunk restriction, nsb_shard_swap_overlap)."""
    n = plan.n
    rec = {}
    fast = not _check()

    def edges(P, gi, n_groups):
        """(load, store) slot -> tile-local index maps of group gi: in a TMA pass
        the first group loads and the last stores in the copy layout, slot =
        swz_tma(perm(l)) (PassDesc.tperm), un-permuted here."""
        if not int(P["tma"]):
            return _swz, _swz
        k = int(P["k"])
        perm = [int(x) for x in P["tperm"][:k]]

        def u_edge(x):
            y = _swz_edge(x)
            out = y & ~((1 << k) - 1)
            for i in range(k):
                out = out | (((y >> perm[i]) & 1) << i)
            return out
        return (u_edge if gi == 0 else _swz), (u_edge if gi == n_groups - 1 else _swz)

    for P in passes:
        k = int(P["k"])
        lidx = _scatter(np.arange(1 << k, dtype=np.int64), P["tq"][:k])
        n_tiles = 1 << (n - k)
        tb_all = _scatter(np.arange(n_tiles, dtype=np.int64), P["oq"][:n - k])
        if chunk is not None:
            cm, cv = chunk
            assert not np.any(lidx & cm), "chunk qubits inside a pass's tile"
            tb_all = tb_all[(tb_all & cm) == cv]
            n_tiles = len(tb_all)
        nb = 1 if k >= TILE_MAX else min(1 << (TILE_MAX - k), 4)
        block = plan.mats[int(P["mat_begin"]):int(P["mat_begin"]) + int(P["mat_count"])]
        groups = plan.groups[int(P["group_begin"]):int(P["group_end"])]
        pops = plan.ops[int(P["op_begin"]):int(P["op_end"])]
        assert len(groups) <= 40 and len(pops) <= 80 and len(block) <= 384
        cq = int(P["collapse_q"])
        per, extra = divmod(n_tiles, workers)
        if fast:  # every batch of nb consecutive tiles at once
            nv = min(nb, n_tiles)
            tbs = tb_all.reshape(-1, nv)
            idx = (tbs[:, :, None] | lidx[None, None, :]).reshape(tbs.shape[0], -1)
            B = state[idx]
            if cq >= 0:
                B = np.where((idx >> cq) & 1, 0.0, B * (1.0 / np.sqrt(carry_p0)))
            for gi, G in enumerate(groups):
                sw = edges(P, gi, len(groups))
                _apply_group_batches(B, G, pops, block, tbs, k, nv, *sw, tb=plan.thread_bits,
                                     octets=plan.octets)
            state[idx] = B
        for cta in range(0 if fast else min(workers, n_tiles)):
            t_begin = cta * per + min(cta, extra)
            t_end = t_begin + per + (1 if cta < extra else 0)
            for t0 in range(t_begin, t_end, nb):
                nvalid = min(nb, t_end - t0)
                tbs = tb_all[t0:t0 + nvalid]
                idx = (tbs[:, None] | lidx[None, :]).reshape(-1)
                B = state[idx]
                if cq >= 0:
                    B = np.where((idx >> cq) & 1, 0.0, B * (1.0 / np.sqrt(carry_p0)))
                prev = None  # (loads, stores) of the previous sweep when only __syncwarp follows it
                for gi, G in enumerate(groups):
                    sw = edges(P, gi, len(groups))
                    loads, stores = _apply_group(B, G, pops, block, tbs, k, nvalid, *sw,
                                                 tb=plan.thread_bits, octets=plan.octets)
                    if prev is not None and loads is not None:
                        for w in range(len(loads)):
                            # each warp reads its own writes (RAW) and overwrites
                            # only slots it read itself in the other buffer (WAR)
                            assert np.array_equal(loads[w], prev[1][w])
                            assert np.array_equal(stores[w], prev[0][w])
                    prev = (loads, stores) if int(G["n_ops_sync"]) >> 7 == 0 else None
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
