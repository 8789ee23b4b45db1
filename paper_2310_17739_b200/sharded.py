"""State vectors larger than one GPU: one process per GPU, state split on its
top qubits, NCCL qubit swaps.

The reference keeps the whole 2^n state in one host array
(nucsim/engine.py:42-84) and applies every gate to it (engine.py:92-156,
383-430).  Here a state of n qubits lives on P = 2^g ranks: rank r holds the
2^(n-g) amplitudes whose top g index bits equal r, as the ordinary
(n-g)-qubit state of its own context.  The logical-to-physical qubit layout
is a permutation: a gate runs through the single-GPU plan (k_blocked) when
all its qubits sit at local positions; otherwise a *qubit swap* trades a
global position with a local one (nsb_shard_swap: each rank exchanges half
its shard with one partner over NVLink).

`schedule` is the host half: it walks the op stream in a dependency-
respecting order (an op may run ahead of earlier ops on disjoint qubits,
measurements stay in their order), emits maximal local gate groups, and
when no op can proceed swaps in the qubits of the oldest waiting op,
evicting the local qubits whose next use is furthest away (Belady).  At the
end the layout is restored to the identity so every rank's shard is the
canonical slice of the state.

MMA measurements (engine.py:183-191, 414-423) are collective: every rank
computes its partial P(q=0) with the fixed-order device reduction, the
partials are all-gathered and summed in rank order (identical on every
rank), and every rank collapses with the same p0.  Resets are no-ops in MMA
mode as in the reference; rejection mode is single-GPU only.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import FilterAssertionError
from .gates import Gate

EPS_MMA = 1e-12


@dataclass
class Step:
    kind: str                        # "gates" | "swap" | "measure" | "reset"
    ops: np.ndarray | None = None    # "gates": op records on LOCAL positions
    global_bit: int = -1             # "swap": rank bit that trades places ...
    local_q: int = -1                # ... with this local position
    step: int = -1                   # "measure": reference step index


def _qubits(rec) -> tuple[int, ...]:
    return tuple(int(q) for q in rec["q"][: int(rec["nq"])])


def _translate(ops: np.ndarray, idx: list[int], pos: list[int]) -> np.ndarray:
    out = ops[np.asarray(idx, np.int64)].copy()
    lut = np.asarray(pos, np.int32)
    q = out["q"]
    for j in range(q.shape[1]):
        live = out["nq"] > j
        q[live, j] = lut[q[live, j]]
    out["q"] = q
    mask = np.zeros(len(out), np.uint64)
    for j in range(q.shape[1]):
        live = out["nq"] > j
        mask[live] |= np.left_shift(np.uint64(1), q[live, j].astype(np.uint64))
    out["mask"] = mask
    return out


def schedule(ops: np.ndarray, n: int, g: int, window: int = 4096,
             keep_resets: bool = False) -> list[Step]:
    """Split an MMA op stream (gates, measures, resets, barriers; no trailing
    sampling block) into local gate groups, qubit swaps and collective
    measurements for 2^g ranks.  Resets are MMA no-ops and dropped, unless
    `keep_resets` (the rejection-mode path: "reset" steps, ordered like
    measurements).  Pure host logic (tested on CPU)."""
    if g < 0 or g >= n:
        raise ValueError("need 0 <= g < n")
    nl = n - g
    kinds = ops["kind"]
    step_of = {}
    pending = []
    s = 0
    for i in range(len(ops)):
        k = int(kinds[i])
        if k == N.OP_MEASURE:
            step_of[i] = s
            s += 1
            pending.append(i)
        elif k == N.OP_GATE or (k == N.OP_RESET and keep_resets):
            pending.append(i)
        elif k not in (N.OP_RESET, N.OP_BARRIER):
            raise ValueError(f"op {i}: unknown kind {k}")
    qs = {i: _qubits(ops[i]) for i in pending}
    pos = list(range(n))   # logical qubit -> position
    at = list(range(n))    # position -> logical qubit
    steps: list[Step] = []
    group: list[int] = []

    def flush():
        if group:
            steps.append(Step("gates", ops=_translate(ops, group, pos)))
            group.clear()

    def swap(gpos: int, lpos: int):
        flush()
        steps.append(Step("swap", global_bit=gpos - nl, local_q=lpos))
        a, b = at[gpos], at[lpos]
        at[gpos], at[lpos] = b, a
        pos[a], pos[b] = lpos, gpos

    while pending:
        blocked: set[int] = set()
        measure_waiting = False
        waiting: list[int] = []
        for j, i in enumerate(pending):
            if j >= window or len(blocked) == n:
                waiting.extend(pending[j:])
                break
            q = qs[i]
            is_m = int(kinds[i]) in (N.OP_MEASURE, N.OP_RESET)  # markers keep their order
            if (all(pos[x] < nl for x in q) and blocked.isdisjoint(q)
                    and not (is_m and measure_waiting)):
                if is_m:
                    flush()
                    if int(kinds[i]) == N.OP_MEASURE:
                        steps.append(Step("measure", local_q=pos[q[0]], step=step_of[i]))
                    else:
                        steps.append(Step("reset", local_q=pos[q[0]]))
                else:
                    group.append(i)
            else:
                waiting.append(i)
                blocked.update(q)
                measure_waiting |= is_m
        pending = waiting
        if not pending:
            break
        head = qs[pending[0]]
        if all(pos[x] < nl for x in head):
            continue  # the scan stopped at the window; keep going
        nxt = {}
        for j, i in enumerate(pending[:window]):
            for x in qs[i]:
                nxt.setdefault(x, j)
        for x in head:
            if pos[x] < nl:
                continue
            victims = [p for p in range(nl) if at[p] not in head]
            if not victims:
                raise ValueError("op needs more qubits than the local range holds")
            far = max(victims, key=lambda p: (nxt.get(at[p], 1 << 62), p))
            swap(pos[x], far)
    flush()
    # restore the identity layout: global positions first, then a local
    # permutation as exact SWAP gates (the planner's frame makes them free)
    for gp in range(nl, n):
        if at[gp] == gp:
            continue
        if pos[gp] >= nl:  # wanted qubit sits in another global position
            p = max(p for p in range(nl))
            swap(pos[gp], p)
        swap(gp, pos[gp])
    perm_ops = []
    for p in range(nl):
        while at[p] != p:
            t = at[p]
            perm_ops.append((p, t))
            a, b = at[p], at[t]
            at[p], at[t] = b, a
            pos[a], pos[b] = t, p
    if perm_ops:
        rec = np.zeros(len(perm_ops), N.OP_DTYPE)
        rec["kind"], rec["tag"], rec["nq"], rec["cbit"] = N.OP_GATE, Gate.SWAP.code, 2, -1
        rec["q"] = -1
        rec["src"], rec["param"], rec["payload"] = -1, -1, -1
        for j, (a, b) in enumerate(perm_ops):
            rec["q"][j, 0], rec["q"][j, 1] = a, b
            rec["mask"][j] = (1 << a) | (1 << b)
        steps.append(Step("gates", ops=rec))
    assert pos == list(range(n))
    return steps


def sample_shard(rank: int, nl: int, draws: np.ndarray, starts: np.ndarray, last: bool,
                 chunk_sums: np.ndarray, chunk_log2: int, probs_range) -> np.ndarray:
    """This rank's part of `sample` (engine.py:207-222) on a sharded state.

    The reference draws u * cum[-1] and takes searchsorted(cum, ., "right")
    on the sequential cumulative sum of |a_i|^2 over the whole state.  Here
    `starts` are the global cumulative masses before each rank (rank-order
    sums of the ranks' totals), `chunk_sums` this rank's fixed-order sums
    over chunks of 2^chunk_log2 local amplitudes.  A draw belongs to the
    rank whose mass interval holds it; inside the rank the chunk prefix
    finds its chunk, whose probabilities are fetched (`probs_range(offset,
    count)`) and summed sequentially from the carried prefix exactly as
    np.cumsum, then searched with side="right".  With one rank and one chunk
    this is the reference's arithmetic; otherwise the chunk and rank carries
    are regrouped sums, so a draw within ~1e-16 (relative) of a cumulative
    boundary may land on the neighbouring index -- the same caveat as the
    amplitudes' own rounding.  Returns the global index of
    every owned draw, -1 elsewhere.
    """
    out = np.full(draws.size, -1, np.int64)
    lo = float(starts[rank])
    own = draws >= lo
    if not last:
        own &= draws < float(starts[rank + 1])
    if not own.any():
        return out
    sums = np.asarray(chunk_sums, np.float64)
    n_chunks = sums.size
    clen = 1 << chunk_log2
    excl = np.empty(n_chunks, np.float64)
    excl[0] = 0.0
    if n_chunks > 1:
        np.cumsum(sums[:-1], out=excl[1:])
    incl = lo + np.cumsum(sums)          # approximate global chunk ends
    cache: dict[int, np.ndarray] = {}

    def chunk_cum(c: int, carry: float) -> np.ndarray:
        p = cache.get(c)
        if p is None:
            p = np.empty(clen, np.float64)
            probs_range(c * clen, clen, p)
            cache[c] = p
        return np.cumsum(np.concatenate(([carry], p)))[1:]

    base = rank << nl
    for j in np.nonzero(own)[0]:
        x = float(draws[j])
        c = min(int(np.searchsorted(incl, x, side="right")), n_chunks - 1)
        carry = lo + excl[c] if c else lo
        while c > 0 and x < carry:         # regrouped carry overshot: step back
            c -= 1
            carry = lo + excl[c] if c else lo
        local = clen * n_chunks - 1        # past every cumulative value: clip
        while c < n_chunks:
            cum = chunk_cum(c, carry)
            pos = int(np.searchsorted(cum, x, side="right"))
            if pos < clen:
                local = c * clen + pos
                break
            carry = float(cum[-1])
            c += 1
        out[j] = base + local
    return out


def replayable(ops: np.ndarray) -> bool:
    """Filter-shaped: every MEASURE is followed by a RESET of the same qubit and
    every RESET follows such a MEASURE (all accepted rejection-mode shots then
    take the same path, engine.py:431-474)."""
    marks = [(int(r["kind"]), int(r["q"][0])) for r in ops
             if int(r["kind"]) in (N.OP_MEASURE, N.OP_RESET)]
    if not marks or len(marks) % 2:
        return False
    return all(marks[i][0] == N.OP_MEASURE and marks[i + 1] == (N.OP_RESET, marks[i][1])
               for i in range(0, len(marks), 2))


def replay_rejection(path, n_steps: int, shots: int, rng):
    """Rejection-mode tallies from the accepted path (engine.py:436-463):
    `path` = [(is_measure, step, p)] of one pass along the all-zero outcomes; the
    Philox stream is consumed in the reference's order -- one draw per MEASURE and
    RESET of a shot until it is rejected, one more for an accepted shot's sample.
    Returns (accepted, step_rejections, unit draws of the accepted shots' samples).
    A reset draw of 1 (probability ~1e-16 when p < 1) leaves the path: raised."""
    step_rej = [0] * n_steps
    draws = []
    for _ in range(shots):
        rejected = False
        for is_m, step, p in path:
            u = rng.random()
            if is_m:
                if not u < p:
                    step_rej[step] += 1
                    rejected = True
                    break
            elif not u < p:
                raise NotImplementedError("a reset drew outcome 1: the shot leaves the "
                                          "accepted path (run it on one GPU)")
        if not rejected:
            draws.append(rng.random())
    return len(draws), step_rej, np.asarray(draws, np.float64)


def swap_count(steps: list[Step]) -> int:
    return sum(1 for s in steps if s.kind == "swap")


class ShardedState:
    """The local shard of an n-qubit state on this rank (torch.distributed
    supplies rank / world size and carries the NCCL id; the data path is the
    library's own NCCL communicator on the context's stream)."""

    def __init__(self, n_qubits: int, rank: int, world: int, device: int, nccl_id: bytes):
        g = world.bit_length() - 1
        if world < 1 or (1 << g) != world:
            raise ValueError("rank count must be a power of two")
        if n_qubits - g < 2:
            raise ValueError("need at least 2 local qubits per rank")
        self.n, self.g, self.nl = n_qubits, g, n_qubits - g
        self.rank, self.world = rank, world
        self.dev = N.Device(device)
        self.dev.call("nsb_state_init", self.nl)
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
        self.dev.call("nsb_comm_init", buf, world, rank)
        self.peer_swaps = False  # set by from_torch_distributed (IPC-mapped partner shards)
        self.reset()

    @staticmethod
    def unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        st = N.Status()
        N.check(N.lib().nsb_comm_unique_id(buf, ctypes.byref(st)), st)
        return bytes(buf)

    @classmethod
    def from_torch_distributed(cls, n_qubits: int, device: int | None = None,
                               peer_swaps: bool | None = None):
        """Collective: rank 0 makes the NCCL id, torch.distributed broadcasts it.
        With peer_swaps (default: on unless NSB_SWAP_NCCL=1) the ranks also
        exchange CUDA IPC handles of their shards, and qubit swaps run as one
        peer-memory kernel over NVLink (nsb_shard_swap_p2p) instead of
        pack / NCCL send-recv / unpack."""
        import os
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        box = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", rank))
        st = cls(n_qubits, rank, world, device, box[0])
        if peer_swaps is None:
            peer_swaps = os.environ.get("NSB_SWAP_NCCL", "0") == "0"
        if peer_swaps and world > 1:
            h = (ctypes.c_uint8 * 64)()
            st.dev.call("nsb_shard_ipc_handle", h)
            handles = [None] * world
            dist.all_gather_object(handles, bytes(h))
            buf = (ctypes.c_uint8 * (64 * world)).from_buffer_copy(b"".join(handles))
            st.dev.call("nsb_shard_open_peers", buf)
            st.peer_swaps = True
        return st

    def close(self):
        """Collective when peer shards are mapped: every rank unmaps its
        partners' shards and the ranks rendezvous before any shard is freed."""
        if getattr(self, "peer_swaps", False) and self.dev.handle:
            self.dev.call("nsb_shard_close_peers")
            self.peer_swaps = False
        self.dev.close()

    # -- collectives -----------------------------------------------------------
    def allgather(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, np.float64).reshape(-1)
        out = np.zeros(v.size * self.world, np.float64)
        self.dev.call("nsb_shard_allgather", N.ptr(v), v.size, N.ptr(out))
        return out.reshape(self.world, v.size)

    def _sum(self, local: float) -> float:
        total = 0.0
        for x in self.allgather([local])[:, 0]:  # rank order on every rank
            total += float(x)
        return total

    def norm(self) -> float:
        out = ctypes.c_double(0.0)
        self.dev.call("nsb_state_norm2", ctypes.byref(out))
        return float(np.sqrt(self._sum(out.value)))

    def sample(self, shots: int, seed, chunk_log2: int = 13) -> dict[str, int]:
        """Collective `sample` (engine.py:194-222) of the full n-qubit state:
        every rank draws the same Philox stream, owns the draws inside its
        probability mass, locates them from device chunk sums plus one
        fetched chunk per hit, and the indices are all-gathered; returns the
        reference's {bitstring: count} on every rank (sample_shard)."""
        from .engine import _as_rng, bitstring
        if shots < 0:
            raise ValueError("shots must be nonnegative")
        rng = _as_rng(seed)
        if shots == 0:
            return {}
        return self.sample_draws(rng.random(shots), chunk_log2)

    def sample_draws(self, units: np.ndarray, chunk_log2: int = 13) -> dict[str, int]:
        """`sample` for given unit draws (u in [0, 1), scaled by the total mass as
        engine.py:217 scales rng.random(shots)); collective."""
        from .engine import bitstring
        shots = len(units)
        if shots == 0:
            return {}
        clog = max(0, min(int(chunk_log2), self.nl))
        sums = np.empty(1 << (self.nl - clog), np.float64)
        self.dev.call("nsb_prob_chunk_sums", clog, N.ptr(sums))
        total_local = float(np.cumsum(sums)[-1])
        totals = self.allgather([total_local])[:, 0]
        starts = np.zeros(self.world + 1, np.float64)
        for r in range(self.world):  # rank order on every rank
            starts[r + 1] = starts[r] + totals[r]
        draws = np.asarray(units, np.float64) * starts[-1]

        def fetch(off, count, out):
            self.dev.call("nsb_probabilities_range", off, count, N.ptr(out))

        mine = sample_shard(self.rank, self.nl, draws, starts, self.rank == self.world - 1,
                            sums, clog, fetch)
        idx = self.allgather(mine.astype(np.float64)).max(axis=0).astype(np.int64)
        np.clip(idx, 0, (1 << self.n) - 1, out=idx)
        values, counts = np.unique(idx, return_counts=True)
        return {bitstring(int(v), self.n): int(c) for v, c in zip(values, counts)}

    def reset(self):
        """|0...0>: amplitude 1 on rank 0, zeros elsewhere (on the device)."""
        self.dev.call("nsb_shard_reset")

    def upload(self, full: np.ndarray):
        """Load this rank's slice of a full host state (tests, small n)."""
        lo = self.rank << self.nl
        sl = np.ascontiguousarray(full[lo: lo + (1 << self.nl)], np.complex128)
        self.dev.call("nsb_state_upload", N.ptr(sl))

    def download(self) -> np.ndarray:
        host = np.empty(1 << self.nl, np.complex128)
        self.dev.call("nsb_state_download", N.ptr(host))
        return host

    # -- execution --------------------------------------------------------------
    def compile(self, ops, params, payloads, window: int = 4096) -> "ShardedProgram":
        """Schedule an MMA op stream and upload one device plan per gate group."""
        return ShardedProgram(self, schedule(ops, self.n, self.g, window), params, payloads)

    def run_rejection(self, ops, params, payloads, shots: int, seed, window: int = 4096):
        """Rejection mode (engine.py:431-474) on the sharded state, for
        filter-shaped circuits: one collective pass along the accepted path
        (exact plans: every gate runs), the Philox stream replayed on the host
        identically on every rank, the accepted shots' samples drawn from the
        final sharded state.  Returns (accepted, {bitstring: count},
        step_rejections), the reference's tallies."""
        from .engine import _as_rng
        if not replayable(ops):
            raise NotImplementedError("sharded rejection mode needs a filter-shaped circuit "
                                      "(each MEASURE followed by a RESET of the same qubit)")
        rng = _as_rng(seed)
        n_steps = int(np.count_nonzero(ops["kind"] == N.OP_MEASURE))
        prog = ShardedProgram(self, schedule(ops, self.n, self.g, window, keep_resets=True),
                              params, payloads)
        try:
            self.reset()
            path, reachable = prog.run_path()
        finally:
            prog.close()
        del reachable  # a path cut at P(0) = 0 rejects every shot there (u < 0 never holds)
        accepted, step_rej, units = replay_rejection(path, n_steps, shots, rng)
        counts = self.sample_draws(units) if accepted else {}
        return accepted, counts, step_rej

    def run_mma(self, ops, params, payloads, eps: float = EPS_MMA, window: int = 4096):
        prog = self.compile(ops, params, payloads, window)
        try:
            probs = prog.run(eps)
            self.last_overlapped_passes = prog.overlapped_passes
        finally:
            prog.close()
        return [probs[k] for k in sorted(probs)], prog.steps

    def timer_start(self):
        self.dev.call("nsb_timer_start")

    def timer_stop(self) -> float:
        ms = ctypes.c_double(0.0)
        self.dev.call("nsb_timer_stop", ctypes.byref(ms))
        return float(ms.value)


class ShardedProgram:
    """A schedule with its gate groups compiled into device plans (nsb_plan)
    bound to one rank's context."""

    def __init__(self, state: ShardedState, steps: list[Step], params, payloads):
        self.state, self.steps = state, steps
        self.plans: list[tuple[ctypes.c_void_p, int] | None] = []
        st = N.Status()
        try:
            for s in steps:
                if s.kind != "gates":
                    self.plans.append(None)
                    continue
                h = ctypes.c_void_p()
                # exact: assertions are measured between the groups by the host
                N.check(N.lib().nsb_plan_create_ex(state.dev.handle, N.ptr(s.ops), len(s.ops),
                                                   N.ptr(params), N.ptr(payloads.view(np.float64)),
                                                   N.PLAN_EXACT, ctypes.byref(h),
                                                   ctypes.byref(st)), st)
                info = N.PlanInfo()
                N.lib().nsb_plan_info_get(h, ctypes.byref(info))
                self.plans.append((h, int(info.n_items)))
        except Exception:
            self.close()
            raise
        self.n_swaps = swap_count(steps)
        self.overlapped_passes = 0  # gate passes run under a swap (last run)

    def close(self):
        for e in self.plans:
            if e is not None:
                N.lib().nsb_plan_destroy(e[0])
        self.plans = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _swap(self, i: int, s: Step, chunk_amps: int) -> bool:
        """Execute swap step i.  With peer-memory swaps the swap is overlapped
        with the first item of the gate step that follows it: that item's
        chunkable passes run chunk by chunk as the swapped chunks land.
        NSB_SWAP_OVERLAP selects how the chunks move: "ce" (default) on the
        copy engines (nsb_shard_swap_overlap_ce: no SMs taken from the gate
        passes), "1" with a swap kernel on some SMs (nsb_shard_swap_overlap:
        measured slower), "0" not overlapped (the swap
        kernel, then the item).  Returns True when that item has run."""
        S = self.state
        nxt = self.plans[i + 1] if i + 1 < len(self.plans) else None
        mode = os.environ.get("NSB_SWAP_OVERLAP", "ce")
        if S.peer_swaps and nxt is not None and nxt[1] > 0 and mode in ("1", "ce"):
            n = ctypes.c_int32(0)
            bits = int(os.environ.get("NSB_SWAP_CHUNK_BITS", "3"))
            if mode == "ce":
                S.dev.call("nsb_shard_swap_overlap_ce", s.global_bit, s.local_q, nxt[0], 0, bits,
                           int(os.environ.get("NSB_SWAP_STAGE_BYTES", "0")), ctypes.byref(n))
            else:
                S.dev.call("nsb_shard_swap_overlap", s.global_bit, s.local_q, nxt[0], 0, bits,
                           int(os.environ.get("NSB_SWAP_CTAS", "0")), ctypes.byref(n))
            self.overlapped_passes += n.value
            return True
        if S.peer_swaps:
            S.dev.call("nsb_shard_swap_p2p", s.global_bit, s.local_q)
        else:
            S.dev.call("nsb_shard_swap", s.global_bit, s.local_q, chunk_amps)
        return False

    def _gates(self, plan, first: int):
        h, n_items = plan
        st = N.Status()
        for i in range(first, n_items):
            N.check(N.lib().nsb_plan_run_segment(self.state.dev.handle, h, i, ctypes.byref(st)), st)

    def run(self, eps: float = EPS_MMA, chunk_amps: int = 0,
            times: dict | None = None) -> dict[int, float]:
        """Execute on this rank (collective with the other ranks); returns
        {step: p0}.  Raises FilterAssertionError on every rank when a
        post-selection probability falls below eps.  With `times`, each step
        is bracketed by device events and its time (ms) is added under its
        kind ("gates" / "swap" / "measure"; an overlapped swap and the gate
        item under it: "swap+gates")."""
        S = self.state
        probs: dict[int, float] = {}
        self.overlapped_passes = 0
        done_first = False  # item 0 of this gate step ran under the swap before it
        for i, (s, plan) in enumerate(zip(self.steps, self.plans)):
            if times is not None:
                S.timer_start()
            kind = s.kind
            if s.kind == "gates":
                self._gates(plan, 1 if done_first else 0)
                done_first = False
            elif s.kind == "swap":
                done_first = self._swap(i, s, chunk_amps)
                if done_first:
                    kind = "swap+gates"
            else:
                p = ctypes.c_double(0.0)
                S.dev.call("nsb_branch_probability", s.local_q, 0, ctypes.byref(p))
                p0 = S._sum(p.value)
                probs[s.step] = p0
                if p0 < eps:
                    raise FilterAssertionError(s.step, p0)
                S.dev.call("nsb_project", s.local_q, 0, p0)
            if times is not None:
                times[kind] = times.get(kind, 0.0) + S.timer_stop()
        return probs

    def run_path(self) -> tuple[list, bool]:
        """Rejection mode's accepted path (collective): gates as in run(); at a
        MEASURE the summed P(0) is recorded and the shards collapse onto 0; at a
        RESET likewise, with its renormalisation (engine.py:451-455).  Returns
        ([(is_measure, step, p)], reachable); an outcome-0 probability of 0 ends
        the path (every shot stops there)."""
        S = self.state
        path = []
        done_first = False
        for i, (s, plan) in enumerate(zip(self.steps, self.plans)):
            if s.kind == "gates":
                self._gates(plan, 1 if done_first else 0)
                done_first = False
            elif s.kind == "swap":
                done_first = self._swap(i, s, 0)
            else:
                p = ctypes.c_double(0.0)
                S.dev.call("nsb_branch_probability", s.local_q, 0, ctypes.byref(p))
                p0 = S._sum(p.value)
                path.append((s.kind == "measure", s.step, p0))
                if p0 <= 0.0:
                    return path, False
                S.dev.call("nsb_project", s.local_q, 0, p0)
        return path, True

    def plan_totals(self) -> dict:
        """Summed nsb_plan_info counters over the gate groups."""
        tot: dict[str, int] = {}
        for e in self.plans:
            if e is None:
                continue
            info = N.PlanInfo()
            N.lib().nsb_plan_info_get(e[0], ctypes.byref(info))
            for k, _ in N.PlanInfo._fields_:
                if k != "tile_qubits":
                    tot[k] = tot.get(k, 0) + int(getattr(info, k))
        return tot
