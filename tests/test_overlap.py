"""Chunked pass execution: the building block of overlapped qubit swaps.

nsb_shard_swap_overlap (device.cu) runs the gate item after a qubit swap
chunk by chunk -- chunk c of the item's passes as soon as chunk c of the swap
has landed.  That is only valid when every pass of the chunked prefix leaves
the chunk qubits out of its tiles (a pass never moves data between tiles).
These tests pin (1) the prefix / chunk-qubit choice (nsb_host_plan_chunk_prefix),
(2) on the CPU executor, that running the prefix chunk by chunk gives the
plain run's state exactly, and (3) on the GPU, the same for k_blocked's chunk
restriction (nsb_plan_run_segment_chunked).  The 2- and 4-rank overlapped swap
itself runs in tests/sharded_gpu_job.py (test_sharded.py).
"""

import ctypes
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests"):
    sys.path.insert(0, str(p))

import plan_exec as PE  # noqa: E402
from paper_2310_17739_b200 import _native as N  # noqa: E402
from paper_2310_17739_b200 import workloads as W  # noqa: E402


def _plan(n, layers, seed):
    wl = W.layered_workload(n, layers=layers, seed=seed)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    return wl, fops, pool, PE.HostPlan(fops, wl.params, pool, n, 296)


def _chunk_prefix(hp, item, avoid_q, want):
    n_pass, cm = ctypes.c_int32(-1), ctypes.c_uint64(0)
    assert N.lib().nsb_host_plan_chunk_prefix(hp.h, item, avoid_q, want, ctypes.byref(n_pass),
                                              ctypes.byref(cm)) == 0
    return int(n_pass.value), int(cm.value)


def _tiles(P):
    return {int(q) for q in P["tq"][: int(P["k"])]}


@pytest.mark.parametrize("n,seed", [(16, 1), (18, 2), (20, 3)])
def test_chunk_prefix_properties(n, seed):
    _, _, _, hp = _plan(n, 6, seed)
    assert hp.items[0][0] == 0  # a gate item
    pb, pe = int(hp.items[0][1]), int(hp.items[0][2])
    rng = np.random.default_rng(seed)
    seen = 0
    for avoid in [-1, 0, n - 1] + [int(x) for x in rng.integers(0, n, 3)]:
        for want in (1, 2, 3):
            n_pass, cm = _chunk_prefix(hp, 0, avoid, want)
            bits = bin(cm).count("1")
            if n_pass == 0:
                assert cm == 0
                continue
            seen += 1
            assert 1 <= bits <= want and 0 < n_pass <= pe - pb
            assert avoid < 0 or not (cm >> avoid) & 1
            used = set() if avoid < 0 else {avoid}
            for P in hp.passes[pb:pb + n_pass]:
                assert not any((cm >> q) & 1 for q in _tiles(P))  # chunk qubits stay out of tiles
                used |= _tiles(P)
            # the chunk qubits are the highest qubits the prefix leaves free
            free = sorted(set(range(n)) - used)
            assert sorted(q for q in range(n) if (cm >> q) & 1) == free[-bits:]
            # maximal: one more pass would leave fewer than `bits` qubits free
            if pb + n_pass < pe:
                assert len(set(range(n)) - used - _tiles(hp.passes[pb + n_pass])) < bits
    assert seen > 0


def test_chunk_prefix_bad_items():
    _, _, _, hp = _plan(14, 2, 7)
    assert _chunk_prefix(hp, -1, -1, 3) == (0, 0)
    assert _chunk_prefix(hp, len(hp.items), -1, 3) == (0, 0)
    assert _chunk_prefix(hp, 0, -1, 0) == (0, 0)


@pytest.mark.parametrize("n,seed,want", [(16, 4, 3), (18, 5, 2), (18, 6, 1)])
def test_chunked_execution_is_the_plain_run(n, seed, want):
    """CPU executor: the prefix run chunk by chunk (every chunk through all
    prefix passes before the next chunk starts), then the rest, gives the
    plain run's state bit for bit."""
    _, _, _, hp = _plan(n, 4, seed)
    pb, pe = int(hp.items[0][1]), int(hp.items[0][2])
    n_pass, cm = _chunk_prefix(hp, 0, n // 2, want)
    assert n_pass > 0
    rng = np.random.default_rng(seed)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    plain = psi.copy()
    PE.run_passes(hp, hp.passes[pb:pe], plain)
    chunked = psi.copy()
    bits = [q for q in range(n) if (cm >> q) & 1]
    for c in range(1 << len(bits)):
        cv = sum(((c >> j) & 1) << q for j, q in enumerate(bits))
        PE.run_passes(hp, hp.passes[pb:pb + n_pass], chunked, chunk=(cm, cv))
    PE.run_passes(hp, hp.passes[pb + n_pass:pe], chunked)
    assert np.array_equal(plain, chunked)


def test_chunk_outside_the_prefix_is_refused():
    """The executor (like the planner) refuses a chunk qubit inside a tile."""
    _, _, _, hp = _plan(14, 2, 8)
    P = hp.passes[:1]
    q = sorted(_tiles(P[0]))[-1]
    with pytest.raises(AssertionError, match="chunk qubits inside"):
        PE.run_passes(hp, P, np.zeros(1 << 14, np.complex128), chunk=(1 << q, 0))


@pytest.mark.gpu
@pytest.mark.parametrize("n,want", [(20, 3), (22, 2), (24, 1)])
def test_run_item_chunked_gpu(n, want):
    """k_blocked's chunk restriction on the GPU: item 0 of a layered circuit
    run with its prefix chunk by chunk equals the plain run bit for bit."""
    from paper_2310_17739_b200.engine import DeviceProgram, StateVector
    wl, fops, pool, _ = _plan(n, 4, n)
    rng = np.random.default_rng(n)
    psi = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    psi /= np.linalg.norm(psi)
    a = StateVector.from_amplitudes(psi)
    pa = DeviceProgram(a, fops, wl.params, pool, exact=True)
    b = StateVector.from_amplitudes(psi)
    pb = DeviceProgram(b, fops, wl.params, pool, exact=True)
    kinds = pa.items()
    assert kinds and kinds[0][0] == 0
    pa.run_item(0)
    n_chunked = pb.run_item_chunked(0, want)
    assert n_chunked > 0
    assert np.array_equal(a.amps, b.amps)
    for i in range(1, len(kinds)):  # the remaining items, plain on both
        pa.run_item(i)
        pb.run_item(i)
    assert np.array_equal(a.amps, b.amps)
