"""TMA tiles on the GPU (planner.h "TMA tiles", csrc/device.cu k_blocked<.., true>).

Plans whose tiles hold qubits 0..2 at full size move the tiles of eligible
passes by cp.async.bulk.tensor; the arithmetic per amplitude is the same as on
the cp.async path, so the final state must be bit-identical with TMA off
(NSB_TMA=0) -- and it must match the oracle (tests/test_fullsize_parity_gpu.py
covers the 24-qubit HBM policy and the forced policy at 12..18 qubits).
"""

import numpy as np
import pytest

from paper_2310_17739_b200 import Circuit, Gate
from paper_2310_17739_b200 import workloads as W
from paper_2310_17739_b200._pack import pack
from paper_2310_17739_b200.engine import DeviceProgram, StateVector

pytestmark = pytest.mark.gpu


def _tma_passes(exe, params, pool, n):
    import plan_exec as PE
    plan = PE.HostPlan(exe, params, pool, n, 296)
    return sum(int(p["tma"]) for p in plan.mma_passes)


def _run(exe, params, pool, n, amps=None):
    state = StateVector(n)
    if amps is not None:
        state.amps = amps
    prog = DeviceProgram(state, exe, params, pool)
    probs = prog.run_mma()
    return probs, state.amps.copy()


@pytest.mark.parametrize("n,layers,seed", [(23, 6, 1), (24, 4, 2), (25, 3, 2)])
def test_tma_plan_bit_identical_to_cp_async(monkeypatch, n, layers, seed):
    wl = W.layered_workload(n, layers, seed)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    monkeypatch.setenv("NSB_TMA", "1")
    assert _tma_passes(exe, wl.params, pool, n) > 0
    _, a_tma = _run(exe, wl.params, pool, n)
    monkeypatch.setenv("NSB_TMA", "0")
    _, a_ref = _run(exe, wl.params, pool, n)
    assert np.array_equal(a_tma, a_ref)


@pytest.mark.parametrize("pairs", [((4, 6), (8, 10), (12, 14), (16, 18)),
                                   ((3, 4), (6, 7), (9, 10), (12, 13)),
                                   ((6, 7), (8, 9), (13, 14), (17, 18)),
                                   ((9, 10), (11, 12), (13, 14), (17, 18))])
def test_tma_tile_layout_moves_every_amplitude_home(monkeypatch, pairs):
    """Amplitude i = i, diagonal +-1 gates: any misplaced copy shows as a wrong
    magnitude (forced HBM tile policy at 20 qubits: gaps, traversal strides,
    several copies per tile)."""
    monkeypatch.setenv("NSB_LOW_QUBITS", "3")
    monkeypatch.setenv("NSB_TMA", "1")
    n = 20
    c = Circuit(n, [("c", 1)])
    for a, b in pairs:
        c.gate_op(Gate.CZ, (a, b), ())
    pk = pack(c)
    amps = np.arange(1 << n, dtype=np.float64).astype(np.complex128)
    state = StateVector(n)
    state.amps = amps
    DeviceProgram(state, pk.ops, pk.params, pk.payloads).run_mma()
    idx = np.arange(1 << n)
    want = amps.copy()
    for a, b in pairs:
        want[(((idx >> a) & 1) & ((idx >> b) & 1)) == 1] *= -1
    assert np.array_equal(state.amps, want)


def test_tma_filter_circuit_with_assertions(monkeypatch):
    """Measured passes (collapse prologue, P(0) epilogue) in a TMA plan."""
    monkeypatch.setenv("NSB_LOW_QUBITS", "3")
    n = 16
    wl = W.filter_workload(n - 1, trotter=1, n_steps=2, n_scatter=4, hop_range=6,
                           pair_density=0.2, trial="10" * 7 + "1")
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    monkeypatch.setenv("NSB_TMA", "1")
    assert _tma_passes(exe, wl.params, pool, n) > 0
    p1, a1 = _run(exe, wl.params, pool, n)
    monkeypatch.setenv("NSB_TMA", "0")
    p0, a0 = _run(exe, wl.params, pool, n)
    assert p1 == p0
    assert np.array_equal(a1, a0)


def test_streamed_run_on_tma_plans(monkeypatch):
    """nsb_run_mma_streamed above 22 qubits: parts planned as TMA plans (their
    own tensor maps per part, fresh marker passes on cp.async) reproduce the
    single-launch program."""
    from paper_2310_17739_b200.engine import run_mma_streamed
    n = 23
    wl = W.filter_workload(n - 1, trotter=1, n_steps=2, n_scatter=2, hop_range=4,
                           pair_density=0.05, trial="10" * 11)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    assert _tma_passes(exe, wl.params, pool, n) > 0
    state = StateVector(n)
    p_one = DeviceProgram(state, exe, wl.params, pool).run_mma()
    a_one = state.amps.copy()
    state.restart()
    p_str = run_mma_streamed(state, exe, wl.params, pool)
    np.testing.assert_allclose(p_str, p_one, rtol=0, atol=1e-12)
    assert np.linalg.norm(state.amps - a_one) <= 1e-11
