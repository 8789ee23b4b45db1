"""Parity at the benchmarked sizes on the GPU.

* deep21 (BASELINE config 3, the headline: 21 qubits, 1 948 482 input gates,
  983 376 fused, 8 assertions) and rand28 (config 4: 28 qubits, 4 GiB state,
  HBM tile policy) executed by the blocked kernel (one cooperative launch)
  against the per-op path of the same fused stream (NSB_FORCE_PER_OP=1: one
  k_apply1 / k_apply2 launch per fused gate and the per-op measurement
  kernels, each tested against the oracle and the reference's kernel
  goldens in test_engine_gpu.py): final states within 1e-10 relative L2,
  assertion probabilities within 1e-12.
* the HBM tile policy (n > 22: tiles hold qubits 0..2) at 24 qubits against
  the oracle's einsum kernels on the host, amplitude by amplitude.
* the blocked kernel under forced tile policies (NSB_LOW_QUBITS = 3, several
  NSB_TILE_QUBITS) at 12..18 qubits against the oracle.
"""

import os

import numpy as np
import pytest

import nucsim_oracle as O
from paper_2310_17739_b200 import workloads as W
from paper_2310_17739_b200.engine import DeviceProgram, StateVector

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _blocked_and_per_op(monkeypatch, exe, params, pool, n):
    state = StateVector(n)
    prog = DeviceProgram(state, exe, params, pool)
    assert prog.info.n_passes > 0
    p_blocked = prog.run_mma()
    a_blocked = state.amps.copy()
    del prog
    monkeypatch.setenv("NSB_FORCE_PER_OP", "1")
    state.restart()
    per_op = DeviceProgram(state, exe, params, pool)
    assert per_op.info.n_passes == 0  # the item path: one launch per gate
    p_op = per_op.run_mma()
    a_op = state.amps
    monkeypatch.delenv("NSB_FORCE_PER_OP")
    return p_blocked, a_blocked, p_op, a_op, per_op


def test_deep21_full_headline_blocked_matches_per_op(monkeypatch):
    wl = W.filter_workload(20, trotter=18, n_steps=8, n_scatter=8, trial="10" * 10)
    assert wl.input_gates == 1948482
    fops, pool, stats = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    assert stats["gates_after"] == 983376
    exe = wl.executable(fops)
    pb, ab, po, ao, per_op = _blocked_and_per_op(monkeypatch, exe, wl.params, pool, 21)
    assert per_op.info.n_items > 983376
    assert len(pb) == len(po) == 8
    np.testing.assert_allclose(pb, po, rtol=0, atol=1e-12)
    assert rel_l2(ab, ao) < 1e-10
    assert abs(np.linalg.norm(ab) - 1.0) < 1e-10


def test_rand28_blocked_matches_per_op(monkeypatch):
    wl = W.layered_workload(28, layers=20)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    pb, ab, po, ao, _ = _blocked_and_per_op(monkeypatch, exe, wl.params, pool, 28)
    assert pb == po == []
    assert rel_l2(ab, ao) < 1e-10
    assert abs(np.linalg.norm(ab) - 1.0) < 1e-10


def _oracle_state(exe, params, pool, n):
    import shard_exec as SE
    return SE.full_mma(exe, params, pool, n)


@pytest.mark.parametrize("n,layers", [(24, 4)])
def test_hbm_policy_layered_against_oracle(n, layers):
    """Default HBM policy (n > 22) against the oracle's einsum on the host."""
    wl = W.layered_workload(n, layers, 4242)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(n)
    prog = DeviceProgram(state, exe, wl.params, pool)
    assert prog.info.tile_qubits == 11
    prog.run_mma()
    _, want = _oracle_state(exe, wl.params, pool, n)
    assert rel_l2(state.amps, want) < 1e-10


@pytest.mark.parametrize("n,tile", [(12, 11), (14, 9), (16, 10), (17, 11), (18, 11), (18, 8)])
def test_forced_hbm_policy_filter_workload_against_oracle(monkeypatch, n, tile):
    """NSB_LOW_QUBITS=3 (the policy C4 / C5 run with) on the deep-circuit shape,
    several tile sizes, through the blocked kernel on the GPU."""
    monkeypatch.setenv("NSB_LOW_QUBITS", "3")
    monkeypatch.setenv("NSB_TILE_QUBITS", str(tile))
    wl = W.filter_workload(n - 1, trotter=1, n_steps=2, n_scatter=4, hop_range=6,
                           pair_density=0.2, trial="10" * ((n - 1) // 2) + "1" * ((n - 1) % 2))
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    want_p, want = _oracle_state(exe, wl.params, pool, n)
    state = StateVector(n)
    prog = DeviceProgram(state, exe, wl.params, pool)
    assert prog.info.tile_qubits == tile
    got_p = prog.run_mma()
    assert got_p == pytest.approx(want_p, abs=1e-12)
    assert rel_l2(state.amps, want) < 1e-10
