"""Planner verification on the CPU: the exported device program (relabeling
frame, pivots, dual rows, pass tiling, measurement epilogues) executed by
tests/plan_exec.py must reproduce the oracle's final state and assertion
probabilities.  The GPU tests then check that k_blocked executes the same
program faithfully."""

import numpy as np
import pytest

import nucsim_oracle as O
import plan_exec as PE
from circuit_io import oracle_from_circuit, to_circuit
from paper_2310_17739_b200 import Circuit, Gate, fuse_pipeline
from paper_2310_17739_b200._pack import pack
from test_engine_gpu import ladder_circuit, random_filter_like


def executable(c):
    end = len(c.instructions)
    while end and c.instructions[end - 1].gate.value in ("measure", "barrier"):
        end -= 1
    return pack(c, c.instructions[:end])


def check(c, workers=148):
    n = c.n_qubits
    pk = executable(c)
    plan = PE.HostPlan(pk.ops, pk.params, pk.payloads, n, workers)
    try:
        want_p, _, want_state, _ = O.run_mma(oracle_from_circuit(c), n, 1, 0)
    except O.OracleAssertion:
        pytest.skip("dead assertion branch")
    probs, state = PE.run_mma(plan, workers=workers)
    assert probs == pytest.approx(want_p, abs=1e-12)
    err = np.linalg.norm(state - want_state) / np.linalg.norm(want_state)
    assert err < 1e-10, err
    return plan


@pytest.mark.parametrize("n", [6, 8, 11, 13])
def test_random_filter_like(n):
    rng = np.random.default_rng(1000 + n)
    c = random_filter_like(rng, n, blocks=3, per_block=50)
    check(c)
    check(fuse_pipeline(c)[0])


@pytest.mark.parametrize("n,terms", [(7, 30), (10, 30), (13, 25)])
def test_ladders_through_the_frame(n, terms):
    rng = np.random.default_rng(50 + n)
    c = ladder_circuit(rng, n, terms)
    for circ in (c, fuse_pipeline(c)[0]):
        plan = check(circ)
        assert len(plan.groups) <= len(plan.ops) + len(plan.passes)


@pytest.mark.parametrize("n,workers", [(14, 1), (14, 3), (14, 148), (15, 5), (16, 3)])
def test_small_tiles_multi_pass(n, workers):
    """n > 12 forces several tiles, batches of tiles and multiple passes."""
    rng = np.random.default_rng(7 + n)
    c = ladder_circuit(rng, n, 12, blocks=2)
    check(fuse_pipeline(c)[0], workers)


def test_golden_filter8_plan(golden):
    d = golden("filter8")
    for pre in ("fused_", "in_"):
        check(to_circuit(d, pre))


def test_parallel_planning_matches_serial(monkeypatch):
    """Gate runs between markers are planned on host threads; the merged
    program must be byte-identical to the serial one."""
    from paper_2310_17739_b200 import workloads as W
    wl = W.filter_workload(11, 6, n_steps=4, seed=3, hop_range=8)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    assert len(exe) >= 20000

    def view():
        hp = PE.HostPlan(exe, wl.params, pool, wl.n_qubits, workers=296)
        return (hp.passes.tobytes(), hp.mma_passes.tobytes(), hp.groups.tobytes(),
                hp.ops.tobytes(), hp.mats.tobytes(), hp.items.tobytes())

    par = view()
    monkeypatch.setenv("NSB_PLAN_SERIAL", "1")
    ser = view()
    assert par == ser


@pytest.mark.parametrize("fusion", [True, False])
def test_group_fusion_whole_octet_ops(monkeypatch, fusion):
    """Planner group fusion (fuse_group): on a deep-circuit-shaped workload
    the product of a group's gates replaces them by one whole-octet op
    (axis-targeted blocks or an octet diagonal); the program must still
    reproduce the full-state oracle."""
    import shard_exec as SE
    from paper_2310_17739_b200 import workloads as W
    if not fusion:
        monkeypatch.setenv("NSB_NO_GROUP_FUSION", "1")
    wl = W.filter_workload(9, trotter=1, n_steps=2, n_scatter=4, trial="10" * 5)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    n = wl.n_qubits
    plan = PE.HostPlan(exe, wl.params, pool, n, 148)
    whole = int(((plan.ops["pat"] >= 6) & (plan.ops["pat"] <= 12)).sum())  # not register ops
    assert (whole > 0) == fusion
    want_p, want = SE.full_mma(exe, wl.params, pool, n)
    probs, state = PE.run_mma(plan)
    assert probs == pytest.approx(want_p, abs=1e-12)
    assert np.linalg.norm(state - want) / np.linalg.norm(want) < 1e-10


# ---------------------------------------------------------------------------
# the HBM-regime tile policy (n > 22: every tile holds qubits 0..2) at sizes the
# oracle finishes quickly, forced with NSB_LOW_QUBITS / NSB_TILE_QUBITS


@pytest.mark.parametrize("n,low,tile", [(12, 3, 11), (13, 3, 9), (14, 3, 10), (15, 3, 11),
                                        (16, 3, 8), (16, 3, 11), (18, 3, 11), (17, 3, 10),
                                        (14, 1, 9), (13, 0, 7)])
def test_hbm_tile_policy_filter_workload(monkeypatch, n, low, tile):
    """Deep-circuit shape (JW shell-model filter, native emitter + fusion) under
    the tile policy C4/C5 run with: the exported program reproduces the
    full-state oracle's assertion probabilities and final state."""
    import shard_exec as SE
    from paper_2310_17739_b200 import workloads as W
    monkeypatch.setenv("NSB_LOW_QUBITS", str(low))
    monkeypatch.setenv("NSB_TILE_QUBITS", str(tile))
    if n >= 15:  # all batches of a pass at once (same arithmetic, no per-CTA asserts)
        monkeypatch.setenv("NSB_PLAN_EXEC_CHECK", "0")
    wl = W.filter_workload(n - 1, trotter=1, n_steps=2, n_scatter=2, hop_range=3,
                           pair_density=0.1, trial="10" * ((n - 1) // 2) + "1" * ((n - 1) % 2))
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    plan = PE.HostPlan(exe, wl.params, pool, n, 148)
    assert plan.k == tile
    # full tiles holding qubits 0..2 move by TMA: pass-edge groups on swz_tma
    assert plan.tma == (low >= 3 and tile == 11)
    for p in plan.mma_passes:
        tq = set(int(x) for x in p["tq"][: int(p["k"])])
        assert set(range(low)) <= tq, "tile lacks the always-tiled low qubits"
    want_p, want = SE.full_mma(exe, wl.params, pool, n)
    probs, state = PE.run_mma(plan)
    assert probs == pytest.approx(want_p, abs=1e-12)
    assert np.linalg.norm(state - want) / np.linalg.norm(want) < 1e-10


@pytest.mark.parametrize("n,tile,tma", [(14, 11, "1"), (14, 11, "0"), (16, 10, "1"),
                                        (17, 11, "1")])
def test_hbm_tile_policy_ladders(monkeypatch, n, tile, tma):
    monkeypatch.setenv("NSB_LOW_QUBITS", "3")
    monkeypatch.setenv("NSB_TILE_QUBITS", str(tile))
    monkeypatch.setenv("NSB_TMA", tma)
    rng = np.random.default_rng(900 + n)
    c = ladder_circuit(rng, n, 14, blocks=2)
    check(fuse_pipeline(c)[0])


def test_default_policy_switches_at_l2_size():
    """The planner picks the HBM policy (qubits 0..2 tiled) above 22 qubits and
    the L2 policy (qubits 0, 1) at or below (planner.h kL2ResidentQubits)."""
    from paper_2310_17739_b200 import workloads as W
    for n, low in ((21, 2), (22, 2), (23, 3), (24, 3)):
        wl = W.layered_workload(n, 1, 5)
        fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
        plan = PE.HostPlan(fops, wl.params, pool, n, 296)
        assert plan.tma == (low == 3)
        for p in plan.mma_passes:
            tq = set(int(x) for x in p["tq"][: int(p["k"])])
            assert set(range(low)) <= tq
            if low == 2:
                continue
            assert 2 in tq


@pytest.mark.parametrize("pairs", [((4, 6), (8, 10), (12, 14)),
                                   ((4, 6), (8, 10), (12, 14), (1, 15), (3, 5)),
                                   ((3, 4), (6, 7), (9, 10), (12, 13))])
def test_tma_edges_keep_warp_local_sweeps_race_free(monkeypatch, pairs):
    """TMA plans load the first sweep and store the last one under the TMA
    swizzle: a warp-local transition across such an edge would let one warp
    overwrite slots another warp is still reading (the executor asserts, per
    warp, both read-after-write and write-after-read slot sets)."""
    monkeypatch.setenv("NSB_LOW_QUBITS", "3")
    monkeypatch.setenv("NSB_TMA", "1")
    monkeypatch.setenv("NSB_PLAN_EXEC_CHECK", "1")
    n = 16
    c = Circuit(n, [("c", 1)])
    for a, b in pairs:
        c.gate_op(Gate.CZ, (a, b), ())
        c.gate_op(Gate.RZZ, (b, a), (0.3,))
    pk = executable(c)
    plan = PE.HostPlan(pk.ops, pk.params, pk.payloads, n, 296)
    assert plan.tma
    rng = np.random.default_rng(len(pairs))
    state = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    want = state.copy()
    PE.run_passes(plan, plan.mma_passes, state, workers=296)
    monkeypatch.setenv("NSB_TMA", "0")  # the same circuit planned without TMA edges
    ref = PE.HostPlan(pk.ops, pk.params, pk.payloads, n, 296)
    assert not ref.tma
    PE.run_passes(ref, ref.mma_passes, want, workers=296)
    assert np.allclose(state, want, rtol=0, atol=1e-12)
