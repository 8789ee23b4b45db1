"""GPU parity: the CUDA path (through the C ABI) against the reference's
golden vectors and the pinned oracle.  Tolerances follow north_star:
amplitudes 1e-10 relative L2 (kernels: 1e-12 max abs, as the reference's
own kernel tests), assertion probabilities 1e-12 absolute, samples and
rejection tallies exactly equal for the same seeds."""

import math

import numpy as np
import pytest

import nucsim_oracle as O
from circuit_io import oracle_from_circuit, to_circuit, to_oracle
from paper_2310_17739_b200 import (Circuit, FilterAssertionError, Gate, PauliHamiltonian,
                                   ProjectionError, StateVector, apply_1q, apply_2q, apply_dense,
                                   assert_measure, expectation_pauli, fuse_pipeline,
                                   measure_project, run, sample)
from paper_2310_17739_b200.engine import _as_rng, swap_conjugate

pytestmark = pytest.mark.gpu

X = np.array([[0, 1], [1, 0]], dtype=complex)


def vec(*amps):
    a = np.asarray(amps, dtype=complex)
    return a / np.linalg.norm(a)


def state_of(amps):
    return StateVector.from_amplitudes(np.asarray(amps, dtype=complex))


def golden_samples(d, prefix):
    k = int(d[prefix + "n"])
    return dict(zip(map(str, d[prefix + "keys"][:k]), map(int, d[prefix + "counts"][:k])))


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---------------------------------------------------------------------------
# kernels


def test_pair_and_quad_geometry():
    s = state_of(vec(1, 2, 3, 4))
    apply_1q(s, X, 1)
    assert np.allclose(s.amps, vec(3, 4, 1, 2), atol=1e-15)
    s = state_of(vec(1, 2, 3, 4))
    apply_1q(s, X, 0)
    assert np.allclose(s.amps, vec(2, 1, 4, 3), atol=1e-15)
    u = np.eye(4, dtype=complex)[[0, 2, 1, 3]]
    s = StateVector(3)
    s.amps[0] = 0
    s.amps[4] = 1.0
    apply_2q(s, u, 0, 2)
    assert np.argmax(np.abs(s.amps)) == 1


def test_kernels_against_golden(golden):
    d = golden("kernels")
    for i in range(int(d["n_kernels"])):
        s = state_of(d[f"k{i}_amps"])
        apply_dense(s, d[f"k{i}_u"], tuple(int(x) for x in d[f"k{i}_qubits"]))
        assert np.max(np.abs(s.amps - d[f"k{i}_out"])) <= 1e-12
        if d[f"k{i}_mp"] >= 0:
            s = state_of(d[f"k{i}_amps"])
            p = measure_project(s, int(d[f"k{i}_mq"]), 0)
            assert p == pytest.approx(float(d[f"k{i}_mp"]), abs=1e-14)
            assert np.max(np.abs(s.amps - d[f"k{i}_mout"])) <= 1e-12


@pytest.mark.parametrize("n", [1, 3, 5, 7])
def test_random_kernels_against_oracle(n):
    rng = np.random.default_rng(100 + n)
    for _ in range(20):
        k = int(rng.integers(1, min(n, 5) + 1))
        qs = tuple(int(x) for x in rng.choice(n, k, replace=False))
        u = np.linalg.qr(rng.normal(size=(2 ** k, 2 ** k)) + 1j * rng.normal(size=(2 ** k, 2 ** k)))[0]
        amps = rng.normal(size=2 ** n) + 1j * rng.normal(size=2 ** n)
        amps /= np.linalg.norm(amps)
        s = state_of(amps)
        apply_dense(s, u, qs)
        want = O.lift_matrix(u, qs, n) @ amps
        assert np.max(np.abs(s.amps - want)) <= 1e-12


def test_non_unitary_and_validation():
    s = state_of(vec(1, 1))
    apply_1q(s, np.array([[1, 0], [0, 0]], dtype=complex), 0)
    assert np.allclose(s.amps, [1 / np.sqrt(2), 0], atol=1e-15)
    s = StateVector(2)
    for bad in (lambda: apply_1q(s, np.eye(4), 0), lambda: apply_1q(s, X, 2),
                lambda: apply_2q(s, np.eye(4), 0, 0), lambda: apply_2q(s, np.eye(4), 1, 0),
                lambda: apply_2q(s, np.eye(2), 0, 1), lambda: StateVector(0),
                lambda: StateVector.from_amplitudes(np.ones(3)),
                lambda: StateVector.from_amplitudes(np.array([1.0, 1.0]))):
        with pytest.raises(ValueError):
            bad()


def test_swap_conjugate_route():
    rng = np.random.default_rng(5)
    u = np.linalg.qr(rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4)))[0]
    amps = rng.normal(size=16) + 1j * rng.normal(size=16)
    amps /= np.linalg.norm(amps)
    a = state_of(amps)
    apply_dense(a, u, (3, 1))
    b = state_of(amps)
    apply_2q(b, swap_conjugate(u), 1, 3)
    assert np.array_equal(a.amps, b.amps)


def test_restart_norm_copy():
    s = state_of(vec(0, 1))
    c = s.copy()
    s.restart()
    assert np.allclose(s.amps, [1, 0]) and np.allclose(c.amps, [0, 1])
    assert s.norm() == pytest.approx(1.0, abs=1e-15)


# ---------------------------------------------------------------------------
# measurement and sampling


def test_measure_project_ghz():
    a = np.zeros(8, dtype=complex)
    a[0] = a[7] = 1 / np.sqrt(2)
    s = state_of(a)
    assert measure_project(s, 0, 0) == pytest.approx(0.5, abs=1e-15)
    assert np.allclose(s.amps, np.eye(8)[0], atol=1e-12)
    s = state_of(a)
    measure_project(s, 0, 1)
    assert np.allclose(s.amps, np.eye(8)[7], atol=1e-12)
    with pytest.raises(ProjectionError):
        measure_project(StateVector(1), 0, 1)
    with pytest.raises(ValueError):
        measure_project(StateVector(1), 0, 2)


def test_assert_measure_failure_carries_step_and_prob():
    with pytest.raises(FilterAssertionError) as exc:
        assert_measure(state_of(np.array([0, 1], dtype=complex)), 0, step=3)
    assert exc.value.step == 3 and exc.value.prob <= 1e-12
    s = state_of(vec(1, 1))
    assert assert_measure(s, 0) == pytest.approx(0.5, abs=1e-15)


def test_sampling_matches_reference_exactly(golden):
    d = golden("kernels")
    s = state_of(d["sample_amps"])
    for seed in d["sample_seeds"]:
        assert sample(s, 5000, int(seed)) == golden_samples(d, f"sample_{int(seed)}_")


def test_sampling_contract():
    a = np.zeros(8, dtype=complex)
    a[1] = 1.0
    assert sample(state_of(a), 100, 0) == {"100": 100}
    gen = _as_rng(7)
    assert _as_rng(gen) is gen
    assert sample(StateVector(1), 3, gen) == {"0": 3}
    assert sample(StateVector(1), 0, 0) == {}
    with pytest.raises(ValueError):
        sample(StateVector(1), -1, 0)
    theta = math.asin(math.sqrt(0.3))
    counts = sample(state_of([math.cos(theta), math.sin(theta)]), 100_000, 9)
    assert abs(counts.get("1", 0) - 30_000) <= 5 * math.sqrt(100_000 * 0.21)


def test_expectation_against_reference(golden):
    d = golden("kernels")
    h = PauliHamiltonian(5, dict(zip(map(str, d["exp_letters"]), d["exp_coeffs"])))
    got = expectation_pauli(state_of(d["exp_amps"]), h)
    assert got == pytest.approx(float(d["exp_value"]), abs=1e-12)
    with pytest.raises(ValueError):
        expectation_pauli(StateVector(1), PauliHamiltonian(1, {"Z": 1j}))


# ---------------------------------------------------------------------------
# run(): the fused filter circuits of BASELINE configs 1 and 2


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_mma_run_matches_reference(golden, name):
    d = golden(name)
    fused = to_circuit(d, "fused_")
    n = fused.n_qubits
    hp = PauliHamiltonian(n, dict(zip(map(str, d["energy_letters"]), d["energy_coeffs"])))
    for i, seed in enumerate(d["seeds"]):
        seed = int(seed)
        rep = run(fused, "mma", shots=int(d["shots"]), seed=seed, ancilla=n - 1,
                  hamiltonian=hp if i == 0 else None)
        assert rep.assert_probs == pytest.approx(list(d[f"mma_{seed}_probs"]), abs=1e-12)
        assert rep.samples == golden_samples(d, f"mma_{seed}_")
        if i == 0:
            assert rep.energy == pytest.approx(float(d["energy"]), abs=1e-10)


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_mma_unfused_matches_reference(golden, name):
    d = golden(name)
    circ = to_circuit(d, "in_")
    seed = int(d["seeds"][0])
    rep = run(circ, "mma", shots=int(d["shots"]), seed=seed, ancilla=circ.n_qubits - 1)
    assert rep.assert_probs == pytest.approx(list(d["unfused_probs"]), abs=1e-12)
    assert rep.samples == golden_samples(d, "unfused_")


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_final_state_matches_reference(golden, name):
    from paper_2310_17739_b200._pack import pack
    from paper_2310_17739_b200.engine import DeviceProgram
    d = golden(name)
    fused = to_circuit(d, "fused_")
    end = len(fused.instructions) - fused.n_qubits
    s = StateVector(fused.n_qubits)
    pk = pack(fused, fused.instructions[:end])
    prog = DeviceProgram(s, pk.ops, pk.params, pk.payloads)
    prog.run_mma()
    assert rel_l2(s.amps, d["final_state"]) < 1e-10


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_rejection_run_matches_reference(golden, name):
    d = golden(name)
    fused = to_circuit(d, "fused_")
    rep = run(fused, "rejection", shots=int(d["rej_shots"]), seed=int(d["seeds"][0]),
              ancilla=None)
    assert rep.accepted == int(d["rej_accepted"])
    assert rep.step_rejections == list(d["rej_steps"])
    assert rep.samples == golden_samples(d, "rej_")
    assert rep.overall_success == rep.accepted / int(d["rej_shots"])


def two_step_circuit(theta1=0.6, theta2=0.3, spin=0.8):
    c = Circuit(3, [("c", 2), ("r", 3)])
    c.ry(spin, 0)
    c.ry(2 * theta1, 2)
    c.measure(2, 0)
    c.barrier()
    c.reset(2)
    c.barrier()
    c.cx(0, 1)
    c.ry(2 * theta2, 2)
    c.measure(2, 1)
    c.barrier()
    c.reset(2)
    c.barrier()
    for q in range(3):
        c.measure(q, c.clbit_index("r", q))
    return c


def test_mma_closed_form_and_report_layout():
    rep = run(two_step_circuit(), "mma", shots=2000, seed=11, ancilla=2,
              fusion_stats={"gates_before": 5})
    assert rep.assert_probs == pytest.approx([math.cos(0.6) ** 2, math.cos(0.3) ** 2], abs=1e-12)
    assert all(k[2] == "0" for k in rep.samples) and sum(rep.samples.values()) == 2000
    d = rep.to_dict()
    assert list(d) == ["mode", "n_qubits", "shots", "seed", "ancilla", "assert_probs",
                       "overall_success", "accepted", "rejected", "step_rejections", "samples",
                       "energy", "fusion_stats", "wall_time_s"]


def test_mma_assertion_failure_raises_with_step():
    c = Circuit(2, [("c", 1), ("r", 2)])
    c.x(1)
    c.measure(1, 0)
    c.reset(1)
    c.measure(0, c.clbit_index("c", 0))
    with pytest.raises(FilterAssertionError) as exc:
        run(c, "mma", shots=1, seed=0, ancilla=1)
    assert exc.value.step == 0


def test_blocked_kernel_assertion_failure_raises_with_step():
    """n >= 6 takes the single-launch blocked kernel; the in-kernel check must
    report the first failing step exactly like the reference."""
    n = 8
    c = Circuit(n, [("c", 3), ("r", n)])
    for step in range(3):
        for q in range(n - 1):
            c.h(q)
            c.cx(q, (q + 1) % (n - 1))
        if step == 1:
            c.x(n - 1)
        c.measure(n - 1, step)
        c.reset(n - 1)
    with pytest.raises(FilterAssertionError) as exc:
        run(c, "mma", shots=1, seed=0, ancilla=n - 1)
    assert exc.value.step == 1 and exc.value.prob < 1e-12


def test_rejection_early_abort_counts_first_step():
    c = Circuit(2, [("c", 2), ("r", 2)])
    c.x(1)
    c.measure(1, 0)
    c.reset(1)
    c.h(0)
    c.measure(1, 1)
    c.reset(1)
    c.measure(0, c.clbit_index("r", 0))
    rep = run(c, "rejection", shots=50, seed=2, ancilla=None)
    assert rep.accepted == 0 and rep.step_rejections == [50, 0] and rep.samples == {}


# ---------------------------------------------------------------------------
# blocked kernel vs oracle across tile configurations


def random_filter_like(rng, n, blocks, per_block, dense_frac=0.5):
    anc = n - 1
    c = Circuit(n, [("c", blocks), ("r", n)])
    for b in range(blocks):
        for _ in range(per_block):
            r = rng.random()
            a, bq = (int(x) for x in rng.choice(n, 2, replace=False))
            if r < 0.3:
                c.gate_op(Gate.U3, (a,), tuple(rng.uniform(-3, 3, 3)))
            elif r < 0.3 + 0.4 * dense_frac:
                c.gate_op(Gate.CU3, (a, bq), tuple(rng.uniform(-3, 3, 3)))
            else:
                g = (Gate.CX, Gate.CZ, Gate.SWAP, Gate.RZZ, Gate.CRZ)[int(rng.integers(5))]
                c.gate_op(g, (a, bq), tuple(rng.uniform(-3, 3, g.n_params)))
        c.gate_op(Gate.RY, (anc,), (float(rng.uniform(0.2, 1.2)),))
        c.measure(anc, b)
        c.barrier()
        c.reset(anc)
        c.barrier()
    for q in range(n):
        c.measure(q, blocks + q)
    return c


@pytest.mark.parametrize("n", [6, 9, 12, 13, 15, 17])
def test_blocked_kernel_against_oracle(n):
    rng = np.random.default_rng(1000 + n)
    c = random_filter_like(rng, n, blocks=3, per_block=60)
    fused, _ = fuse_pipeline(c)
    instrs = oracle_from_circuit(fused)
    try:
        probs, samples, state, _ = O.run_mma(instrs, n, 128, 5)
    except O.OracleAssertion:
        pytest.skip("random circuit hit a dead assertion branch")
    rep = run(fused, "mma", shots=128, seed=5, ancilla=n - 1)
    assert rep.assert_probs == pytest.approx(probs, abs=1e-12)
    assert rep.samples == samples


def ladder_circuit(rng, n, terms, blocks=2):
    """JW-ladder rotations (the filter-circuit body, projection.py:191-212)
    with random Pauli words: long CX chains that the relabeling frame absorbs."""
    anc = n - 1
    c = Circuit(n, [("c", blocks), ("r", n)])
    for b in range(blocks):
        for _ in range(terms):
            inv = sorted(int(x) for x in rng.choice(n - 1, int(rng.integers(1, n - 1)),
                                                    replace=False))
            letters = {q: "XYZ"[int(rng.integers(3))] for q in inv}
            for q in inv:
                if letters[q] == "X":
                    c.h(q)
                elif letters[q] == "Y":
                    c.sdg(q)
                    c.h(q)
            c.sdg(anc)
            c.h(anc)
            chain = inv + [anc]
            for x, y in zip(chain, chain[1:]):
                c.cx(x, y)
            c.rz(float(rng.uniform(-1, 1)), anc)
            for x, y in reversed(list(zip(chain, chain[1:]))):
                c.cx(x, y)
            c.h(anc)
            c.gate_op(Gate.S, (anc,))
            for q in reversed(inv):
                if letters[q] == "X":
                    c.h(q)
                elif letters[q] == "Y":
                    c.h(q)
                    c.gate_op(Gate.S, (q,))
            if rng.random() < 0.2:  # stray swaps and reversed CX exercise the frame
                x, y = (int(v) for v in rng.choice(n - 1, 2, replace=False))
                c.gate_op(Gate.SWAP, (x, y))
                c.cx(y, x)
        c.measure(anc, b)
        c.barrier()
        c.reset(anc)
        c.barrier()
    for q in range(n):
        c.measure(q, blocks + q)
    return c


@pytest.mark.parametrize("n,terms", [(7, 30), (12, 40), (14, 60), (18, 40)])
def test_relabeling_frame_against_oracle(n, terms):
    rng = np.random.default_rng(50 + n)
    c = ladder_circuit(rng, n, terms)
    for circ in (c, fuse_pipeline(c)[0]):
        instrs = oracle_from_circuit(circ)
        try:
            probs, samples, state, _ = O.run_mma(instrs, n, 256, 9)
        except O.OracleAssertion:
            pytest.skip("dead assertion branch")
        rep = run(circ, "mma", shots=256, seed=9, ancilla=n - 1)
        assert rep.assert_probs == pytest.approx(probs, abs=1e-12)
        assert rep.samples == samples
        rej = run(circ, "rejection", shots=3, seed=4, ancilla=None)
        acc, steps, counts = O.run_rejection(instrs, n, 3, 4)
        assert (rej.accepted, rej.step_rejections, rej.samples) == (acc, steps, counts)


@pytest.mark.gpu
def test_rejection_replay_equals_explicit_shots(golden):
    """The replay fast path of nsb_plan_run_rejection gives the same tallies,
    samples, accepted count and consumed draws as simulating every shot
    (same seed, same Philox stream), and both equal the reference's goldens."""
    from paper_2310_17739_b200 import engine as E
    d = golden("filter8")
    fused = to_circuit(d, "fused_")
    instrs = fused.instructions
    end = E._sampling_start(instrs)
    packed = E.pack(fused, instrs[:end])
    n_steps = sum(1 for ins in instrs[:end] if ins.gate is E.Gate.MEASURE)
    state = E.StateVector(fused.n_qubits)
    prog = E.DeviceProgram(state, packed.ops, packed.params, packed.payloads, exact=True)
    r1, r2 = E._as_rng(int(d["seeds"][0])), E._as_rng(int(d["seeds"][0]))
    shots = int(d["rej_shots"])
    fast = E._rejection(state, prog, n_steps, shots, r1, False)
    slow = E._rejection(state, prog, n_steps, shots, r2, False, explicit=True)
    assert fast[:3] == slow[:3]
    assert r1.random() == r2.random()  # both generators advanced by the same draws
    assert fast[0] == int(d["rej_accepted"])
    assert fast[2] == list(d["rej_steps"])
    assert fast[1] == golden_samples(d, "rej_")


@pytest.mark.parametrize("env", [{}, {"NSB_NO_GROUP_FUSION": "1"}, {"NSB_EXACT_CLASSES": "1"}])
def test_deep_filter_workload_classes_and_group_fusion(monkeypatch, env):
    """The deep-circuit shape (JW shell-model filter, natively generated and
    fused) through the blocked kernel with the planner's near-zero cleaning,
    real two-block classes and group fusion on (default) and off: final
    state within 1e-10 relative L2 and assertion probabilities within 1e-12
    of the full-state oracle."""
    import shard_exec as SE
    from paper_2310_17739_b200 import workloads as W
    from paper_2310_17739_b200.engine import DeviceProgram, StateVector
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    wl = W.filter_workload(11, trotter=2, n_steps=3, n_scatter=6, trial="10" * 6)
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    n = wl.n_qubits
    want_p, want = SE.full_mma(exe, wl.params, pool, n)
    state = StateVector(n)
    prog = DeviceProgram(state, exe, wl.params, pool)
    got_p = prog.run_mma()
    assert got_p == pytest.approx(want_p, abs=1e-12)
    assert rel_l2(state.amps, want) < 1e-10
    if not env:
        assert prog.info.n_fused_group_ops > 0
