"""engine._compile, infer_ancilla, _run_gates_only and every MmaStructureError
branch (reference engine.py:295-393), which the reference's acceptance
criterion 9 drives by hand (test_acceptance.py:362-404).

CPU: plan tuples against the oracle's restatement of the plan (engine.py:334-358:
opcodes, qubits, steps, classical bits, matrices with the swap-conjugation of
reversed 2q operands), the validation messages verbatim, ancilla inference.
GPU: _compile + _run_gates_only + assert_measure by hand reproduce run()'s
assertion probabilities and the oracle's final state.
"""

import numpy as np
import pytest

import nucsim_oracle as O
from circuit_io import oracle_from_circuit
from paper_2310_17739_b200 import Circuit, Gate, fuse_pipeline
from paper_2310_17739_b200 import engine as E
from paper_2310_17739_b200.errors import MmaStructureError
from test_engine_gpu import random_filter_like


def test_compile_plan_matches_reference_layout():
    rng = np.random.default_rng(9)
    for n in (3, 5, 8):
        c = random_filter_like(rng, n, blocks=3, per_block=25)
        for circ in (c, fuse_pipeline(c)[0]):
            plan, n_steps, finals = E._compile(circ, "mma", n - 1)
            want, want_steps = O._plan(oracle_from_circuit(circ))
            assert n_steps == want_steps == 3
            assert len(plan) == len(want)
            instrs = [ins for ins in circ.instructions[:E._sampling_start(circ.instructions)]
                      if ins.gate is not Gate.BARRIER]
            for entry, w, ins in zip(plan, want, instrs):
                if w[0] == "measure":
                    assert entry == (E._OP_MEASURE, w[1], ins.cbit, w[2])
                elif w[0] == "reset":
                    assert entry == (E._OP_RESET, w[1])
                elif len(w[2]) == 1:
                    assert entry[0] == E._OP_1Q and entry[2] == w[2][0]
                    assert np.array_equal(entry[1], w[1])
                elif len(w[2]) == 2:
                    a, b = w[2]
                    assert entry[0] == E._OP_2Q and entry[1].shape == (2, 2, 2, 2)
                    assert (entry[2], entry[3]) == (min(a, b), max(a, b))
                    m = w[1] if a < b else E.swap_conjugate(w[1])
                    assert np.array_equal(entry[1].reshape(4, 4), m)
                else:
                    assert entry[0] == E._OP_KQ and tuple(entry[2]) == w[2]
                    assert np.array_equal(entry[1], w[1])
            assert finals == [(q, q + 3) for q in range(n)]


def test_compile_rejection_mode_skips_validation():
    c = Circuit(2, [("c", 1)])
    c.h(0)
    c.measure(0, 0)  # not followed by a reset: fine outside MMA mode
    c.h(1)
    plan, steps, finals = E._compile(c, "rejection", None)
    assert steps == 1 and [p[0] for p in plan] == [E._OP_1Q, E._OP_MEASURE, E._OP_1Q]
    assert finals == []


def _filter(n=3, anc=2):
    c = Circuit(n, [("c", 1), ("r", n)])
    c.h(0)
    c.measure(anc, 0)
    c.barrier()
    c.reset(anc)
    for q in range(n):
        c.measure(q, 1 + q)
    return c


@pytest.mark.parametrize("ancilla", [None, -1, 3, 7])
def test_mma_structure_ancilla_out_of_range(ancilla):
    with pytest.raises(MmaStructureError, match=f"^ancilla index {ancilla} out of range$"):
        E._compile(_filter(), "mma", ancilla)


def test_mma_structure_measure_not_on_ancilla():
    c = _filter()
    with pytest.raises(MmaStructureError,
                       match="^mid-circuit measure on qubit 2 is not the ancilla$"):
        E._compile(c, "mma", 1)


def test_mma_structure_measure_without_reset():
    c = Circuit(3, [("c", 2)])
    c.h(0)
    c.measure(2, 0)
    c.barrier()
    c.h(1)
    c.measure(0, 1)
    with pytest.raises(MmaStructureError,
                       match="^measure at instruction 1 lacks a following ancilla reset$"):
        E._compile(c, "mma", 2)
    c2 = Circuit(3, [("c", 1)])
    c2.measure(2, 0)
    c2.reset(1)  # a reset, but not of the ancilla
    c2.h(0)
    with pytest.raises(MmaStructureError, match="^measure at instruction 0 lacks"):
        E._compile(c2, "mma", 2)


def test_mma_structure_unpaired_reset():
    c = Circuit(3, [("c", 1)])
    c.h(0)
    c.reset(2)
    c.h(1)
    with pytest.raises(MmaStructureError,
                       match="^reset at instruction 1 is not paired with an assertion$"):
        E._compile(c, "mma", 2)


def test_run_raises_the_same_structure_errors():
    c = Circuit(3, [("c", 1)])
    c.h(0)
    c.reset(2)
    c.h(1)
    with pytest.raises(MmaStructureError, match="is not paired with an assertion"):
        E.run(c, "mma", shots=4, seed=1, ancilla=2)


def test_infer_ancilla():
    assert E.infer_ancilla(_filter()) == 2
    c = Circuit(3, [("c", 2), ("r", 3)])
    c.h(0)
    for q in range(3):
        c.measure(q, 2 + q)
    assert E.infer_ancilla(c) is None  # only the sampling block measures
    c = Circuit(3, [("c", 2)])
    c.measure(1, 0)
    c.reset(1)
    c.measure(2, 1)
    c.reset(2)
    c.h(0)
    assert E.infer_ancilla(c) is None  # two different targets
    c = Circuit(3, [("c", 2)])
    c.measure(1, 0)
    c.reset(1)
    c.barrier()
    c.measure(1, 1)
    c.reset(1)
    c.h(0)
    assert E.infer_ancilla(c) == 1


@pytest.mark.gpu
@pytest.mark.parametrize("n", [4, 9])
def test_run_gates_only_by_hand_matches_run_and_oracle(n):
    """Criterion 9's loop (test_acceptance.py:373-390): _compile, then per plan
    entry _run_gates_only / assert_measure on a StateVector."""
    rng = np.random.default_rng(40 + n)
    c = random_filter_like(rng, n, blocks=2, per_block=40)
    fused, _ = fuse_pipeline(c)
    try:
        want_p, _, want_state, _ = O.run_mma(oracle_from_circuit(fused), n, 8, 1)
    except O.OracleAssertion:
        pytest.skip("dead assertion branch")
    plan, n_steps, _ = E._compile(fused, "mma", n - 1)
    state = E.StateVector(n)
    probs = []
    for entry in plan:
        if entry[0] == E._OP_MEASURE:
            probs.append(E.assert_measure(state, entry[1], entry[3]))
        elif entry[0] != E._OP_RESET:
            E._run_gates_only(state, entry)
    assert len(probs) == n_steps
    assert probs == pytest.approx(want_p, abs=1e-12)
    rep = E.run(fused, "mma", shots=8, seed=1, ancilla=n - 1)
    assert rep.assert_probs == pytest.approx(probs, abs=1e-12)
    got = state.amps
    assert np.linalg.norm(got - want_state) <= 1e-10 * np.linalg.norm(want_state)
