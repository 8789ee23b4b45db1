"""Native filter-circuit emitter (csrc/generator.cpp) reproduces the
reference's build_filter_circuit (projection.py:191-255) instruction by
instruction: same tags, qubits, float parameters, classical bits, barriers,
for the BASELINE config-1 and config-2 circuits the reference generated."""

import numpy as np
import pytest

from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200 import workloads as W
from paper_2310_17739_b200.gates import BY_CODE

LETTERS = "IXYZ"


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_native_generator_matches_reference_circuit(golden, name):
    d = golden(name)
    n_sys = d["term_letters"].shape[1]
    terms = [("".join(LETTERS[c] for c in row), float(cf))
             for row, cf in zip(d["term_letters"], d["term_coeffs"])]
    steps = [tuple(map(float, s)) for s in d["steps"]]
    trial = "".join(str(int(b)) for b in d["trial"])
    wl = W.filter_workload(n_sys, int(d["trotter"]), terms=terms, steps=steps, trial=trial)
    ops = wl.ops
    names = d["in_names"]
    assert len(ops) == len(names)
    kinds = {"measure": N.OP_MEASURE, "reset": N.OP_RESET, "barrier": N.OP_BARRIER}
    for i, rec in enumerate(ops):
        name_i = str(names[i])
        assert int(rec["kind"]) == kinds.get(name_i, N.OP_GATE), i
        if name_i == "barrier":
            assert int(rec["mask"]) == int(d["in_bmask"][i])
            continue
        nq = int(d["in_nq"][i])
        assert tuple(rec["q"][:nq]) == tuple(d["in_qubits"][i, :nq]), i
        assert int(rec["cbit"]) == int(d["in_cbit"][i])
        if name_i not in kinds:
            assert BY_CODE[int(rec["tag"])].value == name_i, i
            npar = int(d["in_npar"][i])
            got = wl.params[int(rec["param"]):int(rec["param"]) + npar] if npar else []
            assert np.array_equal(np.asarray(got), d["in_params"][i, :npar]), i
    assert wl.input_gates == int(d["fused_stats"][0])


def test_generator_rejects_bad_input():
    with pytest.raises(ValueError):
        W.filter_workload(3, 0, terms=[("XZI", 0.5)], steps=[(1.0, 0.0)])
