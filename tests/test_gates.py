"""Gate vocabulary: Python and native matrices are bit-identical to the
reference's gate_matrix (golden vectors from tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

import nucsim_oracle as O
from paper_2310_17739_b200 import Gate, gate_matrix
from paper_2310_17739_b200 import _native as N


def golden_rows(g):
    d = g("gates")
    for i, name in enumerate(d["names"]):
        k = int(d["npar"][i])
        params = tuple(float(x) for x in d["params"][i, :k])
        gate = Gate(str(name))
        dim = 1 << gate.n_qubits
        off = int(d["mat_off"][i])
        yield gate, params, d["mats"][off:off + dim * dim].reshape(dim, dim)


def test_python_gate_matrix_is_bit_identical(golden):
    n = 0
    for gate, params, want in golden_rows(golden):
        got = gate_matrix(gate, params)
        assert np.array_equal(got, want), (gate, params)
        n += 1
    assert n > 500


def test_native_gate_matrix_is_bit_identical(golden):
    for gate, params, want in golden_rows(golden):
        dim = want.shape[0]
        out = np.zeros(dim * dim, np.complex128)
        p = np.asarray(params if params else [0.0], np.float64)
        assert N.lib().nsb_gate_matrix(gate.code, N.ptr(p), len(params), N.ptr(out)) == 0
        assert np.array_equal(out.reshape(dim, dim), want), (gate, params)


def test_oracle_gate_matrix_is_bit_identical(golden):
    for gate, params, want in golden_rows(golden):
        assert np.array_equal(O.gate_matrix(gate.value, params), want), gate


def test_gate_matrix_validation():
    with pytest.raises(ValueError):
        gate_matrix(Gate.MEASURE)
    with pytest.raises(ValueError):
        gate_matrix(Gate.C2)
    with pytest.raises(ValueError):
        gate_matrix(Gate.RX, ())
    m = gate_matrix(Gate.H)
    m[0, 0] = 7  # callers get a private copy
    assert gate_matrix(Gate.H)[0, 0] == math.sqrt(0.5)


def test_tag_codes_follow_reference_enum_order():
    assert [g.code for g in Gate] == list(range(len(Gate)))
    assert Gate.U3.code == 0 and Gate.BARRIER.code == len(Gate) - 1
    assert Gate.C4X.n_qubits == 5 and Gate.CU3.n_params == 3
