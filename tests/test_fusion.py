"""Native fusion (csrc/fusion.cpp via fuse_pipeline) is bit-exact against the
reference's fused lists (golden) and agrees with the pinned oracle."""

import numpy as np
import pytest

import nucsim_oracle as O
from circuit_io import oracle_from_circuit, to_circuit, to_oracle
from paper_2310_17739_b200 import (Circuit, Gate, absorb_1q, fuse_2q, fuse_pipeline, gate_count,
                                   gate_matrix, merge_1q, normalize_2q_order)
from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200.fusion import blas_variant


@pytest.fixture(autouse=True)
def pin_variant(monkeypatch, golden_variant):
    monkeypatch.setenv("NUCSIM_BLAS_VARIANT", golden_variant)
    blas_variant.cache_clear()
    yield
    blas_variant.cache_clear()


def assert_same(circuit, want):
    got = oracle_from_circuit(circuit)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert (a[0], tuple(a[1]), tuple(a[2]), a[4]) == (b[0], tuple(b[1]), tuple(b[2]), b[4])
        if b[3] is not None:
            assert a[3] is not None and np.array_equal(a[3], b[3]), a


def test_fuse_pipeline_bit_exact_against_reference(golden):
    d = golden("fusion")
    for i in range(int(d["n_cases"])):
        c = to_circuit(d, f"c{i}_in_")
        fused, stats = fuse_pipeline(c)
        want, _ = to_oracle(d, f"c{i}_out_")
        assert_same(fused, want)
        flat = [v for p in stats.per_pass for v in (p.gates_before, p.gates_after)]
        assert [stats.gates_before, stats.gates_after] + flat == list(d[f"c{i}_stats"])


def test_individual_passes_bit_exact(golden):
    d = golden("fusion")
    for i in range(0, int(d["n_cases"]), 5):
        c = to_circuit(d, f"c{i}_in_")
        for tag, fn in (("merge", merge_1q), ("absorb", absorb_1q),
                        ("norm", normalize_2q_order), ("fuse2", fuse_2q)):
            want, _ = to_oracle(d, f"c{i}_{tag}_")
            assert_same(fn(c), want)


@pytest.mark.parametrize("name", ["filter8", "filter16"])
def test_filter_circuit_fusion_bit_exact(golden, name):
    d = golden(name)
    fused, stats = fuse_pipeline(to_circuit(d, "in_"))
    want, _ = to_oracle(d, "fused_")
    assert_same(fused, want)
    assert stats.gates_after == int(d["fused_stats"][1])


def test_native_fusion_matches_oracle_on_random_circuits(golden_variant):
    rng = np.random.default_rng(77)
    pool1 = [Gate.H, Gate.X, Gate.S, Gate.T, Gate.RX, Gate.RZ, Gate.U3, Gate.U2]
    pool2 = [Gate.CX, Gate.CZ, Gate.SWAP, Gate.CRZ, Gate.RZZ, Gate.RXX, Gate.CU3]
    for trial in range(40):
        n = int(rng.integers(2, 7))
        c = Circuit(n, [("c", 2)])
        for _ in range(int(rng.integers(10, 120))):
            r = rng.random()
            if r < 0.5:
                g = pool1[rng.integers(len(pool1))]
                c.gate_op(g, (int(rng.integers(n)),), rng.uniform(-3, 3, g.n_params))
            elif r < 0.95:
                g = pool2[rng.integers(len(pool2))]
                a, b = rng.choice(n, 2, replace=False)
                c.gate_op(g, (int(a), int(b)), rng.uniform(-3, 3, g.n_params))
            elif r < 0.975:
                c.barrier()
            else:
                q = int(rng.integers(n))
                c.measure(q, 0)
                c.reset(q)
        fused, _ = fuse_pipeline(c)
        want, _ = O.fuse_pipeline(oracle_from_circuit(c), golden_variant)
        assert_same(fused, want)


def test_pipeline_idempotent_and_payload_only():
    rng = np.random.default_rng(3)
    c = Circuit(4, [("c", 1)])
    for _ in range(60):
        a, b = rng.choice(4, 2, replace=False)
        c.cx(int(a), int(b))
        c.rz(float(rng.normal()), int(a))
    once, s1 = fuse_pipeline(c)
    twice, s2 = fuse_pipeline(once)
    assert s2.gates_before == s2.gates_after == s1.gates_after
    assert [i.key() for i in once.instructions] == [i.key() for i in twice.instructions]
    assert {i.gate for i in once.instructions} <= {Gate.C1, Gate.C2}


def test_wide_gates_opaque_and_markers():
    c = Circuit(3, [("c", 1)])
    c.h(0)
    c.gate_op(Gate.CCX, (0, 1, 2))
    c.h(0)
    c.barrier()
    c.measure(0, 0)
    out, stats = fuse_pipeline(c)
    assert [i.gate for i in out.instructions] == [Gate.C1, Gate.CCX, Gate.C1, Gate.BARRIER,
                                                  Gate.MEASURE]
    assert out.instructions[1] is c.instructions[1]  # untouched instructions are reused
    assert stats.gates_before == stats.gates_after == 3
    assert stats.reduction_factor == 1.0


def test_cx_triple_is_swap():
    c = Circuit(2)
    c.cx(0, 1)
    c.cx(1, 0)
    c.cx(0, 1)
    out, stats = fuse_pipeline(c)
    (ins,) = out.instructions
    assert ins.qubits == (0, 1) and stats.gates_after == 1
    assert np.max(np.abs(ins.matrix - gate_matrix(Gate.SWAP))) <= 1e-12


def test_blas_variant_probe_matches_numpy(monkeypatch):
    monkeypatch.delenv("NUCSIM_BLAS_VARIANT", raising=False)
    blas_variant.cache_clear()
    v = blas_variant()
    assert v in (N.BLAS_CHAIN2, N.BLAS_FOUR)
    rng = np.random.default_rng(9)
    a = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    b = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
    c = Circuit(1)
    c.fused_1q(np.linalg.qr(b)[0], 0)
    c.fused_1q(np.linalg.qr(a)[0], 0)
    (ins,) = merge_1q(c).instructions
    assert np.array_equal(ins.matrix, np.linalg.qr(a)[0] @ np.linalg.qr(b)[0])


def test_gate_count_excludes_markers():
    c = Circuit(2, [("c", 1)])
    c.h(0)
    c.barrier()
    c.measure(1, 0)
    assert gate_count(c) == 1


def test_segment_parallel_fusion_equals_serial_and_oracle(monkeypatch, golden_variant):
    """Circuits above 2 x 2^15 records fuse on host threads, split after barriers
    that cover every qubit (csrc/fusion.cpp segment_cuts); the result must be
    the serial pipeline's, which is the reference's (fusion.py:240-251)."""
    rng = np.random.default_rng(2310)
    n = 6
    c = Circuit(n, [("c", 2)])
    pool1 = [Gate.H, Gate.RX, Gate.RZ, Gate.U3]
    pool2 = [Gate.CX, Gate.CZ, Gate.RZZ, Gate.CU3]
    payload = None
    for i in range(150_000):
        if i % 37_000 == 36_999:
            c.barrier()  # full barrier: a segment boundary
            continue
        r = rng.random()
        if r < 0.45:
            g = pool1[rng.integers(len(pool1))]
            c.gate_op(g, (int(rng.integers(n)),), tuple(rng.uniform(-3, 3, g.n_params)))
        elif r < 0.93:
            g = pool2[rng.integers(len(pool2))]
            a, b = rng.choice(n, 2, replace=False)
            c.gate_op(g, (int(a), int(b)), tuple(rng.uniform(-3, 3, g.n_params)))
        elif r < 0.95:
            if payload is None:
                payload = gate_matrix(Gate.CU3, (0.3, -1.1, 0.7))
            a, b = rng.choice(n, 2, replace=False)
            c.fused_2q(payload, int(a), int(b))  # input payload records
        elif r < 0.96:
            c.gate_op(Gate.CCX, tuple(int(q) for q in rng.choice(n, 3, replace=False)))
        elif r < 0.98:
            c.barrier(*(int(q) for q in rng.choice(n, 2, replace=False)))  # partial: no cut
        else:
            q = int(rng.integers(n))
            c.measure(q, 0)
            c.reset(q)
    par, s_par = fuse_pipeline(c)
    monkeypatch.setenv("NSB_FUSE_SERIAL", "1")
    ser, s_ser = fuse_pipeline(c)
    assert s_par == s_ser
    want = oracle_from_circuit(ser)
    assert_same(par, want)
    ref, _ = O.fuse_pipeline(oracle_from_circuit(c), golden_variant)
    assert_same(par, ref)
