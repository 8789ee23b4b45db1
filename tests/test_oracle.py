"""Pin the oracle (oracle/nucsim_oracle.py) to the reference's own outputs.

Every check compares the CPU restatement with golden vectors produced by
running the reference in the build container; the product's tests then use
the oracle (and the same fixtures) as the checker.
"""

import numpy as np
import pytest

import nucsim_oracle as O
from circuit_io import to_oracle


def same_instrs(got, want):
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert a[0] == b[0] and tuple(a[1]) == tuple(b[1]) and tuple(a[2]) == tuple(b[2])
        assert a[4] == b[4]
        if b[3] is not None or a[0] in ("c1", "c2"):
            assert np.array_equal(O.resolved(a), b[3])


def test_oracle_fusion_bit_exact_against_reference(golden, golden_variant):
    d = golden("fusion")
    for i in range(int(d["n_cases"])):
        instrs, _ = to_oracle(d, f"c{i}_in_")
        want, _ = to_oracle(d, f"c{i}_out_")
        got, stats = O.fuse_pipeline(instrs, golden_variant)
        same_instrs(got, want)
        flat = [v for _, b, a in stats for v in (b, a)]
        assert [O.gate_count(instrs), O.gate_count(got)] + flat == list(d[f"c{i}_stats"])


def test_oracle_individual_passes(golden, golden_variant):
    d = golden("fusion")
    mm = O.Matmul(golden_variant)
    for i in range(0, int(d["n_cases"]), 5):
        instrs, _ = to_oracle(d, f"c{i}_in_")
        for tag, fn in (("merge", O.merge_1q), ("absorb", O.absorb_1q),
                        ("norm", O.normalize_2q_order), ("fuse2", O.fuse_2q)):
            want, _ = to_oracle(d, f"c{i}_{tag}_")
            same_instrs(fn(instrs, mm), want)


def test_oracle_kernels_against_reference(golden):
    d = golden("kernels")
    for i in range(int(d["n_kernels"])):
        amps, u = d[f"k{i}_amps"], d[f"k{i}_u"]
        qubits = tuple(int(x) for x in d[f"k{i}_qubits"])
        got = O.apply_dense(amps.copy(), u, qubits)
        assert np.array_equal(got, d[f"k{i}_out"])
        if d[f"k{i}_mp"] >= 0:
            a = amps.copy()
            q = int(d[f"k{i}_mq"])
            p = O.branch_probability(a, q, 0)
            assert p == d[f"k{i}_mp"]
            O.project(a, q, 0, p)
            assert np.array_equal(a, d[f"k{i}_mout"])


def test_oracle_sampling_against_reference(golden):
    d = golden("kernels")
    for seed in d["sample_seeds"]:
        seed = int(seed)
        got = O.sample(d["sample_amps"], 10, 5000, seed)
        n = int(d[f"sample_{seed}_n"])
        want = dict(zip(d[f"sample_{seed}_keys"][:n], d[f"sample_{seed}_counts"][:n]))
        assert got == {str(k): int(v) for k, v in want.items()}


def test_oracle_expectation_against_reference(golden):
    d = golden("kernels")
    terms = sorted(zip([str(x) for x in d["exp_letters"]], d["exp_coeffs"]))
    got = O.expectation_pauli(d["exp_amps"].copy(), [(l, complex(c)) for l, c in terms])
    assert got == pytest.approx(float(d["exp_value"]), abs=1e-14)


@pytest.mark.parametrize("name", ["filter8"])
def test_oracle_filter_run_against_reference(golden, golden_variant, name):
    d = golden(name)
    instrs, n = to_oracle(d, "in_")
    fused, _ = O.fuse_pipeline(instrs, golden_variant)
    want, _ = to_oracle(d, "fused_")
    same_instrs(fused, want)
    terms = list(zip([str(x) for x in d["energy_letters"]], d["energy_coeffs"]))
    for seed in d["seeds"]:
        seed = int(seed)
        probs, samples, state, energy = O.run_mma(want, n, int(d["shots"]), seed,
                                                  terms if seed == int(d["seeds"][0]) else None)
        assert probs == pytest.approx(list(d[f"mma_{seed}_probs"]), abs=1e-13)
        k = int(d[f"mma_{seed}_n"])
        assert samples == dict(zip(map(str, d[f"mma_{seed}_keys"][:k]),
                                   map(int, d[f"mma_{seed}_counts"][:k])))
        if seed == int(d["seeds"][0]):
            assert np.max(np.abs(state - d["final_state"])) < 1e-12
            assert energy == pytest.approx(float(d["energy"]), abs=1e-12)
    acc, rej, counts = O.run_rejection(want, n, int(d["rej_shots"]), int(d["seeds"][0]))
    assert acc == int(d["rej_accepted"]) and rej == list(d["rej_steps"])
    k = int(d["rej_n"])
    assert counts == dict(zip(map(str, d["rej_keys"][:k]), map(int, d["rej_counts"][:k])))
