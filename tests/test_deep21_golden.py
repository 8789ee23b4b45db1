"""Parity at the benchmarked size (BASELINE config 3, deep21: 21 qubits,
1 948 482 input gates) against fixtures the UNMODIFIED reference produced
(tests/golden/make_deep21_golden.py, tests/golden/deep21.npz).

CPU: the native emitter reproduces the reference's build_filter_circuit
(projection.py:215-255) of the whole headline circuit, and native fusion
reproduces the reference's fuse_pipeline (fusion.py:240-251) of it bit for bit
-- compared through a canonical sha256 of all 983 376 fused instructions and
their payload bits, plus the first 1 500 fused instructions in full.

GPU: the blocked kernel runs the Trotter-1, two-step version of the same
circuit at full width (21 qubits) and must reproduce the reference run's
assertion probabilities, samples for two seeds, and final-state digest.
"""

import numpy as np
import pytest

from circuit_io import canonical_from_arrays, canonical_from_packed, digest, to_oracle
from paper_2310_17739_b200 import workloads as W
from paper_2310_17739_b200.fusion import blas_variant


@pytest.fixture(autouse=True)
def pin_variant(monkeypatch, golden_variant):
    monkeypatch.setenv("NUCSIM_BLAS_VARIANT", golden_variant)
    blas_variant.cache_clear()
    yield
    blas_variant.cache_clear()


def deep21(d, trotter=None, n_steps=None):
    terms = [("".join("IXYZ"[c] for c in row), float(cf))
             for row, cf in zip(d["term_letters"], d["term_coeffs"])]
    steps = [tuple(map(float, s)) for s in d["steps"]][:n_steps]
    trial = "".join(str(int(b)) for b in d["trial"])
    return W.filter_workload(20, int(d["trotter"]) if trotter is None else trotter,
                             terms=terms, steps=steps, trial=trial)


def test_deep21_terms_are_the_bench_workload(golden):
    """The fixture's Hamiltonian is the one bench.py generates."""
    d = golden("deep21")
    terms = W.shell_model_terms(20, 21, 20, 0.35, 8)
    assert [l for l, _ in terms] == ["".join("IXYZ"[c] for c in r) for r in d["term_letters"]]
    assert np.array_equal([c for _, c in terms], d["term_coeffs"])
    assert np.array_equal(W.halving_schedule(0.5, 8), d["steps"])


def test_deep21_full_circuit_and_fusion_bit_exact(golden):
    d = golden("deep21")
    wl = deep21(d)
    assert wl.input_gates == int(d["fused_stats"][0]) == 1948482
    assert len(wl.ops) == int(d["input_len"])
    assert digest(canonical_from_packed(wl.ops, wl.params, wl.payloads)) == str(d["input_digest"])
    fops, pool, stats = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    assert stats["gates_after"] == int(d["fused_stats"][1])
    flat = [v for p in stats["per_pass"] for v in p]
    assert flat == list(d["fused_stats"][2:])
    assert len(fops) == int(d["fused_len"])
    got = canonical_from_packed(fops, wl.params, pool)
    # the first PREFIX instructions in full (a readable diff on failure) ...
    want = canonical_from_arrays(d, "prefix_")
    m = len(want["codes"])
    for k in ("codes", "nq", "qubits", "bmask", "npar", "params", "cbit", "mat_len"):
        assert np.array_equal(got[k][:m], want[k]), k
    n_mat = int(want["mat_len"].sum())
    assert np.array_equal(got["mats"][:n_mat], want["mats"])
    # ... and all 983 376 through the digest
    assert digest(got) == str(d["fused_digest"])


def test_deep21_run_circuit_bit_exact(golden):
    d = golden("deep21")
    wl = deep21(d, trotter=1, n_steps=int(d["run_steps"]))
    fops, pool, stats = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    assert [stats["gates_before"], stats["gates_after"]] == list(d["run_fused_stats"])
    assert digest(canonical_from_packed(fops, wl.params, pool)) == str(d["run_fused_digest"])


def test_deep21_prefix_fixture_is_self_consistent(golden):
    """The committed prefix (the CPU reference arm's sample) parses as oracle IR."""
    d = golden("deep21")
    instrs, n = to_oracle(d, "prefix_")
    assert n == 21 and len(instrs) == 1500
    assert all(ins[3] is not None for ins in instrs if ins[0] in ("c1", "c2"))


@pytest.mark.gpu
def test_deep21_run_matches_reference_at_full_width(golden):
    """21 qubits, both assertions, the blocked kernel in one cooperative launch:
    assertion probabilities within 1e-12, samples for two seeds exactly the
    reference's, final-state digest (block norms, strided and largest
    amplitudes) within the 1e-10 relative bound."""
    from paper_2310_17739_b200.engine import DeviceProgram, StateVector, _sample_from, probabilities
    d = golden("deep21")
    wl = deep21(d, trotter=1, n_steps=int(d["run_steps"]))
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(21)
    prog = DeviceProgram(state, exe, wl.params, pool)
    assert prog.info.n_passes > 100
    probs = prog.run_mma()
    np.testing.assert_allclose(probs, d["run_probs"], rtol=0, atol=1e-12)
    p = probabilities(state)
    for seed in d["seeds"]:
        smp = _sample_from(p, 21, int(d["shots"]), np.random.Generator(np.random.Philox(int(seed))))
        want = dict(zip((str(k) for k in d[f"s{seed}_keys"]), (int(c) for c in d[f"s{seed}_counts"])))
        assert smp == want, seed
    amps = state.amps
    blog, stride, top = (int(x) for x in d["digest_params"])
    bn = (amps.real ** 2 + amps.imag ** 2).reshape(-1, 1 << blog).sum(axis=1)
    np.testing.assert_allclose(bn, d["run_block_norms"], rtol=0, atol=1e-12)
    strided = amps[::stride]
    assert np.linalg.norm(strided - d["run_strided"]) <= 1e-10 * np.linalg.norm(d["run_strided"])
    np.testing.assert_allclose(amps[d["run_top_idx"]], d["run_top_amps"], rtol=0, atol=1e-12)
