"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container, where /root/reference exists:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

It imports the unmodified reference package (/root/reference/pkg/src/nucsim)
and its test helpers (/root/reference/pkg/tests/oracles.py) read-only and
writes small .npz fixtures next to this script.  The fixtures travel with the
repository, so GPU-box tests never need the reference.  Records the numpy /
OpenBLAS configuration the vectors came from (fusion payload bits depend on
OpenBLAS's zgemm kernel).
"""

from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import json  # noqa: E402
import math  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, str(ROOT / "tests"))

import nucsim  # noqa: E402
import oracles as ref_oracles  # noqa: E402
from nucsim import engine as ref_engine  # noqa: E402
from nucsim.gates import Gate as RGate  # noqa: E402

from circuit_io import to_arrays  # noqa: E402


def openblas_core() -> str:
    try:
        import ctypes
        import glob
        libs = os.path.join(os.path.dirname(np.__file__), os.pardir, "numpy.libs")
        lib = glob.glob(os.path.join(libs, "libscipy_openblas64_*.so"))[0]
        h = ctypes.CDLL(lib)
        fn = h.scipy_openblas_get_corename64_
        fn.restype = ctypes.c_char_p
        return fn().decode()
    except Exception as exc:  # pragma: no cover - informational only
        return f"unknown ({exc})"


def zgemm_variant() -> str:
    """Which restated FMA order numpy's 2x2 complex `@` follows on this host."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import nucsim_oracle as O
    rng = np.random.default_rng(5)
    for variant in ("chain2", "four"):
        mm = O.Matmul(variant)
        if all(np.array_equal(mm(a, b), a @ b) for a, b in (
                (rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)),
                 rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)))
                for n in (2, 2, 2, 4, 4, 8) for _ in range(50))):
            return variant
    raise RuntimeError("numpy's zgemm matches neither restated order")


def meta() -> dict:
    return {"numpy": np.__version__, "openblas_core": openblas_core(),
            "nucsim": nucsim.__version__, "generated": time.strftime("%Y-%m-%dT%H:%M:%SZ"),
            "variant": zgemm_variant()}


def final_state(circuit) -> np.ndarray:
    """Pre-sampling state through the reference kernels (test_acceptance.py:33-63)."""
    instrs = circuit.instructions
    end = len(instrs)
    while end > 0 and instrs[end - 1].gate in (RGate.MEASURE, RGate.BARRIER):
        end -= 1
    state = nucsim.StateVector(circuit.n_qubits)
    for ins in instrs[:end]:
        g = ins.gate
        if g in (RGate.BARRIER, RGate.RESET):
            continue
        if g is RGate.MEASURE:
            nucsim.assert_measure(state, ins.qubits[0])
            continue
        nucsim.apply_dense(state, ins.resolved_matrix(), ins.qubits)
    return state.amps.copy()


def samples_arrays(samples: dict, prefix: str) -> dict:
    keys = sorted(samples)
    return {prefix + "keys": np.array(keys or [""], dtype="U64"),
            prefix + "counts": np.array([samples[k] for k in keys] or [0], dtype=np.int64),
            prefix + "n": np.int64(len(keys))}


# ---------------------------------------------------------------------------


def make_gates():
    rng = np.random.default_rng(101)
    out = {}
    names, offs, pars, npar = [], [], [], []
    mats = []
    off = 0
    for g in RGate:
        if g in (RGate.C1, RGate.C2, RGate.MEASURE, RGate.RESET, RGate.BARRIER):
            continue
        k = g.n_params
        trials = [()] if k == 0 else (
            [tuple(rng.uniform(-2 * math.pi, 2 * math.pi, size=k)) for _ in range(60)]
            + [(0.0,) * k, (math.pi,) * k, (-math.pi / 2,) * k, (1e-9,) * k, (123.456,) * k])
        for p in trials:
            m = nucsim.gate_matrix(g, p).ravel()
            names.append(g.value)
            row = np.zeros(3)
            row[:k] = p
            pars.append(row)
            npar.append(k)
            offs.append(off)
            mats.append(m)
            off += m.size
    out["names"] = np.array(names, dtype="U8")
    out["params"] = np.array(pars)
    out["npar"] = np.array(npar, np.int32)
    out["mat_off"] = np.array(offs, np.int64)
    out["mats"] = np.concatenate(mats)
    return out


def random_circuit(rng, n, count, walls=True):
    c = nucsim.Circuit(n, [("c", 4)])
    ref_oracles.random_gates(rng, c, count // 2)
    if walls and rng.random() < 0.5:
        c.barrier()
    if walls and n >= 3 and rng.random() < 0.5:
        qs = tuple(int(x) for x in rng.choice(n, size=3, replace=False))
        c.gate_op(RGate.CCX if rng.random() < 0.5 else RGate.RCCX, qs)
    if walls and rng.random() < 0.5:
        q = int(rng.integers(n))
        c.measure(q, 0)
        c.reset(q)
    ref_oracles.random_gates(rng, c, count - count // 2, p_two=0.6)
    return c


def make_fusion():
    rng = np.random.default_rng(202)
    out = {}
    cases = []
    for _ in range(40):
        cases.append(ref_oracles.random_filter_shaped_circuit(
            rng, int(rng.integers(2, 6)), int(rng.integers(1, 4)), int(rng.integers(5, 41))))
    for _ in range(30):
        cases.append(random_circuit(rng, int(rng.integers(2, 7)), int(rng.integers(20, 81))))
    # already-fused inputs (idempotence) and a long 1q/2q chain
    for c in list(cases[:10]):
        cases.append(nucsim.fuse_pipeline(c)[0])
    out["n_cases"] = np.int64(len(cases))
    for i, c in enumerate(cases):
        out.update(to_arrays(c, f"c{i}_in_"))
        fused, stats = nucsim.fuse_pipeline(c)
        out.update(to_arrays(fused, f"c{i}_out_"))
        out[f"c{i}_stats"] = np.array([stats.gates_before, stats.gates_after]
                                      + [v for p in stats.per_pass
                                         for v in (p.gates_before, p.gates_after)], np.int64)
        if i % 5 == 0:  # individual passes
            from nucsim.fusion import absorb_1q, fuse_2q, merge_1q, normalize_2q_order
            out.update(to_arrays(merge_1q(c), f"c{i}_merge_"))
            out.update(to_arrays(absorb_1q(c), f"c{i}_absorb_"))
            out.update(to_arrays(normalize_2q_order(c), f"c{i}_norm_"))
            out.update(to_arrays(fuse_2q(c), f"c{i}_fuse2_"))
    return out


def make_kernels():
    rng = np.random.default_rng(303)
    out = {}
    i = 0
    for n in range(1, 7):
        for _ in range(6):
            amps = ref_oracles.random_state(rng, 2 ** n)
            width = int(rng.integers(1, min(n, 5) + 1))
            qubits = tuple(int(x) for x in rng.choice(n, size=width, replace=False))
            u = ref_oracles.random_unitary(rng, 2 ** width)
            s = nucsim.StateVector.from_amplitudes(amps.copy())
            nucsim.apply_dense(s, u, qubits)
            q = int(rng.integers(n))
            s2 = nucsim.StateVector.from_amplitudes(amps.copy())
            p = nucsim.measure_project(s2, q, 0) if ref_engine._branch_probability(
                s2.amps, q, 0) > 1e-12 else -1.0
            out[f"k{i}_n"] = np.int64(n)
            out[f"k{i}_amps"] = amps
            out[f"k{i}_u"] = u
            out[f"k{i}_qubits"] = np.array(qubits, np.int32)
            out[f"k{i}_out"] = s.amps.copy()
            out[f"k{i}_mq"] = np.int64(q)
            out[f"k{i}_mp"] = np.float64(p)
            out[f"k{i}_mout"] = s2.amps.copy()
            i += 1
    out["n_kernels"] = np.int64(i)
    # sampling: same state, three seeds
    amps = ref_oracles.random_state(rng, 2 ** 10)
    out["sample_amps"] = amps
    for seed in (0, 42, 2 ** 63 + 5):
        smp = nucsim.sample(nucsim.StateVector.from_amplitudes(amps.copy()), 5000, seed)
        out.update(samples_arrays(smp, f"sample_{seed}_"))
    out["sample_seeds"] = np.array([0, 42, 2 ** 63 + 5], dtype=np.uint64)
    # expectation
    letters = ["IXZYI", "YYIIZ", "ZZZZZ", "XIXIX", "IIIII", "YIIIY", "IZIZI"]
    coeffs = rng.normal(size=len(letters))
    h = nucsim.PauliHamiltonian(5, dict(zip(letters, coeffs)))
    amps5 = ref_oracles.random_state(rng, 32)
    out["exp_amps"] = amps5
    out["exp_letters"] = np.array(letters, dtype="U8")
    out["exp_coeffs"] = coeffs
    out["exp_value"] = np.float64(nucsim.expectation_pauli(
        nucsim.StateVector.from_amplitudes(amps5.copy()), h))
    return out


def filter_fixture(h_shifted, schedule, trotter, trial_bits, n_system, seeds, shots,
                   rejection_shots, energy_h, with_unfused: bool):
    out = {}
    circuit = nucsim.build_filter_circuit(h_shifted, schedule, trotter,
                                          nucsim.TrialState.basis(trial_bits), n_system)
    terms = [(l, c.real) for l, c in h_shifted.sorted_terms()]
    out["term_letters"] = np.array([[("IXYZ").index(ch) for ch in l] for l, _ in terms], np.uint8)
    out["term_coeffs"] = np.array([c for _, c in terms])
    out["steps"] = np.array(schedule.steps, dtype=np.float64)
    out["trotter"] = np.int64(trotter)
    out["trial"] = np.array([int(b) for b in trial_bits], np.uint8)
    out.update(to_arrays(circuit, "in_"))
    t0 = time.time()
    fused, stats = nucsim.fuse_pipeline(circuit)
    print(f"  fuse {nucsim.gate_count(circuit)} -> {stats.gates_after} in {time.time()-t0:.1f}s")
    out.update(to_arrays(fused, "fused_"))
    out["fused_stats"] = np.array([stats.gates_before, stats.gates_after]
                                  + [v for p in stats.per_pass for v in (p.gates_before, p.gates_after)],
                                  np.int64)
    ancilla = n_system
    out["seeds"] = np.array(seeds, np.int64)
    out["shots"] = np.int64(shots)
    hp = type(energy_h)(n_system + 1, {s + "I": c for s, c in energy_h.terms.items()})
    e_terms = [(l, c.real) for l, c in hp.sorted_terms()]
    out["energy_letters"] = np.array(["".join(l) for l, _ in e_terms], dtype="U64")
    out["energy_coeffs"] = np.array([c for _, c in e_terms])
    for seed in seeds:
        t0 = time.time()
        rep = nucsim.run(fused, "mma", shots=shots, seed=seed, ancilla=ancilla,
                         hamiltonian=hp if seed == seeds[0] else None)
        print(f"  mma seed {seed}: {time.time()-t0:.1f}s")
        out[f"mma_{seed}_probs"] = np.array(rep.assert_probs)
        out.update(samples_arrays(rep.samples, f"mma_{seed}_"))
        if seed == seeds[0]:
            out["energy"] = np.float64(rep.energy)
    if with_unfused:
        t0 = time.time()
        rep = nucsim.run(circuit, "mma", shots=shots, seed=seeds[0], ancilla=ancilla)
        print(f"  unfused mma: {time.time()-t0:.1f}s")
        out["unfused_probs"] = np.array(rep.assert_probs)
        out.update(samples_arrays(rep.samples, "unfused_"))
    out["final_state"] = final_state(fused)
    t0 = time.time()
    rej = nucsim.run(fused, "rejection", shots=rejection_shots, seed=seeds[0], ancilla=None)
    print(f"  rejection {rejection_shots} shots: {time.time()-t0:.1f}s")
    out["rej_shots"] = np.int64(rejection_shots)
    out["rej_accepted"] = np.int64(rej.accepted)
    out["rej_steps"] = np.array(rej.step_rejections, np.int64)
    out.update(samples_arrays(rej.samples, "rej_"))
    return out


def shell_model_8():
    """C1 `ucc8`: 7 modes + ancilla, seeded one-/two-body shell-model input."""
    rng = np.random.default_rng(7)
    sq = nucsim.SecondQuantizedInput(7)
    levels = np.sort(rng.uniform(-1.0, 1.0, size=7))
    for i in range(7):
        sq.add_t(i, i, float(levels[i]))
    for i in range(6):
        sq.add_t(i, i + 1, float(rng.uniform(-0.3, 0.3)))
    for i in range(7):
        for j in range(i + 1, 7):
            if rng.random() < 0.4:
                sq.add_v(i, j, i, j, float(rng.uniform(-0.4, 0.4)))
    h = nucsim.build_hamiltonian(sq)
    gs = nucsim.ground_state(h)
    shifted = nucsim.shift_rescale(h, gs.energy)
    return h, shifted, gs


def main():
    info = meta()
    print("numpy/openblas:", info)
    t0 = time.time()
    np.savez_compressed(HERE / "gates.npz", **make_gates())
    print(f"gates.npz {time.time()-t0:.1f}s")
    t0 = time.time()
    np.savez_compressed(HERE / "fusion.npz", **make_fusion())
    print(f"fusion.npz {time.time()-t0:.1f}s")
    t0 = time.time()
    np.savez_compressed(HERE / "kernels.npz", **make_kernels())
    print(f"kernels.npz {time.time()-t0:.1f}s")

    h, shifted, gs = shell_model_8()
    schedule = nucsim.default_schedule(gs.gap, 4)
    trial = "1100000"
    for r in range(1, 200):
        c = nucsim.build_filter_circuit(shifted, schedule, r, nucsim.TrialState.basis(trial), 7)
        if nucsim.gate_count(c) >= 10_000:
            break
    print(f"filter8: trotter {r}, {nucsim.gate_count(c)} gates")
    t0 = time.time()
    f8 = filter_fixture(shifted, schedule, r, trial, 7, [7, 11, 1234], 1024, 512, h, True)
    f8["e0"] = np.float64(gs.energy)
    np.savez_compressed(HERE / "filter8.npz", **f8)
    print(f"filter8.npz {time.time()-t0:.1f}s")

    # C2 `mcm16`: 15-site transverse-field chain (test_acceptance.py:66-76 shape)
    n = 15
    terms = {}
    for i in range(n):
        s = ["I"] * n
        s[i] = "X"
        terms["".join(s)] = 0.12 + 0.01 * i
    for i in range(n - 1):
        s = ["I"] * n
        s[i] = s[i + 1] = "Z"
        terms["".join(s)] = 0.08
    chain = nucsim.PauliHamiltonian(n, terms)
    sched16 = nucsim.default_schedule(0.5, 4)
    t0 = time.time()
    f16 = filter_fixture(chain, sched16, 38, "0" * n, n, [3, 42], 1024, 4, chain, True)
    np.savez_compressed(HERE / "filter16.npz", **f16)
    print(f"filter16.npz {time.time()-t0:.1f}s")
    (HERE / "META.json").write_text(json.dumps(info, indent=2) + "\n")


if __name__ == "__main__":
    main()
