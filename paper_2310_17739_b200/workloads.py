"""Synthetic workloads for the BASELINE configs, emitted as packed op lists.

No Python Instruction objects are created for the large configs: the filter
circuit is written by the native emitter (csrc/generator.cpp, the
instruction stream of the reference's build_filter_circuit,
projection.py:191-255) and fused natively, so a 10^8-gate circuit costs
host C++ time only.

* ``shell_model_terms``  -- a seeded Jordan-Wigner shell-model Hamiltonian
  (one-body levels + hoppings, two-body density-density and pair terms) as
  sorted Pauli words; stands in for the paper's nuclear inputs
  (21 qubits = 20 modes + ancilla).
* ``filter_workload``    -- BASELINE config 3 (and 1/2 at other widths):
  projection-filter circuit with the halving schedule (projection.py:74-84).
* ``layered_workload``   -- BASELINE config 4: random layered 1q/2q circuit.
"""

from __future__ import annotations

import ctypes
import math
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .fusion import blas_variant
from .gates import Gate

# ---------------------------------------------------------------------------
# Pauli algebra on letter strings (qubit-0-first), enough for JW products

_MUL = {("I", "I"): (1, "I"), ("I", "X"): (1, "X"), ("I", "Y"): (1, "Y"), ("I", "Z"): (1, "Z"),
        ("X", "I"): (1, "X"), ("X", "X"): (1, "I"), ("X", "Y"): (1j, "Z"), ("X", "Z"): (-1j, "Y"),
        ("Y", "I"): (1, "Y"), ("Y", "X"): (-1j, "Z"), ("Y", "Y"): (1, "I"), ("Y", "Z"): (1j, "X"),
        ("Z", "I"): (1, "Z"), ("Z", "X"): (1j, "Y"), ("Z", "Y"): (-1j, "X"), ("Z", "Z"): (1, "I")}


def _mul(a: dict, b: dict) -> dict:
    out: dict[str, complex] = {}
    for s1, c1 in a.items():
        for s2, c2 in b.items():
            ph = c1 * c2
            word = []
            for p, q in zip(s1, s2):
                f, r = _MUL[(p, q)]
                ph *= f
                word.append(r)
            k = "".join(word)
            out[k] = out.get(k, 0j) + ph
    return out


def _ladder(i: int, n: int, create: bool) -> dict:
    z, pad = "Z" * i, "I" * (n - i - 1)
    return {z + "X" + pad: 0.5, z + "Y" + pad: (-0.5j if create else 0.5j)}


def shell_model_terms(n_modes: int, seed: int = 21, hop_range: int = 20,
                      pair_density: float = 0.35, n_scatter: int = 0) -> list[tuple[str, float]]:
    """Sorted (letters, coeff) of a seeded JW-mapped two-body Hamiltonian."""
    rng = np.random.default_rng(seed)
    cre = [_ladder(i, n_modes, True) for i in range(n_modes)]
    ann = [_ladder(i, n_modes, False) for i in range(n_modes)]
    h: dict[str, complex] = {}

    def add(terms: dict, scale: float):
        for k, v in terms.items():
            h[k] = h.get(k, 0j) + scale * v

    levels = np.sort(rng.uniform(-1.0, 1.0, n_modes))
    for i in range(n_modes):
        add(_mul(cre[i], ann[i]), float(levels[i]))
    for i in range(n_modes):
        for j in range(i + 1, min(n_modes, i + 1 + hop_range)):
            t = float(rng.uniform(-0.2, 0.2))
            add(_mul(cre[i], ann[j]), t)
            add(_mul(cre[j], ann[i]), t)
    for i in range(n_modes):
        for j in range(i + 1, n_modes):
            if rng.random() < pair_density:
                add(_mul(_mul(cre[i], ann[i]), _mul(cre[j], ann[j])), float(rng.uniform(-0.3, 0.3)))
    for _ in range(n_scatter):  # pair scattering a+_i a+_j a_l a_k + h.c.
        i, j, k, l = (int(x) for x in rng.choice(n_modes, 4, replace=False))
        v = float(rng.uniform(-0.1, 0.1))
        fwd = _mul(_mul(cre[i], cre[j]), _mul(ann[l], ann[k]))
        bwd = _mul(_mul(cre[k], cre[l]), _mul(ann[j], ann[i]))
        add(fwd, v)
        add(bwd, v)
    return sorted((k, float(v.real)) for k, v in h.items() if abs(v) > 1e-12)


def halving_schedule(gap: float, n_steps: int) -> list[tuple[float, float]]:
    """t_1 = pi / (2 gap), t_i = t_{i-1} / 2, zero phases (projection.py:74-84)."""
    t1 = math.pi / (2.0 * gap)
    return [(t1 / 2.0 ** i, 0.0) for i in range(n_steps)]


# ---------------------------------------------------------------------------
# packed workloads


@dataclass
class Workload:
    name: str
    n_qubits: int
    ancilla: int | None
    ops: np.ndarray              # packed input instruction list (OP_DTYPE)
    params: np.ndarray           # float64 params pool
    payloads: np.ndarray         # complex128 payload pool
    input_gates: int
    meta: dict = field(default_factory=dict)

    def executable(self, ops: np.ndarray) -> np.ndarray:
        """Drop the trailing measure/barrier sampling block (engine.py:305-307)."""
        kinds = ops["kind"]
        end = len(ops)
        while end > 0 and kinds[end - 1] in (N.OP_MEASURE, N.OP_BARRIER):
            end -= 1
        return ops[:end]


def _adopt(ptr, n_bytes: int) -> np.ndarray:
    """A uint8 array over a library-allocated buffer, released with nsb_free
    when the last view of it goes (no copy: 10^8-gate plans are GBs)."""
    addr = ctypes.cast(ptr, ctypes.c_void_p).value
    buf = (ctypes.c_uint8 * n_bytes).from_address(addr)
    weakref.finalize(buf, N.lib().nsb_free, ctypes.c_void_p(addr))
    return np.frombuffer(buf, np.uint8)


def _take_fused(f: N.Fused) -> tuple[np.ndarray, np.ndarray]:
    """Take ownership of nsb_fused's buffers (f's pointers are cleared)."""
    ops = _adopt(f.ops, max(f.n_ops, 1) * N.OP_DTYPE.itemsize).view(N.OP_DTYPE)[: f.n_ops]
    f.ops = None
    if f.payloads and f.n_payload > 0:
        pool = _adopt(f.payloads, 16 * f.n_payload).view(np.complex128)
        f.payloads = None
    else:
        pool = np.zeros(1, np.complex128)
    return ops, pool


def fuse_packed(ops: np.ndarray, params: np.ndarray, payloads: np.ndarray,
                variant: int | None = None):
    """nsb_fuse on packed arrays -> (fused ops, payload pool, stats dict)."""
    f = N.Fused()
    st = N.Status()
    code = N.lib().nsb_fuse(N.ptr(ops), len(ops), N.ptr(params),
                            N.ptr(payloads.view(np.float64)), N.PASS_ALL,
                            blas_variant() if variant is None else variant,
                            ctypes.byref(f), ctypes.byref(st))
    N.check(code, st)
    try:
        fops, pool = _take_fused(f)
        stats = {"gates_before": int(f.gates_before), "gates_after": int(f.pass_after[3]),
                 "per_pass": [(int(b), int(a)) for b, a in zip(f.pass_before, f.pass_after)]}
    finally:
        N.lib().nsb_fused_free(ctypes.byref(f))
    return fops, pool, stats


def filter_workload(n_system: int, trotter: int, n_steps: int = 8, seed: int = 21,
                    gap: float = 0.5, hop_range: int = 20, pair_density: float = 0.35,
                    n_scatter: int = 0,
                    terms: list[tuple[str, float]] | None = None,
                    steps: list[tuple[float, float]] | None = None,
                    trial: str | None = None) -> Workload:
    """Projection-filter circuit (n_system + ancilla qubits) emitted natively."""
    terms = terms if terms is not None else shell_model_terms(n_system, seed, hop_range,
                                                              pair_density, n_scatter)
    steps = steps if steps is not None else halving_schedule(gap, n_steps)
    letters = np.array([["IXYZ".index(c) for c in l] for l, _ in terms], np.uint8).reshape(-1)
    coeffs = np.array([c for _, c in terms], np.float64)
    st_arr = np.array(steps, np.float64).reshape(-1)
    trial_bits = np.array([int(b) for b in (trial or "0" * n_system)], np.uint8)
    f = N.Fused()
    pp = ctypes.POINTER(ctypes.c_double)()
    npar = ctypes.c_int64(0)
    st = N.Status()
    code = N.lib().nsb_generate_filter(n_system, N.ptr(letters), N.ptr(coeffs), len(terms),
                                       N.ptr(st_arr), len(steps), trotter, N.ptr(trial_bits),
                                       ctypes.byref(f), ctypes.byref(pp), ctypes.byref(npar),
                                       ctypes.byref(st))
    N.check(code, st)
    try:
        ops, _ = _take_fused(f)
        params = np.ctypeslib.as_array(pp, shape=(max(npar.value, 1),)).copy()
        gates = int(f.gates_before)
    finally:
        N.lib().nsb_fused_free(ctypes.byref(f))
        N.lib().nsb_free(ctypes.cast(pp, ctypes.c_void_p))
    two_q = int(np.count_nonzero((ops["kind"] == N.OP_GATE) & (ops["nq"] == 2)))
    return Workload(f"filter{n_system + 1}", n_system + 1, n_system, ops, params,
                    np.zeros(1, np.complex128), gates,
                    {"terms": len(terms), "trotter": trotter, "filter_steps": len(steps),
                     "two_qubit_fraction": two_q / max(gates, 1),
                     "gates_per_slice": gates / max(len(steps) * trotter, 1)})


def layered_workload(n: int, layers: int, seed: int = 28) -> Workload:
    """BASELINE config 4: per layer U3 on every qubit, then a random perfect
    matching of {CX, CZ, RZZ} pairs; no mid-circuit measurements."""
    rng = np.random.default_rng(seed)
    n_ops = layers * (n + n // 2)
    ops = np.zeros(n_ops, dtype=N.OP_DTYPE)
    params = []
    i = 0
    two = (Gate.CX, Gate.CZ, Gate.RZZ)
    for _ in range(layers):
        for q in range(n):
            ops[i]["kind"], ops[i]["tag"], ops[i]["nq"] = N.OP_GATE, Gate.U3.code, 1
            ops[i]["q"] = (q, -1, -1, -1, -1)
            ops[i]["param"] = len(params)
            params.extend(rng.uniform(-math.pi, math.pi, 3))
            ops[i]["mask"] = 1 << q
            i += 1
        perm = rng.permutation(n)
        for k in range(0, n - 1, 2):
            a, b = int(perm[k]), int(perm[k + 1])
            g = two[int(rng.integers(3))]
            ops[i]["kind"], ops[i]["tag"], ops[i]["nq"] = N.OP_GATE, g.code, 2
            ops[i]["q"] = (a, b, -1, -1, -1)
            ops[i]["param"] = -1
            if g is Gate.RZZ:
                ops[i]["param"] = len(params)
                params.append(float(rng.uniform(-math.pi, math.pi)))
            ops[i]["mask"] = (1 << a) | (1 << b)
            i += 1
    ops = ops[:i]
    ops["cbit"], ops["src"], ops["payload"] = -1, -1, -1
    return Workload(f"layered{n}", n, None, ops, np.asarray(params, np.float64),
                    np.zeros(1, np.complex128), i, {"layers": layers})


CLASS_NAMES = ("dense1", "diag1", "dense2", "sparse2", "mono2", "diag2", "cx01", "cx10",
               "pair_q", "pair_p", "pair_x", "swap", "permute", "pair_q_real", "pair_p_real",
               "pair_x_real")  # planner.h GateClass order; NSB_N_CLASSES entries


def plan_analyze(ops: np.ndarray, params: np.ndarray, payloads: np.ndarray, n: int) -> dict:
    """Host-only planner dry run (nsb_plan_analyze)."""
    info = N.PlanInfo()
    classes = np.zeros(len(CLASS_NAMES), np.int64)
    st = N.Status()
    N.check(N.lib().nsb_plan_analyze(N.ptr(ops), len(ops), N.ptr(params),
                                     N.ptr(payloads.view(np.float64)), n, ctypes.byref(info),
                                     N.ptr(classes), ctypes.byref(st)), st)
    out = {k: int(getattr(info, k)) for k, _ in N.PlanInfo._fields_}
    out["classes"] = dict(zip(CLASS_NAMES, map(int, classes)))
    return out
