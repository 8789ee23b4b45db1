"""Gate fusion, same four passes and contract as the reference
(nucsim/fusion.py:1-251), executed natively by ``nsb_fuse``
(csrc/fusion.cpp).

Payloads are bit-identical to the reference's because the native matrix
products reproduce OpenBLAS zgemm's FMA order, which is what the
reference's ``@`` executes.  That order depends on the CPU core OpenBLAS
selected on this host, so the variant is probed once against numpy
(``blas_variant``) unless ``NUCSIM_BLAS_VARIANT`` pins it ("chain2" for
SkylakeX/SapphireRapids cores, "four" for Haswell/Zen).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _native as N
from ._pack import pack, unpack_fused
from .circuit import Circuit
from .gates import MARKERS

_PASS_NAMES = ("merge_1q", "absorb_1q", "normalize_2q_order", "fuse_2q")


@dataclass(frozen=True, slots=True)
class PassStats:
    name: str
    gates_before: int
    gates_after: int

    def to_dict(self) -> dict:
        return {"name": self.name, "gates_before": self.gates_before,
                "gates_after": self.gates_after}


@dataclass(frozen=True, slots=True)
class FusionStats:
    gates_before: int
    gates_after: int
    per_pass: tuple[PassStats, ...] = field(default_factory=tuple)

    @property
    def reduction_factor(self) -> float:
        return 1.0 if self.gates_before == 0 else self.gates_before / max(self.gates_after, 1)

    def to_dict(self) -> dict:
        return {"gates_before": self.gates_before, "gates_after": self.gates_after,
                "reduction_factor": self.reduction_factor,
                "per_pass": [p.to_dict() for p in self.per_pass]}


def gate_count(circuit: Circuit) -> int:
    """Unitary gates only; measure / reset / barrier do not count."""
    return sum(1 for ins in circuit.instructions if ins.gate not in MARKERS)


@lru_cache(maxsize=1)
def blas_variant() -> int:
    """zgemm FMA order of this host's numpy `@` for 2x2 complex products."""
    pinned = os.environ.get("NUCSIM_BLAS_VARIANT")
    if pinned:
        return {"chain2": N.BLAS_CHAIN2, "four": N.BLAS_FOUR}[pinned]
    rng = np.random.default_rng(20231017)
    hits = {N.BLAS_CHAIN2: 0, N.BLAS_FOUR: 0}
    for _ in range(64):
        a = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
        b = rng.normal(size=(2, 2)) + 1j * rng.normal(size=(2, 2))
        want = a @ b
        for variant in hits:
            got = _native_product(a, b, variant)
            hits[variant] += bool(np.array_equal(got, want))
    best = max(hits, key=hits.get)
    if hits[best] != 64:
        raise RuntimeError(f"numpy's zgemm order matches no known variant ({hits}); "
                           "set NUCSIM_BLAS_VARIANT")
    return best


def _native_product(a: np.ndarray, b: np.ndarray, variant: int) -> np.ndarray:
    """a @ b through the native fusion kernel (merge of two 1q payloads)."""
    c = Circuit(1)
    c.instructions.append(_payload_instr(b))
    c.instructions.append(_payload_instr(a))
    out, _ = _run_passes(c, 1, variant)
    return out.instructions[0].matrix


def _payload_instr(m):
    from .circuit import Instruction
    from .gates import Gate
    return Instruction(Gate.C1, (0,), (), np.ascontiguousarray(m, dtype=complex))


def _run_passes(circuit: Circuit, mask: int, variant: int | None = None):
    instrs = circuit.instructions
    packed = pack(circuit, instrs)
    f = N.Fused()
    st = N.Status()
    lib = N.lib()
    code = lib.nsb_fuse(N.ptr(packed.ops), len(instrs), N.ptr(packed.params),
                        N.ptr(packed.payloads.view(np.float64)), mask,
                        blas_variant() if variant is None else variant,
                        ctypes.byref(f), ctypes.byref(st))
    N.check(code, st)
    try:
        ops = np.ctypeslib.as_array(ctypes.cast(f.ops, ctypes.POINTER(ctypes.c_uint8)),
                                    shape=(max(f.n_ops, 1) * N.OP_DTYPE.itemsize,))
        ops = ops.view(N.OP_DTYPE)[: f.n_ops].copy()
        pool = np.ctypeslib.as_array(f.payloads, shape=(max(2 * f.n_payload, 2),))
        pool = pool.copy().view(np.complex128)
        out = unpack_fused(circuit, instrs, ops, pool)
        stats = (int(f.gates_before), list(f.pass_before), list(f.pass_after))
    finally:
        lib.nsb_fused_free(ctypes.byref(f))
    return out, stats


def merge_1q(circuit: Circuit) -> Circuit:
    """Runs of 1q gates on one qubit -> one C1 at the run's first slot (fusion.py:101-131)."""
    return _run_passes(circuit, 1)[0]


def absorb_1q(circuit: Circuit) -> Circuit:
    """Fold 1q gates into adjacent 2q gates until stable (fusion.py:134-184)."""
    return _run_passes(circuit, 2)[0]


def normalize_2q_order(circuit: Circuit) -> Circuit:
    """2q gates onto ascending operands by SWAP conjugation (fusion.py:187-199)."""
    return _run_passes(circuit, 4)[0]


def fuse_2q(circuit: Circuit) -> Circuit:
    """Runs of 2q gates on one ordered pair -> one C2 (fusion.py:202-237)."""
    return _run_passes(circuit, 8)[0]


def fuse_pipeline(circuit: Circuit) -> tuple[Circuit, FusionStats]:
    """All four passes in order, with per-pass gate counts (fusion.py:240-251)."""
    out, (before, pb, pa) = _run_passes(circuit, N.PASS_ALL)
    per_pass = tuple(PassStats(name, int(b), int(a)) for name, b, a in zip(_PASS_NAMES, pb, pa))
    return out, FusionStats(before, int(pa[3]), per_pass)
