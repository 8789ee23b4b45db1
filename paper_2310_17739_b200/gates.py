"""Gate tags and their dense little-endian matrices (the boundary vocabulary).

Semantics follow the reference's nucsim/gates.py:1-17 (slot 0 = least
significant matrix bit, controls in the low slots, U3/U1/RZ/RZZ phase
conventions) and must be *bit-identical* to its ``gate_matrix``
(gates.py:111-291): fused payloads are products of these matrices and the
fusion pass is required to reproduce the reference's fused list exactly.
Every trigonometric value therefore comes from libm (``math.cos`` /
``math.sin``), which the reference reaches through ``np.exp(1j*x)``
(identical for all sampled x).

The integer ``code`` of each tag is the tag id used across the C ABI
(include/nucsim_b200.h, ``NSB_GATE_*``); the native generator in
csrc/gates.cpp rebuilds the 1- and 2-qubit matrices from the same formulas.
"""

from __future__ import annotations

import math
from enum import Enum
from functools import lru_cache

import numpy as np

_R = math.sqrt(0.5)


class Gate(Enum):
    """Instruction tags; values are the OpenQASM spellings (reference gates.py:30-71)."""

    U3 = "u3"
    U2 = "u2"
    U1 = "u1"
    CX = "cx"
    ID = "id"
    X = "x"
    Y = "y"
    Z = "z"
    H = "h"
    S = "s"
    SDG = "sdg"
    T = "t"
    TDG = "tdg"
    RX = "rx"
    RY = "ry"
    RZ = "rz"
    CZ = "cz"
    CY = "cy"
    SWAP = "swap"
    CH = "ch"
    CCX = "ccx"
    CSWAP = "cswap"
    CRX = "crx"
    CRY = "cry"
    CRZ = "crz"
    CU1 = "cu1"
    CU3 = "cu3"
    RXX = "rxx"
    RZZ = "rzz"
    RCCX = "rccx"
    RC3X = "rc3x"
    C3X = "c3x"
    C3SQRTX = "c3sqrtx"
    C4X = "c4x"
    C1 = "c1"
    C2 = "c2"
    MEASURE = "measure"
    RESET = "reset"
    BARRIER = "barrier"

    @property
    def code(self) -> int:
        return _CODE[self]

    @property
    def n_qubits(self) -> int:
        return _ARITY[self][0]

    @property
    def n_params(self) -> int:
        return _ARITY[self][1]

    @property
    def is_unitary(self) -> bool:
        return self not in MARKERS


MARKERS = frozenset((Gate.MEASURE, Gate.RESET, Gate.BARRIER))
_CODE = {g: i for i, g in enumerate(Gate)}
BY_CODE = tuple(Gate)

# (qubits, params); barrier spans any qubit set
_ARITY = {g: (1, 0) for g in Gate}
for _g, _shape in {
    "u3": (1, 3), "u2": (1, 2), "u1": (1, 1), "rx": (1, 1), "ry": (1, 1), "rz": (1, 1),
    "cx": (2, 0), "cz": (2, 0), "cy": (2, 0), "swap": (2, 0), "ch": (2, 0),
    "crx": (2, 1), "cry": (2, 1), "crz": (2, 1), "cu1": (2, 1), "cu3": (2, 3),
    "rxx": (2, 1), "rzz": (2, 1), "c2": (2, 0),
    "ccx": (3, 0), "cswap": (3, 0), "rccx": (3, 0),
    "c3x": (4, 0), "c3sqrtx": (4, 0), "rc3x": (4, 0), "c4x": (5, 0),
    "barrier": (0, 0),
}.items():
    _ARITY[Gate(_g)] = _shape

QASM_NAMES = {g.value: g for g in Gate if g.is_unitary and g not in (Gate.C1, Gate.C2)}


# ---------------------------------------------------------------------------
# matrix construction


def _phase(x: float) -> complex:
    """e^{ix} as libm (cos x, sin x)."""
    return complex(math.cos(x), math.sin(x))


def _u3_entries(theta: float, phi: float, lam: float):
    half = theta / 2
    c, s = math.cos(half), math.sin(half)
    el, ep, epl = _phase(lam), _phase(phi), _phase(phi + lam)
    return (complex(c, 0.0), complex(-el.real * s, -el.imag * s),
            complex(ep.real * s, ep.imag * s), complex(epl.real * c, epl.imag * c))


def _one_qubit(gate: Gate, p: tuple[float, ...]):
    """(u00, u01, u10, u11) of a 1-qubit tag."""
    if gate is Gate.U3:
        return _u3_entries(*p)
    if gate is Gate.U2:
        return _u3_entries(math.pi / 2, p[0], p[1])
    if gate is Gate.U1:
        return (1, 0, 0, _phase(p[0]))
    if gate in (Gate.RX, Gate.RY):
        half = p[0] / 2
        c, s = math.cos(half), math.sin(half)
        if gate is Gate.RX:
            return (c, complex(0.0, -s), complex(0.0, -s), c)
        return (c, -s, s, c)
    if gate is Gate.RZ:
        half = p[0] / 2
        c, s = math.cos(half), math.sin(half)
        return (complex(c, -s), 0, 0, complex(c, s))
    fixed = {
        Gate.ID: (1, 0, 0, 1),
        Gate.X: (0, 1, 1, 0),
        Gate.Y: (0, -1j, 1j, 0),
        Gate.Z: (1, 0, 0, -1),
        Gate.H: (_R, _R, _R, -_R),
        Gate.S: (1, 0, 0, 1j),
        Gate.SDG: (1, 0, 0, -1j),
        Gate.T: (1, 0, 0, _phase(math.pi / 4)),
        Gate.TDG: (1, 0, 0, complex(math.cos(math.pi / 4), -math.sin(math.pi / 4))),
    }
    return fixed[gate]


_CONTROLLED_BASE = {Gate.CX: Gate.X, Gate.CY: Gate.Y, Gate.CZ: Gate.Z, Gate.CH: Gate.H,
                    Gate.CRX: Gate.RX, Gate.CRY: Gate.RY, Gate.CRZ: Gate.RZ,
                    Gate.CU1: Gate.U1, Gate.CU3: Gate.U3}


def _controlled(entries, n_controls: int) -> np.ndarray:
    """Target in the top slot, all controls set selects the 2x2 block."""
    dim = 2 << n_controls
    m = np.eye(dim, dtype=complex)
    lo = (1 << n_controls) - 1
    hi = lo | (1 << n_controls)
    m[lo, lo], m[lo, hi], m[hi, lo], m[hi, hi] = entries
    return m


def _embed(u: np.ndarray, slots: tuple[int, ...], width: int) -> np.ndarray:
    """Scatter a gate over `slots` of a width-slot register (exact placement)."""
    dim = 1 << width
    k = len(slots)
    out = np.zeros((dim, dim), dtype=complex)
    for col in range(dim):
        sub_col = 0
        for j, s in enumerate(slots):
            sub_col |= ((col >> s) & 1) << j
        rest = col
        for s in slots:
            rest &= ~(1 << s)
        for sub_row in range(1 << k):
            v = u[sub_row, sub_col]
            if v != 0:
                row = rest
                for j, s in enumerate(slots):
                    row |= ((sub_row >> j) & 1) << s
                out[row, col] = out[row, col] + v
    return out


def _sequence(width: int, body) -> np.ndarray:
    """Product of a gate list, first element applied first (numpy matmul order)."""
    acc = np.eye(1 << width, dtype=complex)
    for u, slots in body:
        acc = _embed(u, slots, width) @ acc
    return acc


def _relative_phase_toffolis():
    h_like = np.array(_u3_entries(math.pi / 2, 0.0, math.pi), dtype=complex).reshape(2, 2)
    t = np.array(_one_qubit(Gate.U1, (math.pi / 4,)), dtype=complex).reshape(2, 2)
    tdg = np.array(_one_qubit(Gate.U1, (-math.pi / 4,)), dtype=complex).reshape(2, 2)
    cx = _controlled((0, 1, 1, 0), 1)
    rccx = _sequence(3, [(h_like, (2,)), (t, (2,)), (cx, (1, 2)), (tdg, (2,)),
                         (cx, (0, 2)), (t, (2,)), (cx, (1, 2)), (tdg, (2,)),
                         (h_like, (2,))])
    rc3x = _sequence(4, [(h_like, (3,)), (t, (3,)), (cx, (2, 3)), (tdg, (3,)),
                         (h_like, (3,)), (cx, (0, 3)), (t, (3,)), (cx, (1, 3)),
                         (tdg, (3,)), (cx, (0, 3)), (t, (3,)), (cx, (1, 3)),
                         (tdg, (3,)), (h_like, (3,)), (t, (3,)), (cx, (2, 3)),
                         (tdg, (3,)), (h_like, (3,))])
    return rccx, rc3x


def _build(gate: Gate, p: tuple[float, ...]) -> np.ndarray:
    n = gate.n_qubits
    if n == 1:
        return np.array(_one_qubit(gate, p), dtype=complex).reshape(2, 2)
    if gate in _CONTROLLED_BASE:
        return _controlled(_one_qubit(_CONTROLLED_BASE[gate], p), 1)
    if gate is Gate.SWAP:
        return np.eye(4, dtype=complex)[[0, 2, 1, 3]]
    if gate is Gate.RXX:
        half = p[0] / 2
        c, s = math.cos(half), math.sin(half)
        m = np.diag(np.full(4, c, dtype=complex))
        m[[0, 1, 2, 3], [3, 2, 1, 0]] = complex(0.0, -s)
        return m
    if gate is Gate.RZZ:
        e = _phase(p[0])
        return np.diag(np.array([1, e, e, 1], dtype=complex))
    if gate is Gate.CCX:
        return _controlled((0, 1, 1, 0), 2)
    if gate is Gate.C3X:
        return _controlled((0, 1, 1, 0), 3)
    if gate is Gate.C4X:
        return _controlled((0, 1, 1, 0), 4)
    if gate is Gate.C3SQRTX:
        return _controlled((0.5 + 0.5j, 0.5 - 0.5j, 0.5 - 0.5j, 0.5 + 0.5j), 3)
    if gate is Gate.CSWAP:
        return np.eye(8, dtype=complex)[[0, 1, 2, 5, 4, 3, 6, 7]]
    if gate in (Gate.RCCX, Gate.RC3X):
        rccx, rc3x = _relative_phase_toffolis()
        return rccx if gate is Gate.RCCX else rc3x
    raise ValueError(f"{gate.value} has no closed-form matrix")


@lru_cache(maxsize=65536)
def _cached(gate: Gate, params: tuple[float, ...]) -> np.ndarray:
    m = np.ascontiguousarray(_build(gate, params), dtype=complex)
    m.setflags(write=False)
    return m


def gate_matrix(gate: Gate, params: tuple[float, ...] = ()) -> np.ndarray:
    """Dense matrix of a named gate (a fresh writable copy).

    Raises ValueError for markers and for the payload-carrying C1/C2 tags,
    and on a parameter-count mismatch (reference gates.py:283-291).
    """
    if not gate.is_unitary:
        raise ValueError(f"{gate.value} is not a unitary gate")
    if gate in (Gate.C1, Gate.C2):
        raise ValueError(f"{gate.value} carries its matrix on the instruction")
    if len(params) != gate.n_params:
        raise ValueError(f"{gate.value} expects {gate.n_params} parameters, got {len(params)}")
    return _cached(gate, tuple(float(x) for x in params)).copy()
