"""OpenQASM 2.0 input through the native reader (csrc/qasm.cpp).

``parse_qasm(text)`` returns the reference's :class:`Circuit` for the
reference's subset (nucsim/qasm.py:30-347: header and qelib1 include, one
qreg, named cregs, the qelib1 gate names, measure / reset / barrier in
indexed or whole-register form, ``//`` comments, constant angle
expressions); errors raise :class:`QasmError` with the reference's message,
line and column.  ``parse_qasm_packed(text)`` stops at the packed op records
(no Python objects per instruction), the input ``workloads.fuse_packed`` and
``DeviceProgram`` take -- the path for 10^8-gate files.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .circuit import Circuit, Instruction
from .gates import BY_CODE, Gate


@dataclass
class QasmProgram:
    n_qubits: int
    cregs: list[tuple[str, int]]
    ops: np.ndarray             # nsb_op records (N.OP_DTYPE)
    params: np.ndarray          # float64 parameter pool
    barrier_qubits: np.ndarray  # operand lists of barrier records (first-occurrence order)


def parse_qasm_packed(text: str) -> QasmProgram:
    data = text.encode("utf-8")
    q = N.Qasm()
    st = N.Status()
    code = N.lib().nsb_qasm_parse(data, len(data), ctypes.byref(q), ctypes.byref(st))
    try:
        N.check(code, st)
        ops = np.empty(q.n_ops, dtype=N.OP_DTYPE)
        if q.n_ops:
            ctypes.memmove(ops.ctypes.data, q.ops, q.n_ops * N.OP_DTYPE.itemsize)
        params = np.ctypeslib.as_array(q.params, (max(q.n_params, 1),))[: q.n_params].copy()
        bq = np.ctypeslib.as_array(q.barrier_qubits,
                                   (max(q.n_barrier_qubits, 1),))[: q.n_barrier_qubits].copy()
        cregs = []
        if q.n_cregs:
            sizes = np.ctypeslib.as_array(q.creg_sizes, (q.n_cregs,)).copy()
            pos = 0
            for i in range(q.n_cregs):  # NUL-terminated names back to back
                name = ctypes.string_at(q.creg_names + pos)
                pos += len(name) + 1
                cregs.append((name.decode("utf-8"), int(sizes[i])))
        return QasmProgram(int(q.n_qubits), cregs, ops, params, bq)
    finally:
        if code == N.NSB_OK:
            N.lib().nsb_qasm_free(ctypes.byref(q))


def to_circuit(prog: QasmProgram) -> Circuit:
    """The reference Circuit of a parsed program (Instruction per record)."""
    c = Circuit(prog.n_qubits, prog.cregs)
    instrs = c.instructions
    ops, params, bq = prog.ops, prog.params, prog.barrier_qubits
    kinds = ops["kind"].tolist()
    tags = ops["tag"].tolist()
    nqs = ops["nq"].tolist()
    qs = ops["q"].tolist()
    pofs = ops["param"].tolist()
    cbits = ops["cbit"].tolist()
    for i, kind in enumerate(kinds):
        if kind == N.OP_GATE:
            g = BY_CODE[tags[i]]
            p0 = pofs[i]
            pars = tuple(float(x) for x in params[p0: p0 + g.n_params]) if g.n_params else ()
            instrs.append(Instruction(g, tuple(qs[i][: nqs[i]]), pars))
        elif kind == N.OP_MEASURE:
            instrs.append(Instruction(Gate.MEASURE, (qs[i][0],), cbit=cbits[i]))
        elif kind == N.OP_RESET:
            instrs.append(Instruction(Gate.RESET, (qs[i][0],)))
        else:
            o = pofs[i]
            instrs.append(Instruction(Gate.BARRIER, tuple(int(x) for x in bq[o: o + cbits[i]])))
    return c


def parse_qasm(text: str) -> Circuit:
    """Parse OpenQASM 2.0 text into a Circuit (reference qasm.parse_qasm)."""
    return to_circuit(parse_qasm_packed(text))
