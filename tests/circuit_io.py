"""Circuit <-> flat arrays, for the golden fixtures.

Works on any object with the reference's Circuit / Instruction shape
(``n_qubits``, ``cregs``, ``instructions``; ``gate.value``, ``qubits``,
``params``, ``matrix``, ``cbit``), so the fixture generator can serialise
reference circuits and the tests can rebuild them as this package's
circuits or as oracle IR tuples.  Barriers are stored as qubit masks.
"""

from __future__ import annotations

import numpy as np


def to_arrays(circuit, prefix: str = "") -> dict[str, np.ndarray]:
    instrs = circuit.instructions
    n = len(instrs)
    names = np.array([ins.gate.value for ins in instrs], dtype="U8")
    qubits = np.full((n, 5), -1, np.int32)
    nq = np.zeros(n, np.int32)
    bmask = np.zeros(n, np.uint64)
    params = np.zeros((n, 3), np.float64)
    npar = np.zeros(n, np.int32)
    cbit = np.full(n, -1, np.int32)
    mat_off = np.full(n, -1, np.int64)
    mats = []
    off = 0
    for i, ins in enumerate(instrs):
        if ins.gate.value == "barrier":
            m = 0
            for q in ins.qubits:
                m |= 1 << q
            bmask[i] = m
        else:
            nq[i] = len(ins.qubits)
            qubits[i, :len(ins.qubits)] = ins.qubits
        npar[i] = len(ins.params)
        params[i, :len(ins.params)] = ins.params
        if ins.cbit is not None:
            cbit[i] = ins.cbit
        if ins.matrix is not None:
            flat = np.ascontiguousarray(ins.matrix, dtype=np.complex128).ravel()
            mat_off[i] = off
            mats.append(flat)
            off += flat.size
    reg_names = np.array([r for r, _ in circuit.cregs] or [""], dtype="U16")
    reg_sizes = np.array([s for _, s in circuit.cregs] or [0], dtype=np.int64)
    out = {"names": names, "qubits": qubits, "nq": nq, "bmask": bmask, "params": params,
           "npar": npar, "cbit": cbit, "mat_off": mat_off,
           "mats": np.concatenate(mats) if mats else np.zeros(0, np.complex128),
           "n_qubits": np.int64(circuit.n_qubits), "reg_names": reg_names,
           "reg_sizes": reg_sizes}
    return {prefix + k: v for k, v in out.items()}


def _rows(d, prefix):
    g = lambda k: d[prefix + k]
    names, qubits, nq, bmask = g("names"), g("qubits"), g("nq"), g("bmask")
    params, npar, cbit, mat_off, mats = g("params"), g("npar"), g("cbit"), g("mat_off"), g("mats")
    for i in range(len(names)):
        name = str(names[i])
        if name == "barrier":
            m = int(bmask[i])
            qs = tuple(q for q in range(64) if m >> q & 1)
        else:
            qs = tuple(int(x) for x in qubits[i, :nq[i]])
        ps = tuple(float(x) for x in params[i, :npar[i]])
        mat = None
        if mat_off[i] >= 0:
            k = len(qs)
            dim = 1 << k
            mat = mats[mat_off[i]:mat_off[i] + dim * dim].reshape(dim, dim).copy()
        cb = None if cbit[i] < 0 else int(cbit[i])
        yield name, qs, ps, mat, cb


def to_oracle(d, prefix: str = ""):
    """Oracle IR: list of (name, qubits, params, matrix, cbit)."""
    return list(_rows(d, prefix)), int(d[prefix + "n_qubits"])


def to_circuit(d, prefix: str = ""):
    """This package's Circuit (instructions appended without re-validation)."""
    from paper_2310_17739_b200 import Circuit, Gate, Instruction
    regs = [(str(n), int(s)) for n, s in zip(d[prefix + "reg_names"], d[prefix + "reg_sizes"])
            if s > 0]
    c = Circuit(int(d[prefix + "n_qubits"]), regs)
    for name, qs, ps, mat, cb in _rows(d, prefix):
        c.instructions.append(Instruction(Gate(name), qs, ps, mat, cb))
    return c


def oracle_from_circuit(circuit):
    return [(ins.gate.value, tuple(ins.qubits), tuple(ins.params), ins.matrix, ins.cbit)
            for ins in circuit.instructions]
