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


# ---------------------------------------------------------------------------
# canonical digest of an instruction stream (for lists too large to commit)
#
# The stream is reduced to fixed-layout arrays -- gate code (position in the
# reference's Gate enum, gates.py:30-83), qubit count, qubits (-1 padded),
# barrier qubit mask, parameter count, parameters (0 padded), classical bit,
# payload length, and all payloads concatenated in row order (complex128,
# row-major) -- and sha256 runs over their bytes.  Equal digests mean
# identical instructions and bit-identical payloads.


def _gate_codes():
    from paper_2310_17739_b200.gates import Gate
    return {g.value: i for i, g in enumerate(Gate)}


def canonical_from_arrays(d: dict, prefix: str = "") -> dict:
    """Canonical arrays from to_arrays() output (reference circuits)."""
    g = lambda k: d[prefix + k]
    codes_of = _gate_codes()
    names = g("names")
    uniq, inv = np.unique(names, return_inverse=True)
    codes = np.array([codes_of[str(u)] for u in uniq], np.int16)[inv]
    nq = g("nq").astype(np.int8)
    mats = g("mats")
    mat_off = g("mat_off")
    mat_len = np.where(mat_off >= 0, 4 ** nq.astype(np.int64), 0).astype(np.int32)
    return {"codes": codes, "nq": nq, "qubits": g("qubits").astype(np.int32),
            "bmask": g("bmask").astype(np.uint64), "npar": g("npar").astype(np.int8),
            "params": g("params").astype(np.float64), "cbit": g("cbit").astype(np.int32),
            "mat_len": mat_len, "mats": np.ascontiguousarray(mats, np.complex128)}


def canonical_from_packed(ops, params, pool) -> dict:
    """Canonical arrays from a packed op list (nsb_op records + float64 params
    + complex payload pool), vectorised (10^6-row lists in about a second)."""
    from paper_2310_17739_b200 import _native as N
    from paper_2310_17739_b200.gates import BY_CODE, Gate
    n = len(ops)
    kind = ops["kind"].astype(np.int64)
    tag = ops["tag"].astype(np.int64)
    codes = tag.astype(np.int16).copy()
    codes[kind == N.OP_MEASURE] = Gate.MEASURE.code
    codes[kind == N.OP_RESET] = Gate.RESET.code
    codes[kind == N.OP_BARRIER] = Gate.BARRIER.code
    is_bar = kind == N.OP_BARRIER
    nq = np.where(is_bar, 0, ops["nq"]).astype(np.int8)
    q = ops["q"].astype(np.int32).copy()
    q[np.arange(5)[None, :] >= nq[:, None]] = -1
    bmask = np.where(is_bar, ops["mask"], 0).astype(np.uint64)
    npar_of = np.array([g.n_params for g in BY_CODE], np.int64)
    is_gate = kind == N.OP_GATE
    npar = np.where(is_gate & (ops["param"] >= 0), npar_of[np.clip(tag, 0, len(BY_CODE) - 1)], 0)
    pm = np.zeros((n, 3), np.float64)
    for j in range(3):
        sel = npar > j
        pm[sel, j] = params[ops["param"][sel] + j]
    has = is_gate & (ops["payload"] >= 0)
    mat_len = np.where(has, 4 ** nq.astype(np.int64), 0)
    starts = np.repeat(ops["payload"][has].astype(np.int64), mat_len[has])
    within = np.arange(int(mat_len.sum())) - np.repeat(np.cumsum(mat_len[has]) - mat_len[has],
                                                       mat_len[has])
    mats = pool[starts + within] if len(starts) else np.zeros(0, np.complex128)
    cbit = ops["cbit"].astype(np.int32)
    return {"codes": codes, "nq": nq, "qubits": q, "bmask": bmask, "npar": npar.astype(np.int8),
            "params": pm, "cbit": cbit, "mat_len": mat_len.astype(np.int32),
            "mats": np.ascontiguousarray(mats, np.complex128)}


def digest(c: dict) -> str:
    import hashlib
    h = hashlib.sha256()
    for k in ("codes", "nq", "qubits", "bmask", "npar", "params", "cbit", "mat_len", "mats"):
        a = np.ascontiguousarray(c[k])
        h.update(k.encode())
        h.update(np.int64(a.size).tobytes())
        h.update(a.tobytes())
    return h.hexdigest()
