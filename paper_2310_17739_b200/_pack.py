"""Circuit <-> packed op list (the nsb_op records of include/nucsim_b200.h).

``pack`` flattens a :class:`Circuit` into one structured numpy array plus a
float64 params pool and a complex128 payload pool; ``unpack_fused`` turns the
fusion library's output back into Instruction objects, reusing every input
instruction the passes left untouched (``src`` >= 0) so identities and
params survive exactly as in the reference's passes (fusion.py:82-93).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .circuit import Circuit, Instruction
from .gates import BY_CODE, Gate

_KIND = {Gate.MEASURE: N.OP_MEASURE, Gate.RESET: N.OP_RESET, Gate.BARRIER: N.OP_BARRIER}


class Packed:
    __slots__ = ("ops", "params", "payloads", "n_qubits")

    def __init__(self, ops, params, payloads, n_qubits):
        self.ops, self.params, self.payloads, self.n_qubits = ops, params, payloads, n_qubits


def pack(circuit: Circuit, instrs=None) -> Packed:
    instrs = circuit.instructions if instrs is None else instrs
    n = len(instrs)
    ops = np.zeros(n, dtype=N.OP_DTYPE)
    kind = np.zeros(n, np.int32)
    tag = np.zeros(n, np.int32)
    nq = np.zeros(n, np.int32)
    cbit = np.full(n, -1, np.int32)
    q = np.full((n, 5), -1, np.int32)
    param = np.full(n, -1, np.int64)
    payload = np.full(n, -1, np.int64)
    mask = np.zeros(n, np.uint64)
    params: list[float] = []
    pays: list[np.ndarray] = []
    n_pay = 0
    for i, ins in enumerate(instrs):
        g = ins.gate
        kind[i] = _KIND.get(g, N.OP_GATE)
        tag[i] = g.code
        qs = ins.qubits
        m = 0
        for j, qq in enumerate(qs):
            m |= 1 << qq
            if j < 5:
                q[i, j] = qq
        mask[i] = m
        nq[i] = 0 if g is Gate.BARRIER else len(qs)
        if ins.cbit is not None:
            cbit[i] = ins.cbit
        if ins.params:
            param[i] = len(params)
            params.extend(ins.params)
        if ins.matrix is not None or (kind[i] == N.OP_GATE and len(qs) >= 3):
            mat = np.ascontiguousarray(ins.resolved_matrix(), dtype=np.complex128).ravel()
            payload[i] = n_pay
            pays.append(mat)
            n_pay += mat.size
    ops["kind"], ops["tag"], ops["nq"], ops["cbit"] = kind, tag, nq, cbit
    ops["q"], ops["src"], ops["param"], ops["payload"], ops["mask"] = q, -1, param, payload, mask
    params_arr = np.asarray(params if params else [0.0], dtype=np.float64)
    payload_arr = np.concatenate(pays) if pays else np.zeros(1, np.complex128)
    return Packed(ops, params_arr, np.ascontiguousarray(payload_arr), circuit.n_qubits)


def unpack_fused(circuit: Circuit, instrs, fused_ops: np.ndarray, pool: np.ndarray) -> Circuit:
    out = circuit.copy_empty()
    dest = out.instructions
    for rec in fused_ops:
        src = int(rec["src"])
        if src >= 0:
            dest.append(instrs[src])
            continue
        k = int(rec["nq"])
        dim = 1 << k
        off = int(rec["payload"])
        mat = pool[off:off + dim * dim].reshape(dim, dim).copy()
        qubits = tuple(int(x) for x in rec["q"][:k])
        dest.append(Instruction(BY_CODE[int(rec["tag"])], qubits, (), mat))
    return out
