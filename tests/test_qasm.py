"""Native OpenQASM reader (csrc/qasm.cpp via paper_2310_17739_b200.qasm)
against golden outputs of the reference parser (tests/golden/qasm.json,
made by tests/golden/make_qasm_golden.py from nucsim.qasm.parse_qasm):
identical circuits -- tags, qubits, bit-identical folded angles, classical
bits, registers -- and identical QasmError messages, lines and columns."""

import json

import numpy as np
import pytest

from conftest import ROOT
from paper_2310_17739_b200 import QasmError
from paper_2310_17739_b200 import _native as N
from paper_2310_17739_b200.qasm import parse_qasm, parse_qasm_packed

CASES = json.loads((ROOT / "tests" / "golden" / "qasm.json").read_text())


def _summary(c):
    return {"n_qubits": c.n_qubits, "cregs": [list(x) for x in c.cregs],
            "instructions": [[i.gate.value, list(i.qubits), [float(p).hex() for p in i.params],
                              i.cbit] for i in c.instructions]}


@pytest.mark.parametrize("i", range(len(CASES)))
def test_against_reference_parser(i):
    case = CASES[i]
    if "error" in case:
        with pytest.raises(QasmError) as ei:
            parse_qasm(case["text"])
        msg, line, col = case["error"]
        assert (str(ei.value), ei.value.line, ei.value.col) == (
            f"line {line}, column {col}: {msg}", line, col)
    else:
        got = _summary(parse_qasm(case["text"]))
        want = {k: case[k] for k in ("n_qubits", "cregs", "instructions")}
        assert got == want


def test_packed_records_feed_the_device_path():
    """parse_qasm_packed: op records with masks and parameter offsets that
    nsb_fuse accepts directly (no Python instruction objects)."""
    from paper_2310_17739_b200 import workloads as W
    text = next(c["text"] for c in CASES if "error" not in c and len(c["instructions"]) > 30)
    prog = parse_qasm_packed(text)
    ops = prog.ops
    assert ops.dtype == N.OP_DTYPE
    for rec in ops:
        qs = [int(q) for q in rec["q"][: int(rec["nq"])]]
        if int(rec["kind"]) == N.OP_BARRIER:
            o, k = int(rec["param"]), int(rec["cbit"])
            qs = [int(q) for q in prog.barrier_qubits[o: o + k]]
        assert int(rec["mask"]) == sum(1 << q for q in set(qs))
    fops, pool, stats = W.fuse_packed(ops, prog.params, np.zeros(1, np.complex128))
    assert stats["gates_before"] == int((ops["kind"] == N.OP_GATE).sum())


def test_large_file_throughput():
    """A 10^5-gate file parses natively (the reference manages ~45k gates/s)."""
    import time
    body = "".join(f"rz({k % 7}*pi/8) q[{k % 20}];\ncx q[{k % 20}], q[{(k + 1) % 20}];\n"
                   for k in range(50_000))
    text = 'OPENQASM 2.0;\ninclude "qelib1.inc";\nqreg q[20];\n' + body
    t = time.perf_counter()
    prog = parse_qasm_packed(text)
    dt = time.perf_counter() - t
    assert len(prog.ops) == 100_000
    assert dt < 5.0


def test_deep_nesting_and_garbage_do_not_crash():
    deep = "OPENQASM 2.0;\nqreg q[1];\nrz(" + "(" * 100000 + "1" + ")" * 100000 + ") q[0];\n"
    with pytest.raises(QasmError, match="nested too deeply"):
        parse_qasm(deep)
    rng = np.random.default_rng(5)
    alphabet = list("OPENQASM2.0;qregcx[](),->pi+*/ \n\"qelib1.inc\"measurebarrier0123456789")
    for _ in range(300):
        text = "".join(rng.choice(alphabet, size=int(rng.integers(0, 200))))
        try:
            parse_qasm(text)
        except QasmError:
            pass
