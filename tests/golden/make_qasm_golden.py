"""Golden fixtures for the native OpenQASM reader, made by running the
REFERENCE parser (nucsim.qasm.parse_qasm, read-only from /root/reference)
on inputs generated here.  Run in the build container:

    python tests/golden/make_qasm_golden.py

Writes qasm.json: for every input text either the parsed circuit (qubits,
cregs, and per instruction the tag, qubits, params as float.hex, cbit) or
the QasmError's message, line and column.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from nucsim.errors import QasmError  # noqa: E402
from nucsim.gates import QASM_NAMES  # noqa: E402
from nucsim.qasm import parse_qasm  # noqa: E402

HEADER = 'OPENQASM 2.0;\ninclude "qelib1.inc";\n'


def rand_angle(rng: random.Random) -> str:
    """A constant expression in the accepted grammar."""
    atoms = ["pi", "0", "1", "2", "3.5", ".25", "1e-3", "2.5E+2", "7.", "1.5e1"]

    def gen(depth):
        r = rng.random()
        if depth > 2 or r < 0.35:
            a = rng.choice(atoms) if rng.random() < 0.6 else repr(round(rng.uniform(-4, 4), 6))
            if a.startswith("-"):
                a = "(" + a + ")"
            return a
        if r < 0.5:
            return rng.choice(["-", "+"]) + gen(depth + 1)
        if r < 0.65:
            return "(" + gen(depth + 1) + ")"
        op = rng.choice(["+", "-", "*", "/"])
        rhs = gen(depth + 1)
        if op == "/":
            rhs = "(" + rhs + "+9.75)"  # keep divisors away from zero
        return gen(depth + 1) + " " + op + " " + rhs

    return gen(0)


def random_program(rng: random.Random) -> str:
    n = rng.randint(1, 9)
    lines = [HEADER.rstrip("\n")]
    cregs = []
    if rng.random() < 0.5:
        cregs.append(("pre", rng.randint(1, 4)))
        lines.append(f"creg pre[{cregs[-1][1]}];  // before the qreg")
    lines.append(f"qreg q[{n}];")
    cregs.append(("c", n))
    lines.append(f"creg c[{n}];")
    names = [g for g, gate in QASM_NAMES.items() if gate.n_qubits <= n]
    for _ in range(rng.randint(5, 60)):
        r = rng.random()
        if r < 0.75:
            name = rng.choice(names)
            g = QASM_NAMES[name]
            qs = rng.sample(range(n), g.n_qubits)
            ps = "(" + ", ".join(rand_angle(rng) for _ in range(g.n_params)) + ")" if g.n_params else ""
            lines.append(f"{name}{ps} " + ", ".join(f"q[{q}]" for q in qs) + ";")
        elif r < 0.82:
            qs = [rng.randrange(n) for _ in range(rng.randint(1, 4))]
            parts = [f"q[{q}]" for q in qs] + (["q"] if rng.random() < 0.2 else [])
            lines.append("barrier " + ",".join(parts) + ";")
        elif r < 0.9:
            reg, size = rng.choice(cregs)
            lines.append(f"measure q[{rng.randrange(n)}] -> {reg}[{rng.randrange(size)}];")
        elif r < 0.95:
            lines.append(f"reset q[{rng.randrange(n)}];" if rng.random() < 0.8 else "reset q;")
        else:
            lines.append("// a comment line")
    if rng.random() < 0.5:
        lines.append("measure q -> c;")
    sep = rng.choice(["\n", "\n", "\r\n", "\n\t "])
    return sep.join(lines) + "\n"


ERRORS = [
    "OPENQASM 3.0;\nqreg q[1];\n",
    "qreg q[1];\n",
    'OPENQASM 2.0;\ninclude "other.inc";\nqreg q[1];\n',
    'OPENQASM 2.0;\ninclude "qelib1.inc"\nqreg q[1];\n',
    HEADER + "qreg q[2];\nfoo q[0];\n",
    HEADER + "qreg q[2];\ngate g a { x a; }\n",
    HEADER + "qreg q[2];\nopaque g a;\n",
    HEADER + "qreg q[2];\ncreg c[2];\nif (c==1) x q[0];\n",
    HEADER + "qreg q[2];\nqreg r[2];\n",
    HEADER + "qreg q[0];\n",
    HEADER + "qreg q;\n",
    HEADER + "creg c[2];\ncreg c[1];\nqreg q[2];\n",
    HEADER + "creg c[2];\nqreg q[2];\ncreg c[1];\n",
    HEADER + "creg c[0];\nqreg q[2];\n",
    HEADER + "x q[0];\nqreg q[2];\n",
    HEADER + "qreg q[2];\nrx q[0];\n",
    HEADER + "qreg q[2];\nrx(1, 2) q[0];\n",
    HEADER + "qreg q[2];\ncx q[0];\n",
    HEADER + "qreg q[2];\ncx q[1], q[1];\n",
    HEADER + "qreg q[2];\nx q;\n",
    HEADER + "qreg q[2];\nx q[2];\n",
    HEADER + "qreg q[2];\nx r[0];\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure q[0] -> c;\n",
    HEADER + "qreg q[2];\ncreg c[3];\nmeasure q -> c;\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure q[0] -> d[0];\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure r[0] -> c[0];\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure q[5] -> c[0];\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure q[0] -> c[7];\n",
    HEADER + "qreg q[2];\ncreg c[2];\nmeasure q[0] c[0];\n",
    HEADER + "qreg q[2];\nreset r[0];\n",
    HEADER + "qreg q[2];\nreset q[9];\n",
    HEADER + "qreg q[2];\nbarrier q[0], r[1];\n",
    HEADER + "qreg q[2];\nbarrier q[3];\n",
    HEADER + "qreg q[2];\nrx(1/0) q[0];\n",
    HEADER + "qreg q[2];\nrx(1/(pi-pi)) q[0];\n",
    HEADER + "qreg q[2];\nrx(*) q[0];\n",
    HEADER + "qreg q[2];\nrx(tau) q[0];\n",
    HEADER + "qreg q[2];\nrx(1.5 q[0];\n",
    HEADER + "qreg q[2];\nx q[0] @\n",
    HEADER + "qreg q[2];\nx q[0]",
    HEADER + "qreg q[2];\n5 x q[0];\n",
    HEADER + "qreg q[2];\nx q[0];\n\n   cz q[0], q[0];\n",
    'OPENQASM 2.0;\ninclude "qelib1.inc;\n',
    HEADER,
    HEADER + "  // only a comment\n",
    "OPENQASM 2.0;\nqreg q[1];\nc1 q[0];\n",
    "OPENQASM 2.0;\nqreg q[1];\nx q[0] -> q[0];\n",
    "OPENQASM 2.0;\nqreg q[1];\nrz(1e) q[0];\n",
    "OPENQASM 2.0;\nqreg q[1];\nrz(.) q[0];\n",
    "OPENQASM 2.0;\nqreg q[1];\nu2(-(-pi)/2,  +3) q[0];\nbarrier q[0],;\n",
]


def record(text: str) -> dict:
    try:
        c = parse_qasm(text)
    except QasmError as exc:
        msg = str(exc).split(": ", 1)[1]
        return {"text": text, "error": [msg, exc.line, exc.col]}
    return {"text": text, "n_qubits": c.n_qubits, "cregs": [list(x) for x in c.cregs],
            "instructions": [[i.gate.value, list(i.qubits), [float(p).hex() for p in i.params],
                              i.cbit] for i in c.instructions]}


def main():
    rng = random.Random(2310)
    cases = [record(random_program(rng)) for _ in range(120)] + [record(t) for t in ERRORS]
    (HERE / "qasm.json").write_text(json.dumps(cases, indent=0))
    n_err = sum("error" in c for c in cases)
    print(f"{len(cases)} cases ({n_err} errors) -> {HERE / 'qasm.json'}")


if __name__ == "__main__":
    main()
