"""Command line (paper_2310_17739_b200.cli, the reference's simulate / fuse
subcommands): QASM written from the golden filter8 circuit goes through the
native reader, native fusion and the GPU run; the JSON report must carry the
reference's assertion probabilities and samples (tests/golden/filter8.npz)."""

import json

import pytest

from circuit_io import to_circuit
from paper_2310_17739_b200 import fuse_pipeline
from paper_2310_17739_b200.cli import main
from paper_2310_17739_b200.gates import Gate


def emit(circuit) -> str:
    """OpenQASM 2.0 for a named-gate circuit (test helper; repr() round-trips)."""
    lines = ['OPENQASM 2.0;', 'include "qelib1.inc";', f"qreg q[{circuit.n_qubits}];"]
    lines += [f"creg {name}[{size}];" for name, size in circuit.cregs]
    for ins in circuit.instructions:
        qs = ", ".join(f"q[{q}]" for q in ins.qubits)
        if ins.gate is Gate.MEASURE:
            reg, off = circuit.clbit_location(ins.cbit)
            lines.append(f"measure q[{ins.qubits[0]}] -> {reg}[{off}];")
        elif ins.gate in (Gate.RESET, Gate.BARRIER):
            lines.append(f"{ins.gate.value} {qs};")
        else:
            ps = "(" + ", ".join(repr(float(p)) for p in ins.params) + ")" if ins.params else ""
            lines.append(f"{ins.gate.value}{ps} {qs};")
    return "\n".join(lines) + "\n"


@pytest.fixture
def filter8_qasm(golden, tmp_path):
    d = golden("filter8")
    c = to_circuit(d, "in_")
    path = tmp_path / "filter8.qasm"
    path.write_text(emit(c))
    return d, c, path


def test_fuse_command_prints_reference_stats(filter8_qasm, capsys):
    d, c, path = filter8_qasm
    assert main(["fuse", "--input", str(path)]) == 0
    stats = json.loads(capsys.readouterr().out)
    assert stats == fuse_pipeline(c)[1].to_dict()


def test_bad_input_exit_code(tmp_path, capsys):
    bad = tmp_path / "bad.qasm"
    bad.write_text("OPENQASM 2.0;\nqreg q[2];\nx q[5];\n")
    assert main(["fuse", "--input", str(bad)]) == 2
    assert "line 3, column 3" in capsys.readouterr().err


@pytest.mark.gpu
def test_simulate_command_matches_reference(filter8_qasm, tmp_path):
    d, c, path = filter8_qasm
    seed = int(d["seeds"][0])
    out = tmp_path / "report.json"
    assert main(["simulate", "--input", str(path), "--shots", str(int(d["shots"])),
                 "--seed", str(seed), "--ancilla", str(c.n_qubits - 1),
                 "--output", str(out)]) == 0
    rep = json.loads(out.read_text())
    assert rep["assert_probs"] == pytest.approx(list(d[f"mma_{seed}_probs"]), abs=1e-12)
    k = int(d[f"mma_{seed}_n"])
    want = dict(zip(map(str, d[f"mma_{seed}_keys"][:k]), map(int, d[f"mma_{seed}_counts"][:k])))
    assert rep["samples"] == want
