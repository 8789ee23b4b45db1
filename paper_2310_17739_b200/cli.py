"""Command line for the device path: the reference CLI's ``simulate`` and
``fuse`` subcommands (nucsim/cli.py:98-131) over this package.

    python -m paper_2310_17739_b200 simulate --input c.qasm [--mode mma|rejection]
        [--shots N] [--seed S] [--ancilla Q] [--no-fuse] [--output report.json]
    python -m paper_2310_17739_b200 fuse --input c.qasm

``simulate`` reads OpenQASM through the native reader, fuses natively
unless --no-fuse, runs on the GPU and writes the reference's RunReport JSON;
``fuse`` prints the FusionStats JSON.  Exit codes as the reference
(cli.py:37-40): 0 success, 2 parse or configuration error, 3 assertion
failure, 4 resource guard.  Hamiltonian tooling (prepare / spectrum /
filter-lcu, --hamiltonian) is outside the gate-application path.
"""

from __future__ import annotations

import argparse
import json
import sys

from .engine import infer_ancilla, run
from .errors import (FilterAssertionError, MmaStructureError, ProjectionError, QasmError,
                     ResourceLimitError)
from .fusion import fuse_pipeline
from .qasm import parse_qasm

_CONFIG_ERRORS = (QasmError, MmaStructureError, ValueError, OSError, KeyError)
_ASSERT_ERRORS = (FilterAssertionError, ProjectionError)
_RESOURCE_ERRORS = (ResourceLimitError, MemoryError)


def _read(path: str) -> str:
    with open(path, encoding="utf-8") as fh:
        return fh.read()


def _write(text: str, path: str | None) -> None:
    if path is None:
        sys.stdout.write(text)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)


def cmd_simulate(a: argparse.Namespace) -> int:
    if a.shots < 1:
        raise ValueError(f"shots must be >= 1, got {a.shots}")
    if not 0 <= a.seed < 2 ** 64:
        raise ValueError("seed must fit in 64 bits")
    circuit = parse_qasm(_read(a.input))
    fused, stats = circuit, None
    if not a.no_fuse:
        fused, fusion = fuse_pipeline(circuit)
        stats = fusion.to_dict()
    ancilla = a.ancilla
    if a.mode == "mma" and ancilla is None:
        ancilla = infer_ancilla(circuit)
        if ancilla is None:
            raise MmaStructureError(
                "cannot infer the ancilla from mid-circuit measures; give --ancilla")
    report = run(fused, a.mode, a.shots, a.seed, ancilla, fusion_stats=stats)
    _write(report.to_json() + "\n", a.output)
    return 0


def cmd_fuse(a: argparse.Namespace) -> int:
    _, stats = fuse_pipeline(parse_qasm(_read(a.input)))
    print(json.dumps(stats.to_dict(), indent=2))
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2310_17739_b200")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("simulate", help="QASM in, fusion unless --no-fuse, run, JSON report out")
    p.add_argument("--input", required=True, help="OpenQASM 2.0 circuit file")
    p.add_argument("--mode", choices=("mma", "rejection"), default="mma")
    p.add_argument("--shots", type=int, default=1024)
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--ancilla", type=int, default=None)
    p.add_argument("--no-fuse", action="store_true", dest="no_fuse")
    p.add_argument("--threads", type=int, default=1, help="accepted; no effect (as the reference)")
    p.add_argument("--output", default=None, help="write the report here instead of stdout")
    p.set_defaults(func=cmd_simulate)
    p = sub.add_parser("fuse", help="QASM in, fusion statistics out")
    p.add_argument("--input", required=True)
    p.set_defaults(func=cmd_fuse)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except _ASSERT_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3
    except _RESOURCE_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except _CONFIG_ERRORS as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
