"""Microbenchmark: device time of the blocked kernel vs gates per pass.

Builds packed op lists directly (no fusion) for n qubits:
  chain: 2q dense-ish gates walking the register (forces many passes)
  local: 2q gates confined to qubits 0..5 (one pass per 64 gates)
and reports ms, passes, device gates, us/pass, us/gate.
"""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2310_17739_b200 import _native as N, Gate
from paper_2310_17739_b200.engine import DeviceProgram, StateVector


def ops_for(pairs, tag=Gate.CU3, params=(0.3, 0.2, 0.1)):
    ops = np.zeros(len(pairs), dtype=N.OP_DTYPE)
    for i, (a, b) in enumerate(pairs):
        ops[i]["kind"], ops[i]["tag"], ops[i]["nq"] = N.OP_GATE, tag.code, 2
        ops[i]["q"] = (a, b, -1, -1, -1)
        ops[i]["mask"] = (1 << a) | (1 << b)
        ops[i]["param"] = 0
    ops["cbit"], ops["src"], ops["payload"] = -1, -1, -1
    return ops, np.asarray(params, np.float64)


def measure(n, pairs, reps=3):
    ops, params = ops_for(pairs)
    s = StateVector(n)
    prog = DeviceProgram(s, ops, params, np.zeros(1, np.complex128))
    prog.run_mma()
    ts = []
    for _ in range(reps):
        prog.run_mma()
        ts.append(prog.last_timing()[0])
    ms = min(ts)
    info = prog.info
    return ms, info.n_passes, info.n_device_gates


if __name__ != "__main__":
    pass
else:
  n = int(sys.argv[1]) if len(sys.argv) > 1 else 21
  for label, pairs in [
    ("local x640", [(i % 5, i % 5 + 1) for i in range(640)]),
    ("local x6400", [(i % 5, i % 5 + 1) for i in range(6400)]),
    ("chain x640", [(i % (n - 1), i % (n - 1) + 1) for i in range(640)]),
    ("chain x6400", [(i % (n - 1), i % (n - 1) + 1) for i in range(6400)]),
    ("far x640", [(0, n - 1 - (i % 9)) for i in range(640)]),
]:
    ms, passes, gates = measure(n, pairs)
    print(f"{label:14s} n={n} {ms:9.3f} ms  passes={passes:6d} gates={gates:6d} "
          f"us/pass={1e3 * ms / passes:8.2f} us/gate={1e3 * ms / gates:7.3f}", flush=True)
