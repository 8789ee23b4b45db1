"""TMA tile debugging: amplitude i = i + 0j, a pass of diagonal +-1 gates, so
|out[i]| names the input amplitude that landed at i.  Prints mismatches."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17739_b200 import Circuit, Gate  # noqa: E402
from paper_2310_17739_b200._pack import pack  # noqa: E402
from paper_2310_17739_b200.engine import DeviceProgram, StateVector  # noqa: E402

os.environ["NSB_LOW_QUBITS"] = "3"


def case(n, gates, tma, debug="0"):
    os.environ["NSB_TMA"] = tma
    c = Circuit(n, [("c", 1)])
    for g, qs in gates:
        c.gate_op(g, qs, ())
    pk = pack(c)
    a = np.arange(1 << n, dtype=np.float64).astype(np.complex128)
    st = StateVector(n)
    st.amps = a
    prog = DeviceProgram(st, pk.ops, pk.params, pk.payloads)
    prog.run_mma()
    out = st.amps
    want = a.copy()
    idx = np.arange(1 << n)
    for g, qs in (gates if not (int(debug) & 3) else []):
        if g == Gate.Z:
            want[((idx >> qs[0]) & 1) == 1] *= -1
        elif g == Gate.CZ:
            want[(((idx >> qs[0]) & 1) & ((idx >> qs[1]) & 1)) == 1] *= -1
    bad = np.nonzero(out != want)[0]
    if len(bad):
        freq = [int(np.count_nonzero((bad >> b) & 1)) for b in range(n)]
        print("   bit frequency among wrong:", freq)
    print(f"n={n} TMA={tma} debug={debug} passes={prog.info.n_passes} gates={gates}: {len(bad)} wrong of {1 << n}")
    for i in bad[:3]:
        src = int(round(abs(out[i])))
        print(f"   at {i:0{n}b} got |{src:0{n}b}| ({out[i]:.0f}) want {want[i]:.0f}")
    return len(bad)


TMA = sys.argv[1] if len(sys.argv) > 1 else "1"
DEBUG = os.environ.get("NSB_DEBUG_BLOCKED", "0")
for rep in range(2):
    case(20, [(Gate.CZ, (4, 6)), (Gate.CZ, (8, 10)), (Gate.CZ, (12, 14)), (Gate.CZ, (16, 18))], TMA, DEBUG)
    case(20, [(Gate.CZ, (4, 6)), (Gate.CZ, (8, 10)), (Gate.CZ, (12, 14))], TMA, DEBUG)
    case(20, [(Gate.CZ, (3, 4)), (Gate.CZ, (6, 7)), (Gate.CZ, (9, 10)), (Gate.CZ, (12, 13))], TMA, DEBUG)
    case(20, [(Gate.CZ, (6, 7)), (Gate.CZ, (8, 9)), (Gate.CZ, (13, 14)), (Gate.CZ, (17, 18))], TMA, DEBUG)
    case(20, [(Gate.CZ, (5, 6)), (Gate.CZ, (7, 8)), (Gate.CZ, (12, 13)), (Gate.CZ, (15, 16))], TMA, DEBUG)
    case(20, [(Gate.CZ, (9, 10)), (Gate.CZ, (11, 12)), (Gate.CZ, (13, 14)), (Gate.CZ, (17, 18))], TMA, DEBUG)
