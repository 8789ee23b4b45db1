"""Thread layout vs state size: MMA run time of a filter circuit at n qubits with
one or two octets per thread (NSB_PLAN_OCTETS; run once per setting)."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2310_17739_b200 import workloads as W  # noqa: E402
from paper_2310_17739_b200.engine import DeviceProgram, StateVector  # noqa: E402
from paper_2310_17739_b200 import _native as N  # noqa: E402
import ctypes  # noqa: E402

for n in [int(x) for x in sys.argv[1:]] or [14, 16, 17, 18, 19, 20, 21]:
    wl = W.filter_workload(n - 1, trotter=2, n_steps=4, n_scatter=4, trial="10" * ((n - 1) // 2) + "1" * ((n - 1) % 2))
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    st = StateVector(n)
    prog = DeviceProgram(st, exe, wl.params, pool)
    ms = []
    for rep in range(4):
        st.restart()
        st.device_call("nsb_timer_start")
        prog.run_mma()
        m = ctypes.c_double()
        st.device_call("nsb_timer_stop", ctypes.byref(m))
        ms.append(m.value)
    print(f"n={n} octets={os.environ.get('NSB_PLAN_OCTETS', 'auto')} gates={wl.input_gates} "
          f"passes={prog.info.n_passes} ms={min(ms[1:]):.3f}", flush=True)
