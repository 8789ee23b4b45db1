"""Host planner timing on the deep21 workload (serial vs threaded)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17739_b200 import workloads as W  # noqa: E402

wl = W.filter_workload(20, trotter=18, n_steps=8, n_scatter=8, trial="10" * 10)
fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
exe = wl.executable(fops)
print("cpus", os.cpu_count(), "sched", len(os.sched_getaffinity(0)))
for serial in (False, True):
    if serial:
        os.environ["NSB_PLAN_SERIAL"] = "1"
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        a = W.plan_analyze(exe, wl.params, pool, wl.n_qubits)
        ts.append(time.perf_counter() - t)
    print("serial" if serial else "threaded", round(min(ts), 3), a["n_passes"], a["n_device_gates"])
