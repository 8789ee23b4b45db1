"""Split the bench's e2e step into its parts (plan+upload, run, read-back, sampling)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_2310_17739_b200 import _native as N  # noqa: E402
from paper_2310_17739_b200 import workloads as W  # noqa: E402
from paper_2310_17739_b200.engine import DeviceProgram, StateVector, _sample_from  # noqa: E402

wl = W.filter_workload(20, trotter=18, n_steps=8, n_scatter=8, trial="10" * 10)
fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
exe = wl.executable(fops)
state = StateVector(21)
probs = np.empty(1 << 21)
rng = np.random.Generator(np.random.Philox(7))
for it in range(3):
    t = [time.perf_counter()]
    state.restart()
    p = DeviceProgram(state, exe, wl.params, pool)
    t.append(time.perf_counter())
    p.run_mma()
    t.append(time.perf_counter())
    state.device_call("nsb_probabilities", N.ptr(probs))
    t.append(time.perf_counter())
    _sample_from(probs, 21, 1024, rng)
    t.append(time.perf_counter())
    del p
    t.append(time.perf_counter())
    print("plan+upload %.3f run %.3f probs %.3f sample %.3f free %.3f" %
          tuple(np.diff(t)), flush=True)
