"""Where the e2e time of the headline call goes (streamed MMA run)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_2310_17739_b200 import _native as N  # noqa: E402
from paper_2310_17739_b200 import workloads as W  # noqa: E402
from paper_2310_17739_b200.engine import StateVector, _sample_from, run_mma_streamed  # noqa: E402

wl = W.filter_workload(20, trotter=18, n_steps=8, n_scatter=8, trial="10" * 10)
fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
exe = wl.executable(fops)
state = StateVector(21)
probs = np.empty(1 << 21)
rng = np.random.Generator(np.random.Philox(7))
for rep in range(4):
    t0 = time.perf_counter()
    state.restart()
    t1 = time.perf_counter()
    run_mma_streamed(state, exe, wl.params, pool)
    t2 = time.perf_counter()
    state.device_call("nsb_probabilities", N.ptr(probs))
    t3 = time.perf_counter()
    _sample_from(probs, 21, 1024, rng)
    t4 = time.perf_counter()
    print(f"restart {1e3*(t1-t0):.1f} ms, streamed run {1e3*(t2-t1):.1f} ms "
          f"(device {state.last_device_ms:.1f}), probabilities {1e3*(t3-t2):.1f}, "
          f"sampling {1e3*(t4-t3):.1f}, total {1e3*(t4-t0):.1f}", flush=True)
