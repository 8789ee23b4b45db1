"""compute-sanitizer driver for k_blocked (race / memory checks).

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_blocked.py

Small blocked programs in both tile policies (L2: qubits 0,1 tiled; HBM:
qubits 0..2 tiled, forced with NSB_LOW_QUBITS=3), several tile sizes,
with mid-circuit assertions (epilogue / prologue collapse), the frame, read
maps, warp-local sweeps and group fusion all exercised."""

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2310_17739_b200 import workloads as W  # noqa: E402
from paper_2310_17739_b200.engine import DeviceProgram, StateVector  # noqa: E402

cases = [(12, "2", "11"), (13, "3", "11"), (14, "3", "9"), (16, "2", "11"), (16, "3", "10")]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for n, low, tile in cases:
    os.environ["NSB_LOW_QUBITS"] = low
    os.environ["NSB_TILE_QUBITS"] = tile
    wl = W.filter_workload(n - 1, trotter=1, n_steps=2, n_scatter=2, hop_range=4,
                           pair_density=0.2, trial="10" * ((n - 1) // 2) + "1" * ((n - 1) % 2))
    fops, pool, _ = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    exe = wl.executable(fops)
    state = StateVector(n)
    prog = DeviceProgram(state, exe, wl.params, pool)
    probs = prog.run_mma()
    print(f"n={n} low={low} tile={tile}: {prog.info.n_passes} passes, "
          f"{prog.info.n_sweeps} sweeps, p0 {np.round(probs, 6).tolist()}, "
          f"norm {state.norm():.12f}", flush=True)
