"""Host fusion time, segment-parallel vs serial (NSB_FUSE_SERIAL), on the deep21
workload; checks that both produce the same fused ops and resolved payloads.
    python tools/fuse_time.py [trotter]"""
import hashlib
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17739_b200 import workloads as W  # noqa: E402


def resolved(fops, pool):
    h = hashlib.sha1()
    f2 = fops.copy()
    pay = f2["payload"].copy()
    f2["payload"] = 0
    h.update(f2.tobytes())
    for i in (pay >= 0).nonzero()[0]:
        dim = 1 << int(fops["nq"][i])
        h.update(pool[pay[i]:pay[i] + dim * dim].tobytes())
    return h.hexdigest()[:16]


trotter = int(sys.argv[1]) if len(sys.argv) > 1 else 18
wl = W.filter_workload(20, trotter=trotter, n_steps=8, n_scatter=8, trial="10" * 10)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "input ops", len(wl.ops))
for serial in (False, True):
    if serial:
        os.environ["NSB_FUSE_SERIAL"] = "1"
    t = time.perf_counter()
    fops, pool, st = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    dt = time.perf_counter() - t
    print("serial" if serial else "segment-parallel", round(dt, 3), "s", len(fops), "ops",
          st["per_pass"], resolved(fops, pool) if trotter <= 100 else "", flush=True)
    del fops, pool
