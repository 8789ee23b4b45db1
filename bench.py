"""Benchmark: input gates/s of the 21-qubit deep projection-filter circuit
(BASELINE.json `metric`, config 3, paper P9 shape) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config deep21|rand28] [--trotter R]

One step = one MMA-mode execution of the whole fused circuit from |0...0>
(every gate, all 8 mid-circuit assertions with collapse) plus the final
probability read-out used for sampling.  The workload is generated and fused
natively before timing (host time reported separately in `host`).

value  device-resident: the fused plan is already in HBM; timed with CUDA
       events around each cooperative kernel launch (library stream), K steps
       after W warm-ups; L2 flushed (256 MiB write) between steps because the
       21-qubit state (32 MiB) would otherwise stay L2-resident across steps.
e2e    through the C ABI with host buffers: per step the packed fused op list
       (host) is planned + uploaded + executed (nsb_run_mma_streamed: part s+1
       planned while part s runs), and the probabilities are read back (D2H)
       and sampled on the host -- what `run()` does per call.
cpu_baseline / --impl reference: the oracle port of the reference engine
       (numpy einsum, as nucsim.engine) on a bounded prefix of the same fused
       gate stream, single-threaded, extrapolated per gate.  The reference
       arm never imports the product: deep21's fused stream is the prefix
       the unmodified reference produced (tests/golden/deep21.npz).

Multi-GPU (torchrun, N > 1), default configs: replicas -- every rank runs
the same circuit on its own GPU (no data-path collective), value = total
gates / max time over ranks, "scaling": "weak".  Every default line also
carries "sharded": the multi-GPU design measured at this N -- ONE 32-qubit
layered circuit split over all N GPUs (strong scaling; 64 GiB state, fits one
GPU at N = 1) and, from N = 2, the 34-qubit config 5 state (256 GiB).

--config shard [--qubits Q] (BASELINE config 5, default Q = 34): ONE layered
random circuit whose state is split over the N ranks (sharded.py: 2^(Q-g)
amplitudes per GPU, NCCL qubit swaps over NVLink, "scaling": "strong").
value = input gates / max-over-ranks device time of one full execution.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

METRIC = "gates/sec on 21-qubit deep circuit; achieved GB/s vs roofline at 1/2/4/8 GPUs"
UNIT = "input gates/s"
FP64_DFMA_PER_CLK_PER_SM = 64  # B200: 64 FP64 FMA lanes per SM per clock (spec)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965)),
                "source": "measured"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}


def l2_copy_gbs(state_bytes: int, reps: int = 200) -> float | None:
    """Measured L2-resident copy bandwidth (read + write bytes per second) for
    a buffer of the state's size: the roof for a state that stays in the
    126 MB L2 inside a launch.  None if the source and
    destination together would not fit in half the L2."""
    import torch
    if 2 * state_bytes > 64 << 20:
        return None
    a = torch.ones(state_bytes // 8, dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    for _ in range(20):
        b.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    torch.cuda.synchronize()
    return 2 * state_bytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def make_workload(config: str, trotter: int | None):
    from paper_2310_17739_b200 import workloads as W
    t0 = time.perf_counter()
    if config == "deep21":
        r = trotter or 18
        wl = W.filter_workload(20, trotter=r, n_steps=8, n_scatter=8, trial="10" * 10)
    elif config == "rand28":
        wl = W.layered_workload(28, layers=trotter or 20)
    elif config in SMALL:
        d = small_fixture(config)
        terms = [("".join("IXYZ"[c] for c in row), float(cf))
                 for row, cf in zip(d["term_letters"], d["term_coeffs"])]
        wl = W.filter_workload(d["term_letters"].shape[1], int(d["trotter"]), terms=terms,
                               steps=[tuple(map(float, x)) for x in d["steps"]],
                               trial="".join(str(int(b)) for b in d["trial"]))
    else:
        raise SystemExit(f"unknown config {config}")
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    fops, pool, stats = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    t_fuse = time.perf_counter() - t0
    exe = wl.executable(fops)
    return wl, exe, pool, stats, {"generate_s": round(t_gen, 3), "fuse_s": round(t_fuse, 3),
                                  "fuse_input_gates_per_s": round(wl.input_gates / t_fuse)}


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.proc = None
        self.path = Path(f"/tmp/nsb_clocks_{os.getpid()}.csv")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(name)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference arm (--impl reference) and cpu_baseline: the oracle port of the
# reference engine (oracle/nucsim_oracle.py, numpy einsum exactly as
# nucsim/engine.py:92-156) on a bounded prefix of the SAME fused stream.  This
# path never imports paper_2310_17739_b200: the deep21 fused stream comes from
# tests/golden/deep21.npz (the first 1 500 fused gates the unmodified reference
# itself produced, make_deep21_golden.py), rand28's from a pure-numpy restatement
# of workloads.layered_workload fused by the oracle's fuse_pipeline.


# BASELINE configs 1 and 2: the filter circuits the reference generated for the
# golden fixtures (tests/golden/make_golden.py): C1 `ucc8` = 7-mode shell
# model + ancilla, 10 554 gates; C2 `mcm16` = 15-site chain + ancilla,
# 39 676 gates, 4 mid-circuit assertions each
SMALL = {"ucc8": "filter8", "mcm16": "filter16"}


def small_fixture(config: str) -> dict:
    return dict(np.load(ROOT / "tests" / "golden" / f"{SMALL[config]}.npz"))


def host_cpu() -> dict:
    model = "unknown"
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def _oracle():
    sys.path.insert(0, str(ROOT / "oracle"))
    sys.path.insert(0, str(ROOT / "tests"))
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import nucsim_oracle as O
    return O


def reference_stream(config: str, trotter: int | None):
    """(oracle IR prefix of the fused stream, n_qubits, input gates, fused gates)
    of the bench workload, without the product package."""
    O = _oracle()
    if config == "deep21":
        if trotter not in (None, 18):
            raise SystemExit("the reference arm's deep21 sample is the Trotter-18 headline")
        from circuit_io import to_oracle
        d = dict(np.load(ROOT / "tests" / "golden" / "deep21.npz"))
        instrs, n = to_oracle(d, "prefix_")
        return instrs, n, int(d["fused_stats"][0]), int(d["fused_stats"][1])
    if config in SMALL:  # the reference's own fused list of the whole circuit
        from circuit_io import to_oracle
        d = small_fixture(config)
        instrs, n = to_oracle(d, "fused_")
        return instrs, n, int(d["fused_stats"][0]), int(d["fused_stats"][1])
    if config == "rand28":  # workloads.layered_workload(28, layers, seed 28), restated
        import math
        n, layers = 28, trotter or 20
        rng = np.random.default_rng(28)
        instrs = []
        for _ in range(layers):
            for q in range(n):
                instrs.append(("u3", (q,), tuple(float(x) for x in rng.uniform(-math.pi, math.pi, 3)),
                               None, None))
            perm = rng.permutation(n)
            for k in range(0, n - 1, 2):
                a, b = int(perm[k]), int(perm[k + 1])
                g = ("cx", "cz", "rzz")[int(rng.integers(3))]
                ps = (float(rng.uniform(-math.pi, math.pi)),) if g == "rzz" else ()
                instrs.append((g, (a, b), ps, None, None))
        fused = O.fuse_pipeline(instrs)[0]
        return fused, n, len(instrs), O.gate_count(fused)
    raise SystemExit(f"unknown config {config}")


def cpu_sample(instrs, n, input_per_fused, budget_s):
    """Oracle port on the fused stream from |0...0>, fused gates applied in
    order until `budget_s` seconds have passed; input gates/s extrapolated."""
    O = _oracle()
    a = np.zeros(1 << n, np.complex128)
    a[0] = 1.0
    done = 0
    t0 = time.perf_counter()
    for ins in instrs:
        name, qs = ins[0], tuple(ins[1])
        if name in ("barrier", "reset"):
            continue
        if name == "measure":
            p0 = O.branch_probability(a, qs[0], 0)
            O.project(a, qs[0], 0, p0)
            continue
        a = O.apply_dense(a, O.resolved(ins), qs)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done, dt, done * input_per_fused / dt


def cpu_baseline(args, budget_s: float) -> dict:
    instrs, n, n_in, n_fused = reference_stream(args.config, args.trotter)
    ratio = n_in / max(n_fused, 1)
    done, dt, value = cpu_sample(instrs, n, ratio, budget_s)
    return {"value": round(value, 3), "unit": UNIT, "cores": 1, "kind": "port", **host_cpu(),
            "sample": f"first {done} fused gates of the same fused stream at {n} qubits "
                      f"({dt:.1f} s; oracle port of nucsim.engine, numpy einsum, one thread: "
                      f"the reference's gate kernels are single-threaded), scaled by the "
                      f"input/fused gate ratio {ratio:.3f}"}


def run_reference(args, rank):
    """--impl reference: rank 0 times the oracle port on bounded samples
    (each step = fused gates from |0...0> for --ref-step-s seconds)."""
    if rank != 0:
        return
    instrs, n, n_in, n_fused = reference_stream(args.config, args.trotter)
    ratio = n_in / max(n_fused, 1)
    for _ in range(args.warmup):
        cpu_sample(instrs, n, ratio, 0.2)
    gates = secs = 0.0
    for _ in range(args.steps):
        done, dt, _ = cpu_sample(instrs, n, ratio, args.ref_step_s)
        gates += done
        secs += dt
    value = gates * ratio / secs
    line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(secs * 1e3 / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic", "impl": "reference",
            "config": workload_config(args, n, n_in, n_fused, args.gpus),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": 1, "kind": "port",
                             **host_cpu(),
                             "sample": f"{args.steps} steps x {args.ref_step_s:.1f} s: "
                                       f"{int(gates)} fused gates of the same fused stream "
                                       f"from |0...0> at {n} qubits (oracle port of "
                                       f"nucsim.engine, numpy einsum, one thread), scaled by "
                                       f"the input/fused ratio {ratio:.3f}"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(args, n, input_gates, fused_gates, world) -> dict:
    """The `config` both arms print (workload identity only)."""
    c = {"workload": workload_name(args), "n_qubits": n, "input_gates": input_gates,
         "fused_gates": fused_gates, "parallelism": f"replicas{world}",
         "l2": "flushed between steps (256 MiB write); state (2^n x 16 B) L2-resident "
               "within a step when it fits"}
    if args.config == "deep21":
        c.update({"trotter": args.trotter or 18, "filter_steps": 8})
    elif args.config in SMALL:
        d = small_fixture(args.config)
        c.update({"trotter": int(d["trotter"]), "filter_steps": int(len(d["steps"]))})
    else:
        c.update({"layers": args.trotter or 20})
    return c


def workload_name(args) -> str:
    if args.config == "ucc8":
        return ("ucc8 (BASELINE config 1): 7-mode shell-model projection filter + ancilla "
                "(8 qubits), 4 filter steps, MMA mode")
    if args.config == "mcm16":
        return ("mcm16 (BASELINE config 2): 15-site transverse-field chain projection filter + "
                "ancilla (16 qubits), 4 mid-circuit assertions, MMA mode")
    if args.config == "deep21":
        return (f"deep21: 20-mode JW shell-model projection filter + ancilla (21 qubits), "
                f"8 filter steps x {args.trotter or 18} Trotter slices (paper P9 shape), MMA mode")
    return f"rand28: 28-qubit random layered U3 + {{CX,CZ,RZZ}} circuit, {args.trotter or 20} layers"


def sharded_measure(n: int, layers: int, rank: int, world: int, local: int, steps: int,
                    warmup: int, extras: bool = False) -> dict:
    """ONE n-qubit layered circuit (BASELINE config 4/5 generator) whose state is
    split over all `world` ranks (sharded.py: 2^(n-g) amplitudes per GPU, qubit
    swaps through peer memory over NVLink, collective assertions).  Device time
    per full execution, max over ranks.  Collective: every rank calls it."""
    import torch.distributed as dist
    from paper_2310_17739_b200 import workloads as W
    from paper_2310_17739_b200.sharded import ShardedState

    t0 = time.perf_counter()
    wl = W.layered_workload(n, layers=layers, seed=34)
    fops, pool, stats = W.fuse_packed(wl.ops, wl.params, wl.payloads)
    host = {"generate_fuse_s": round(time.perf_counter() - t0, 3)}
    if world > 1:
        st = ShardedState.from_torch_distributed(n, device=local)
    else:
        st = ShardedState(n, 0, 1, local, ShardedState.unique_id())
    t0 = time.perf_counter()
    prog = st.compile(fops, wl.params, pool)
    host["schedule_plan_s"] = round(time.perf_counter() - t0, 3)
    tot = prog.plan_totals()

    def barrier():
        if world > 1:
            dist.barrier()

    def one():
        st.reset()
        barrier()
        st.timer_start()
        prog.run()
        return st.timer_stop()

    for _ in range(warmup):
        one()
    barrier()
    ms = [one() for _ in range(steps)]
    dev_s = sum(ms) / 1e3
    if world > 1:
        box = [None] * world
        dist.all_gather_object(box, dev_s)
        dev_s = max(box)
    # profiled executions (per-step device events; outside the timed region):
    # swaps on their own (NSB_SWAP_OVERLAP=0), then overlapped with the gate
    # item after them as the timed runs do (the default: copy engines) -- the
    # swap cost the overlap hides
    def profiled(overlap: str) -> dict:
        prev = os.environ.get("NSB_SWAP_OVERLAP")
        os.environ["NSB_SWAP_OVERLAP"] = overlap
        try:
            st.reset()
            barrier()
            t: dict = {}
            prog.run(times=t)
            return t
        finally:
            if prev is None:
                os.environ.pop("NSB_SWAP_OVERLAP", None)
            else:
                os.environ["NSB_SWAP_OVERLAP"] = prev

    ov_mode = os.environ.get("NSB_SWAP_OVERLAP", "ce")
    seq = profiled("0")
    times = profiled(ov_mode) if st.peer_swaps and ov_mode != "0" else seq
    overlapped_passes = prog.overlapped_passes
    nl = st.nl
    pk = peaks()
    gate_bytes = tot["n_passes"] * 32 * (1 << nl)
    swap_bytes = prog.n_swaps * 16 * (1 << (nl - 1))  # sent (= received) per rank
    gate_s = seq.get("gates", 0.0) / 1e3
    swap_s = seq.get("swap", 0.0) / 1e3
    seq_ms, ov_ms = sum(seq.values()), sum(times.values())
    achieved = gate_bytes / gate_s / 1e9 if gate_s else 0.0
    out = {"workload": f"shard{n}: {n}-qubit random layered U3 + {{CX,CZ,RZZ}} circuit, "
                       f"{layers} layers, state split over {world} GPU(s)",
           "n_qubits": n, "local_qubits": nl, "input_gates": wl.input_gates,
           "fused_gates": stats["gates_after"],
           "value": round(wl.input_gates * steps / dev_s, 1), "unit": UNIT,
           "ms_per_run": round(dev_s * 1e3 / steps, 3), "steps": steps, "warmup": warmup,
           "scaling": "strong", "n_gpus": world, "qubit_swaps": prog.n_swaps,
           "qubit_swap_path": ({"ce": "copy engines over NVLink, overlapped with the next gate "
                                      "item (nsb_shard_swap_overlap_ce)",
                                "1": "peer-memory swap kernel overlapped with the next gate item "
                                     "(nsb_shard_swap_overlap)",
                                "0": "peer-memory swap kernel (nsb_shard_swap_p2p)"}.get(ov_mode)
                               if st.peer_swaps else "pack + NCCL send/recv + unpack"),
           "passes_per_rank": tot["n_passes"], "device_gate_ops": tot["n_device_gates"],
           "breakdown_ms": {k: round(v, 3) for k, v in seq.items()},
           "swap_overlap": {
               "mode": ov_mode,
               "breakdown_ms": {k: round(v, 3) for k, v in times.items()},
               "overlapped_passes": overlapped_passes,
               "run_ms_overlapped": round(ov_ms, 3), "run_ms_sequential": round(seq_ms, 3),
               "swap_ms_sequential": round(seq.get("swap", 0.0), 3),
               "hidden_frac": round((seq_ms - ov_ms) / seq["swap"], 4) if seq.get("swap") else None,
               "note": "the gate item after a swap runs its chunkable passes chunk by chunk "
                       "as the swapped chunks land (mode ce: 2-D peer copies into a staging "
                       "slot + local copies on the copy engines, flag words by stream memory "
                       "operations, no SMs taken); hidden_frac = (sequential - overlapped run) "
                       "/ sequential swap time, one profiled run each; the timed value runs "
                       "in this mode"},
           "gate_groups_hbm": {"achieved_gbs": round(achieved, 1), "peak": pk["hbm_gbs"],
                               "frac": round(achieved / pk["hbm_gbs"], 4)},
           "nvlink": {"bytes_sent_per_rank": swap_bytes,
                      "achieved_gbs": round(swap_bytes / swap_s / 1e9, 1) if swap_s else None},
           "host": host}
    if extras:
        t0 = time.perf_counter()
        st.reset()
        p2 = st.compile(fops, wl.params, pool)
        p2.run()
        out["norm"] = st.norm()
        e2e_s = time.perf_counter() - t0
        p2.close()
        out["e2e"] = {"value": round(wl.input_gates / e2e_s, 1), "unit": UNIT,
                      "h2d_bytes_per_step": int(fops.nbytes + wl.params.nbytes + pool.nbytes),
                      "d2h_bytes_per_step": 8, "s_per_step": round(e2e_s, 4),
                      "note": "schedule + plan upload from host op arrays + run + norm read-back"}
        barrier()
        t0 = time.perf_counter()
        smp = st.sample(1024, 2310)  # collective sampling of the full 2^n state (sharded.py)
        out["sampling"] = {"shots": 1024, "s": round(time.perf_counter() - t0, 4),
                           "distinct": len(smp)}
    prog.close()
    st.close()
    return out


def run_sharded(args, rank, world, local):
    """BASELINE config 5: one state split over all ranks (sharded.py)."""
    import torch
    import torch.distributed as dist

    if world > 1:
        dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    clocks = Clocks(local)
    m = sharded_measure(args.qubits, args.trotter or 10, rank, world, local, args.steps,
                        args.warmup, extras=True)
    clk = clocks.stop()
    line = {"metric": METRIC, "value": m["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["ms_per_run"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": m["workload"], "n_qubits": m["n_qubits"],
                       "input_gates": m["input_gates"], "fused_gates": m["fused_gates"],
                       "parallelism": f"shard{world}",
                       "l2": f"state shard 2^{m['local_qubits']} x 16 B >> L2; no flush needed"},
            "sharded": m,
            "roofline": {"bound": "hbm", "achieved": m["gate_groups_hbm"]["achieved_gbs"],
                         "peak": m["gate_groups_hbm"]["peak"], "unit": "GB/s",
                         "frac": m["gate_groups_hbm"]["frac"], "traffic": None,
                         "note": "k_blocked only: passes x 32 B x 2^local per rank over the "
                                 "summed gate-group device time of one profiled execution"},
            "e2e": m["e2e"], "gpu_launches": None, "clocks": clk,
            "cpu_baseline": {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                             "sample": f"infeasible: the reference holds 2 x 2^{args.qubits} "
                                       "x 16 B on one host (engine.py:51, 68-71)"}}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_ours(args, rank, world, local):
    import ctypes
    import torch
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    os.environ["NUCSIM_DEVICE"] = str(local)
    from paper_2310_17739_b200 import _native as N
    from paper_2310_17739_b200.engine import (DeviceProgram, StateVector, _sample_from,
                                              _streamable, run_mma_streamed)

    wl, exe, pool, stats, host = make_workload(args.config, args.trotter)
    n = wl.n_qubits
    state = StateVector(n)
    t0 = time.perf_counter()
    prog = DeviceProgram(state, exe, wl.params, pool)
    host["plan_s"] = round(time.perf_counter() - t0, 3)
    info = prog.info
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        state.restart()
        prog.run_mma()
        return prog.last_timing()

    for _ in range(args.warmup):
        flush.zero_()
        torch.cuda.synchronize()
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    ms_list, launches = [], 0
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ms, nl = step()
        ms_list.append(ms)
        launches += nl + 1  # + the |0...0> reset kernel
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    dev_s = sum(ms_list) / 1e3
    if world > 1:
        t = torch.tensor([dev_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        dev_s = float(t.item())
    total_gates = wl.input_gates * args.steps * world
    value = total_gates / dev_s
    ms_per_step = dev_s * 1e3 / args.steps

    # e2e: the C-ABI path with host buffers, one full call per step
    probs = np.empty(1 << n, np.float64)
    e2e_times = []
    rng = np.random.Generator(np.random.Philox(7))
    for _ in range(max(1, args.e2e_steps)):
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        state.restart()
        if _streamable(exe, n):  # run()'s MMA path: planning streamed behind execution
            run_mma_streamed(state, exe, wl.params, pool)
        else:
            p2 = DeviceProgram(state, exe, wl.params, pool)
            p2.run_mma()
            del p2  # the program is released inside the call, as run() does
        state.device_call("nsb_probabilities", N.ptr(probs))
        _sample_from(probs, n, 1024, rng)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_times))
    if world > 1:  # whole job: every rank's call, slowest rank's time
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = (exe.nbytes + wl.params.nbytes + pool.nbytes) * world
    d2h = (probs.nbytes + 8 * info.n_measures) * world

    # roofline of the dominant kernel (k_blocked): algorithmic bytes =
    # passes x (read + write) x 16 B x 2^n per launch
    pk = peaks()
    bytes_per_launch = info.n_passes * 2 * 16 * (1 << n)
    kernel_s = dev_s / args.steps if world == 1 else sum(ms_list) / 1e3 / args.steps
    achieved = bytes_per_launch / kernel_s / 1e9
    sm_mhz = clk.get("sm_mhz") or pk["sm_max_mhz"]
    fp64_peak = 148 * FP64_DFMA_PER_CLK_PER_SM * 2 * sm_mhz * 1e6 / 1e12
    fp64_ach = info.flops / kernel_s / 1e12
    smem_peak = 148 * 128 * sm_mhz * 1e6 / 1e12
    smem_ach = info.n_sweeps * 32 * (1 << n) / kernel_s / 1e12
    l2_gbs = l2_copy_gbs(16 << n)
    profile = ROOT / "profiles" / "r02_dram_bytes.json"
    traffic = None
    if profile.exists():
        traffic = json.loads(profile.read_text()).get(args.config)
    line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": workload_config(args, n, wl.input_gates, stats["gates_after"], world),
            "plan": {"fusion_reduction": round(wl.input_gates / max(stats["gates_after"], 1), 3),
                     "passes": info.n_passes,
                     "device_gate_ops": info.n_device_gates,
                     "octet_sweeps": info.n_sweeps,
                     "group_fused_ops": info.n_fused_group_ops,
                     "frame_absorbed_gates": info.n_frame_gates,
                     "frame_flush_gates": info.n_flush_gates,
                     "gates_per_pass": round(info.n_gates / max(info.n_passes, 1), 2),
                     "tile_qubits": info.tile_qubits,
                     **{k: v for k, v in wl.meta.items() if k != "terms"}},
            "host": host,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": round(achieved / pk["hbm_gbs"], 4),
                         "traffic": traffic, "peak_source": pk["source"],
                         "note": "algorithmic bytes = passes x 32 B x 2^n per launch; the "
                                 "21-qubit state is L2-resident inside a launch"},
            "l2": None if l2_gbs is None else {
                "achieved_gbs": round(achieved, 1), "copy_gbs_measured": round(l2_gbs, 1),
                "frac": round(achieved / l2_gbs, 4),
                "note": "same algorithmic bytes over the measured L2-resident copy bandwidth "
                        "(torch copy of a state-sized buffer, 200 reps): the state never "
                        "leaves L2 within a launch"},
            "smem": {"achieved_tbs": round(smem_ach, 2), "peak_tbs": round(smem_peak, 2),
                     "frac": round(smem_ach / smem_peak, 4),
                     "note": "octet sweeps x 32 B x 2^n (each sweep reads and writes the "
                             "state in shared memory) over kernel time; peak = 148 SMs x "
                             "128 B/clk at the sampled SM clock"},
            "fp64": {"achieved_tflops": round(fp64_ach, 3), "peak_tflops": round(fp64_peak, 2),
                     "frac": round(fp64_ach / fp64_peak, 4),
                     "flops_per_launch": info.flops},
            "e2e": {"value": round(wl.input_gates * world / e2e_s, 1), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "s_per_step": round(e2e_s, 4)},
            "wall_s": round(wall, 3), "gpu_launches": launches, "clocks": clk}
    if not args.no_sharded and args.config == "deep21":
        # the multi-GPU design itself (the replicas above need no exchange):
        # strong scaling of one 32-qubit state split over all N GPUs, and the
        # 34-qubit config 5 state from N = 2 on
        del prog, state
        torch.cuda.empty_cache()
        sh = []
        try:  # a failure here must not cost the headline line (same on every rank)
            sh.append(sharded_measure(32, 10, rank, world, local, 2, 1))
            if world >= 2:
                sh.append(sharded_measure(34, 10, rank, world, local, 1, 1))
        except Exception as e:  # noqa: BLE001 -- reported in the JSON line
            sh.append({"error": f"{type(e).__name__}: {e}"[:300]})
        line["sharded"] = sh
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, args.ref_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="deep21",
                    choices=("deep21", "rand28", "ucc8", "mcm16", "shard"))
    ap.add_argument("--qubits", type=int, default=34, help="--config shard: total qubits")
    ap.add_argument("--trotter", type=int, default=None)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-budget", type=float, default=12.0,
                    help="cpu_baseline sample length (s)")
    ap.add_argument("--ref-step-s", type=float, default=1.5,
                    help="--impl reference: seconds of oracle work per timed step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sharded", action="store_true",
                    help="skip the sharded strong-scaling sub-measurement (shard32 / shard34)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        if args.config == "shard":
            if rank == 0:
                print(json.dumps({"impl": "reference", "metric": METRIC, "value": None,
                                  "unit": UNIT, "unavailable": f"the reference keeps 2 x 2^"
                                  f"{args.qubits} x 16 B in one host process"}), flush=True)
            return
        run_reference(args, rank)
        return
    if args.config == "shard":
        run_sharded(args, rank, world, local)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
