"""Summarise ncu outputs for profiles/: launch list shares and the key
metrics of one --set full capture.  Usage:
    python tools/ncu_summary.py launches gpurun_out/launches.csv
    python tools/ncu_summary.py full gpurun_out/prof_full.ncu-rep
    python tools/ncu_summary.py dram gpurun_out  > profiles/r01_dram_bytes.json
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
         "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= iv:
            continue
        name = r[ik].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | device ms (ncu, serialised) | share |")
    print("|---|---|---|---|")
    for k, (c, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| `{k}` | {c} | {ms:.3f} | {100 * ms / tot:.2f} % |")


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2 sector throughput %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "shared bank conflicts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed",
     "shared pipe busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    print("| metric | value |")
    print("|---|---|")
    for k, label in KEYS:
        if k in d:
            v, u = d[k]
            print(f"| {label} (`{k}`) | {v} {u} |")
    stalls = []
    for h, (v, _) in d.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
            try:
                stalls.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    tot = sum(s for s, _ in stalls) or 1.0
    print()
    print("| stall reason (pc sampling) | share |")
    print("|---|---|")
    for s, h in sorted(stalls, reverse=True)[:8]:
        print(f"| {h} | {100 * s / tot:.1f} % |")


def dram(folder):
    """JSON {config: DRAM bytes (read + write) of one k_blocked launch}."""
    import json
    import pathlib
    out = {}
    for f in sorted(pathlib.Path(folder).glob("dram_*.csv")):
        rows = list(csv.reader(open(f)))
        try:
            start = next(i for i, r in enumerate(rows) if "Metric Name" in r)
        except StopIteration:
            continue
        hdr = rows[start]
        iname, ival, iunit = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        tot = 0.0
        for r in rows[start + 1:]:
            if len(r) > ival and r[iname].startswith("dram__bytes"):
                tot += float(r[ival].replace(",", "")) * scale.get(r[iunit], 1)
        out[f.stem[len("dram_"):]] = int(tot)
    print(json.dumps(out))


if __name__ == "__main__":
    {"launches": launches, "full": full, "dram": dram}[sys.argv[1]](sys.argv[2])
