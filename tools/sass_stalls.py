"""Aggregate per-instruction stall samples of an ncu source-page CSV (SASS)
by opcode: python tools/sass_stalls.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = defaultdict(lambda: defaultdict(float))
tot = 0.0
for r in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0]
    for h in reasons:
        v = float(r[hdr.index(h)] or 0)
        agg[op][h] += v
        tot += v
rank = sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))
print(f"{'opcode':22s} {'share':>6s}  top reasons")
for op, d in rank[:18]:
    s = sum(d.values())
    top = sorted(d.items(), key=lambda kv: -kv[1])[:4]
    print(f"{op:22s} {100 * s / tot:5.1f}%  " +
          ", ".join(f"{k[6:]} {100 * v / tot:.1f}" for k, v in top))
