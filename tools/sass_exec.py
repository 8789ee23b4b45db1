"""Executed-instruction mix of an ncu capture (source page, SASS): share of
warp instructions per opcode, and the hottest address ranges.
usage: python tools/sass_exec.py report.ncu-rep [top]"""
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
isrc, iex, iad = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Address")
by_op = defaultdict(float)
tot = 0.0
seq = []
for r in data:
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0]
    n = float(r[iex] or 0)
    by_op[op] += n
    tot += n
    seq.append((int(r[iad], 16) if r[iad].startswith("0x") else int(r[iad] or 0), op, n))
print(f"total warp instructions {tot:.4g}")
for op, n in sorted(by_op.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{op:24s} {100 * n / tot:6.2f} %")
