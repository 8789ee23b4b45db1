"""Executed-instruction mix of one ncu capture (source page, SASS): warp
instructions executed per opcode, plus the TMA / bulk-copy opcodes in full.
Usage: python tools/sass_mix.py report.ncu-rep"""
import csv
import io
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source",
                      "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
name = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else "?"
hdr = rows[1]
isrc, iex = hdr.index("Source"), hdr.index("Instructions Executed")
mix, tma = Counter(), Counter()
for r in rows[2:]:
    src = r[isrc].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
    n = int(float(r[iex] or 0))
    mix[op] += n
    if op.startswith(("UTMA", "UBLKCP", "SYNCS", "UTMACMDFLUSH")):
        tma[re.sub(r"\s+", " ", src)[:70]] += n
tot = sum(mix.values())
print(f"kernel: `{name}`, {tot:,} warp instructions executed\n")
print("| opcode | warp instructions | share |\n|---|---|---|")
for op, n in mix.most_common(16):
    print(f"| {op} | {n:,} | {100 * n / tot:.2f} % |")
print("\nTMA / mbarrier instructions (SASS, executed):\n")
print("| instruction | executed |\n|---|---|")
for s, n in tma.most_common():
    print(f"| `{s}` | {n:,} |")
