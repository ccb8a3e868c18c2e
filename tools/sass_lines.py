#!/usr/bin/env python
"""Per-CUDA-source-line attribution of one captured kernel (ncu source page,
cuda,sass view; needs -lineinfo and --import-source on): thread instructions
executed per unit, the opcode mix and the warp-stall samples of each line.

Usage: sass_lines.py REPORT.ncu-rep UNITS [TOP]
(UNITS: divide executed thread-instructions by this, e.g. attempted steps.)"""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
lines = collections.defaultdict(lambda: [0, 0, collections.Counter(), ""])
path, cur = "?", None
hdr = None
for row in csv.reader(io.StringIO(raw)):
    if not row:
        continue
    if row[0] == "File Path":
        path = row[1].rsplit("/", 1)[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        iT = hdr.index("Thread Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or row[0] == "Function Name":
        continue
    if row[0]:                                    # a CUDA source line (aggregate)
        cur = (path, int(row[0]))
        lines[cur][3] = row[1].strip()[:90]
        continue
    if cur is None or len(row) <= iT or row[2] in ("...", "-"):
        continue
    try:
        n = int(row[iT])
        smp = int(row[iS]) if row[iS] not in ("-", "") else 0
    except ValueError:
        continue
    toks = row[3].strip().split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    e = lines[cur]
    e[0] += n
    e[1] += smp
    e[2][op] += n
tot = sum(e[0] for e in lines.values())
stot = sum(e[1] for e in lines.values()) or 1
print(f"thread instructions per unit: {tot / units:.1f}")
for (f, ln), (n, smp, ops, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
    mix = " ".join(f"{o}:{c / units:.1f}" for o, c in ops.most_common(5))
    print(f"{n / units:7.1f}  stall {smp / stot * 100:4.1f}%  {f}:{ln:<5d} {mix:60s} | {src}")
