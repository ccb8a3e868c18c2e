#!/usr/bin/env python
"""Instruction mix of one captured kernel from an ncu report (SASS source page).
Usage: sass_mix.py REPORT.ncu-rep UNITS [TOP]   (UNITS: divide executed thread-instructions by this,
e.g. trajectories × steps, to print instructions per unit)."""
import collections
import csv
import io
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
iS, iT = hdr.index("Source"), hdr.index("Thread Instructions Executed")
by, tot = collections.Counter(), 0
for r in rows[2:]:
    if len(r) <= iT:
        continue
    try:
        n = int(r[iT])
    except ValueError:
        continue
    toks = r[iS].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    by[op.split(".")[0]] += n
    tot += n
print(f"thread instructions per unit: {tot / units:.1f}")
for op, n in by.most_common(top):
    print(f"{op:10s} {n / tot * 100:5.1f}%  {n / units:7.2f}/unit")
