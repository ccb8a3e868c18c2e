#!/usr/bin/env python
"""Summarise `nvcc -Xptxas=-v` output: one line per kernel (registers, spill bytes, stack)."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        stack, st, ld = m.groups()
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        name = re.sub(r"^_ZN3ens", "", cur)
        print(f"{m.group(1):>4} regs  stack {stack:>5}  spill {st:>5}/{ld:<5} {name[:110]}")
        cur = None
