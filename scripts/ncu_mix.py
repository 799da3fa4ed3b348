#!/usr/bin/env python
"""Dynamic SASS instruction mix of an ncu report (per opcode, and per source line).

  python scripts/ncu_mix.py <report.ncu-rep> [units]   # units: divide counts by this (e.g. rows x warps)
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = r[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
c, st = collections.Counter(), collections.Counter()
tot = 0
for x in r[2:]:
    s = x[iS].strip()
    e = int(x[iE] or 0)
    op = s.split()[0]
    if op.startswith("@"):
        op = s.split()[1]
    op = op.split(".")[0]
    c[op] += e
    st[op] += int(x[iW] or 0)
    tot += e
print(f"total warp instructions {tot}  per unit {tot / units:.1f}")
for k, v in c.most_common(32):
    print(f"{k:8s} {v:12d} {100 * v / tot:5.1f}%  per-unit {v / units:8.1f}  stall-samples {st[k]}")
