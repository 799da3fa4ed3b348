#!/usr/bin/env python
"""Instruction mix and stall samples of ONE row phase of a kernel (development tool).

  ncu -i <rep> --page source --csv --print-source sass > sass.csv
  python scripts/ncu_phase_mix.py sass.csv <phase index>   # phases as numbered by ncu_phases.py
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if len(r) > 2 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cuts = [-1] + [i for i, r in enumerate(data) if "BAR.SYNC" in r[isrc]] + [len(data)]
segs = [(cuts[j] + 1, cuts[j + 1]) for j in range(len(cuts) - 1)]
tot = sum(float(r[ist] or 0) for r in data)
segs = [(a, b) for a, b in segs if sum(float(data[i][ist] or 0) for i in range(a, min(b + 1, len(data)))) / tot > 0.003]
a, b = segs[int(sys.argv[2])]
c, st = collections.Counter(), collections.Counter()
for i in range(a, min(b + 1, len(data))):
    op = re.sub(r"^@!?U?P\w+\s+", "", data[i][isrc].strip()).split(" ")[0]
    c[op] += float(data[i][iex] or 0)
    st[op] += float(data[i][ist] or 0)
print(f"phase {sys.argv[2]}: SASS {a}-{b}, {sum(c.values()) / 1e6:.1f} M warp instructions, "
      f"{100 * sum(st.values()) / tot:.1f} % of stall samples")
for k, v in c.most_common(40):
    print(f"  {k:28s} {v / 1e6:8.1f} M   stall {100 * st[k] / tot:5.2f} %")
