#!/usr/bin/env python
"""Warp-stall samples of one kernel split at its CTA barriers (development tool).

  ncu -i <rep> --page source --csv --print-source sass > sass.csv; python scripts/ncu_phases.py sass.csv
"""
import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if len(r)>2 and r[0]=="Address": hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(r)
isrc=hdr.index("Source"); ist=hdr.index("Warp Stall Sampling (All Samples)")
reasons=[k for k in hdr if k.startswith('stall_') and 'Not Issued' not in k]
idx={k:hdr.index(k) for k in reasons}
tot=sum(float(r[ist] or 0) for r in data)
seg=[]; start=0
for i,r in enumerate(data):
    if "BAR.SYNC" in r[isrc]:
        seg.append((start,i)); start=i+1
seg.append((start,len(data)-1))
for a,b in seg:
    s=sum(float(data[i][ist] or 0) for i in range(a,b+1))
    if s/tot<0.003: continue
    rs={k:sum(float(data[i][idx[k]] or 0) for i in range(a,b+1)) for k in reasons}
    top=sorted(rs.items(), key=lambda x:-x[1])[:6]
    print(f"{a:6d}-{b:6d} {100*s/tot:5.1f}% | " + ", ".join(f"{k[6:]} {100*v/tot:.1f}" for k,v in top))
