#!/usr/bin/env python
"""Summarise an ncu report (--set full) into a committed text file.

  python scripts/ncu_summary.py <report.ncu-rep> <out.txt> [--traffic-key cN]

Writes: the speed-of-light / occupancy / launch figures, warp-stall breakdown,
dram bytes (the roofline 'traffic'), and the top source lines by stall samples.
With --traffic-key it also merges dram read+write bytes into profiles/traffic.json
(read by bench.py).
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Occupancy", "Grid Size",
        "Block Size", "Executed Instructions", "No Eligible", "Warp Cycles Per Issued Instruction",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput", "Compute (SM) Throughput",
        "Dynamic Shared Memory Per Block", "Memory Throughput", "L2 Hit Rate"]
RAW = re.compile(r"(average_warps_issue_stalled_.*_per_issue_active|dram__bytes_(read|write)\.sum$|"
                 r"sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active|"
                 r"sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active|"
                 r"l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct|launch__func)")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    lines = [f"# ncu summary of {os.path.basename(rep)}"]
    r = list(csv.reader(ncu(rep, "--page", "details", "--csv").splitlines()))
    hdr = r[0]
    kname = None
    for row in r[1:]:
        d = dict(zip(hdr, row))
        kname = kname or d.get("Kernel Name")
        if d.get("Metric Name") in KEEP:
            lines.append(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
    lines.insert(1, f"kernel: {kname}")
    r = list(csv.reader(ncu(rep, "--page", "raw", "--csv").splitlines()))
    h, u, v = r[0], r[1], r[2]
    dram = 0.0
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for a, b, c in zip(h, u, v):
        if RAW.search(a):
            lines.append(f"{a:80s} {c} {b}")
            if re.search(r"dram__bytes_(read|write)\.sum$", a):
                dram += float(c.replace(",", "")) * scale.get(b, 1)
    lines.append(f"dram bytes (read + write) per launch: {dram:.6g}")
    # hot source lines by stall samples
    txt = ncu(rep, "--page", "source", "--csv", "--print-source", "cuda,sass")
    rows = list(csv.reader(txt.splitlines()))
    cur, hdr, src = None, None, None
    inst, stall, text = collections.Counter(), collections.Counter(), {}
    for row in rows:
        if len(row) == 2 and row[0] == "File Path":
            cur = row[1].split("/")[-1]
            continue
        if len(row) >= 2 and row[0] == "Line No":
            hdr = row
            ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr and len(row) == len(hdr):
            if row[0]:
                src = (cur, row[0])
                text[src] = row[1].strip()
            elif src is not None:
                try:
                    inst[src] += float(row[ie] or 0)
                    stall[src] += float(row[st] or 0)
                except ValueError:
                    pass
    ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
    lines.append("")
    lines.append("top source lines by warp-stall samples (inst% / stall%):")
    for k, s in stall.most_common(25):
        lines.append(f"  {k[0][:18]:18s} L{k[1]:>4} {100 * inst[k] / ti:5.1f}% {100 * s / ts:5.1f}%  {text.get(k, '')[:100]}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if key:
        tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        d[key] = dram
        d.setdefault("_note", "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant "
                              "af_rows_kernel, from one ncu --set full capture (scripts/ncu_summary.py)")
        json.dump(d, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
