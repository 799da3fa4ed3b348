#!/usr/bin/env python
"""Per-shard compute time of the c5 delay-sharded step on ONE GPU (development tool).

The pool gives one GPU per call, so the NCCL step itself cannot be timed.  This script
times what each rank of a G-way delay sharding would compute (folded rows
k = r mod G): shard r's single pass (sp_begin), then, with the partials of all G shards
combined as the all_gather would deliver them, its phase 2 (sp_end) and the two guarded
fallback launches.  Shards run one after another, never concurrently, so no kernel waits
on another rank.  Output: per G the max and mean over shards of the compute time, the
ratio to the unsharded step, and a check that the summed shard gradients equal the
unsharded gradient.  The collectives (two B x 48 B all_gathers and a 1 MiB all_reduce)
are not in these numbers.

  python scripts/shard_times.py [G ...]      # default 1 2 4 8
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_22935_b200 as graf  # noqa: E402
from graf_inputs import CONFIGS, config_waveforms  # noqa: E402
from paper_2506_22935_b200.sharding import GrafBackend  # noqa: E402

CID = 5
REPS = 5


def main():
    Gs = [int(a) for a in sys.argv[1:]] or [1, 2, 4, 8]
    c = CONFIGS[CID]
    M = c["M"]
    spec = graf.LossSpec.from_dict(dict(c["loss"]))
    s = torch.from_numpy(config_waveforms(CID)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    be = GrafBackend()
    loss0, g0, _ = graf.af_loss_grad(s, M, spec)
    torch.cuda.synchronize()
    out = {"config": c.get("name", f"c{CID}"), "B": c["B"], "N": c["N"], "M": M, "reps": REPS, "G": {}}
    for G in Gs:
        if G == 1:   # the unsharded ABI call (the single pass needs shard_count >= 2)
            ts = []
            for rep in range(REPS + 1):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graf.af_loss_grad(s, M, spec)
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    ts.append(e0.elapsed_time(e1))
            med = sorted(ts)[len(ts) // 2]
            out["G"][1] = {"shard_ms_max": med, "shard_ms_mean": med, "shard_ms": [med]}
            continue
        assert be.single_pass_eligible(s, M, spec, (0, G))
        bes = [GrafBackend() for _ in range(G)]
        times = [[] for _ in range(G)]
        times1 = [[] for _ in range(G)]
        gsum = None
        for rep in range(REPS + 1):   # the first repetition warms up
            parts, t1 = [], []
            for r in range(G):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                parts.append(bes[r].sp_begin(s, M, spec, (r, G)))
                e1.record()
                torch.cuda.synchronize()
                t1.append(e0.elapsed_time(e1))
            glob = be.combine(spec, torch.stack(parts))
            gsum = torch.zeros_like(g0)
            for r in range(G):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                loss, g, valid = bes[r].sp_end(s, M, spec, glob, (r, G))
                skip = valid.to(torch.int32).contiguous()
                p2 = bes[r].forward_partials(s, M, spec, (r, G), skip=skip)
                e1.record()
                torch.cuda.synchronize()
                t2 = e0.elapsed_time(e1)
                # (the second gather would go here; with every waveform valid the guarded
                # launches exit at once, so the combined record is not needed for timing)
                glob2 = be.combine(spec, torch.stack([p2] * G)) if G > 1 else be.combine(spec, p2[None])
                e0.record()
                loss, g = bes[r].loss_grad(s, M, spec, glob2, (r, G), skip=skip, loss_out=loss, grad=g)
                e1.record()
                torch.cuda.synchronize()
                t2 += e0.elapsed_time(e1)
                assert bool(valid.all()), "c5 inputs satisfy the R13 rule"
                gsum += g
                if rep:
                    times[r].append(t1[r] + t2)
                    times1[r].append(t1[r])
        per = [sorted(t)[len(t) // 2] for t in times]
        per1 = [sorted(t)[len(t) // 2] for t in times1]
        err = float((gsum - g0).abs().max() / g0.abs().max())
        out["G"][G] = {"shard_ms_max": max(per), "shard_ms_mean": sum(per) / G, "shard_ms": per, "phase1_ms": per1,
                       "sum_of_shards_vs_unsharded_grad_relerr": err}
    base = out["G"].get(1, {}).get("shard_ms_max")
    for G, d in out["G"].items():
        if base:
            d["compute_speedup_vs_G1"] = base / d["shard_ms_max"]
            d["compute_efficiency"] = base / d["shard_ms_max"] / G
    print(json.dumps(out))


if __name__ == "__main__":
    main()
