#!/usr/bin/env python
"""One delay-sharded single pass (phase 1, phase 2, guarded fallback) of shard r of G at c5,
after a warm-up round: the launch list for ncu (development tool).
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python scripts/sp_one.py 8 0"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_22935_b200 as graf  # noqa: E402
from graf_inputs import CONFIGS, config_waveforms  # noqa: E402
from paper_2506_22935_b200.sharding import GrafBackend  # noqa: E402

G, r = int(sys.argv[1]), int(sys.argv[2])
c = CONFIGS[5]
M = c["M"]
spec = graf.LossSpec.from_dict(dict(c["loss"]))
s = torch.from_numpy(config_waveforms(5)).cuda()
be = GrafBackend()
for it in range(2):
    parts = [be.sp_begin(s, M, spec, (q, G)) for q in range(G) if q != r]
    torch.cuda.synchronize()
    print("MARK begin", it, flush=True)
    mine = be.sp_begin(s, M, spec, (r, G))     # last: the workspace holds shard r's gradient
    glob = be.combine(spec, torch.stack(parts[:r] + [mine] + parts[r:]))
    loss, g, valid = be.sp_end(s, M, spec, glob, (r, G))
    skip = valid.to(torch.int32).contiguous()
    p2 = be.forward_partials(s, M, spec, (r, G), skip=skip)
    loss, g = be.loss_grad(s, M, spec, be.combine(spec, torch.stack([p2] * G)), (r, G), skip=skip, loss_out=loss, grad=g)
    torch.cuda.synchronize()
print("ok", loss[0].item(), bool(valid.all()))
