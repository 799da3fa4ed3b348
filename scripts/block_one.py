#!/usr/bin/env python
"""One graf_af_loss_grad call on the first B waveforms of a config, after two warm-up calls
(launch list / grid sizes under ncu; development tool).  Usage: block_one.py <config> <B>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_22935_b200 as graf  # noqa: E402
from graf_inputs import CONFIGS, config_waveforms  # noqa: E402

cid, B = int(sys.argv[1]), int(sys.argv[2])
c = CONFIGS[cid]
s = torch.from_numpy(config_waveforms(cid, batch=B)).cuda()
spec = dict(c["loss"])
if cid in (1, 3):
    spec["normalize"] = 0
spec = graf.LossSpec.from_dict(spec)
for _ in range(3):
    lo, g, _ = graf.af_loss_grad(s, c["M"], spec, out=c["surface"])
torch.cuda.synchronize()
print("ok", lo[0].item())
