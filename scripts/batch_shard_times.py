#!/usr/bin/env python
"""Per-rank compute time of the batch-sharded step (c2-c4) on ONE GPU:
graf_af_loss_grad on rank 0's block of B/G waveforms for G = 1, 2, 4, 8 (development tool;
CUDA-graph replay per step, L2 flushed between steps, CUDA events, median).  No collective
is on this data path, so this is the whole per-rank step.

  python scripts/batch_shard_times.py [config ...]      # default 2 3 4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_22935_b200 as graf  # noqa: E402
from graf_inputs import CONFIGS, config_waveforms  # noqa: E402
from paper_2506_22935_b200.sharding import batch_slice  # noqa: E402

REPS = 15


def time_block(s, M, spec, surface):
    B, N = s.shape
    ws = graf.graf.Workspace()
    st = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    grad = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    lo = torch.empty((B,), dtype=torch.float64, device="cuda")
    surf = None
    if surface:
        surf = torch.empty((B, 2 * N - 1, M), dtype=torch.complex64 if surface == "c64" else torch.float32,
                           device="cuda")

    fwd = os.environ.get("GRAF_TUNE_MODE") == "forward"   # full-surface forward (c3 --mode forward)

    def call():
        if fwd:
            graf.af_forward(s, M, out=surface, layout="centered", ws=ws, surface=surf)
        else:
            graf.af_loss_grad(s, M, spec, out=surface, surface=surf, loss_out=lo, grad=grad, ws=ws)

    with torch.cuda.stream(st):
        for _ in range(3):
            call()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            call()
        ts = []
        for _ in range(REPS):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            g.replay()
            e1.record(st)
            st.synchronize()
            ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [2, 3, 4]
    out = {}
    for cid in cfgs:
        c = CONFIGS[cid]
        spec = dict(c["loss"])
        if cid in (1, 3):
            spec["normalize"] = 0
        spec = graf.LossSpec.from_dict(spec)
        s_all = torch.from_numpy(config_waveforms(cid)).cuda()
        res = {}
        for G in (1, 2, 4, 8):
            sl = batch_slice(c["B"], 0, G)
            ms = time_block(s_all[sl].contiguous(), c["M"], spec, c["surface"])
            res[G] = {"B_per_rank": sl.stop - sl.start, "ms": ms}
        for G in res:
            res[G]["efficiency"] = res[1]["ms"] / res[G]["ms"] / G
        out[f"c{cid}"] = res
    out["lib"] = os.path.basename(os.environ.get("GRAF_LIB_PATH", "libgraf.so"))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
