"""Timing sweep of the c2 fused-ISL step over the delay mask k_max and batch B
(row-count / wave-quantisation effects).  Usage: python scripts/c2_rows.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22935_b200 as graf

def t_of(B, N, M, kmax, dmax=32, reps=50):
    s = torch.polar(torch.ones(B, N, device="cuda"), torch.rand(B, N, device="cuda") * 6.2832).to(torch.complex64)
    spec = graf.LossSpec(k_max=kmax, d_max=dmax, lambda_isl=1.0)
    from paper_2506_22935_b200.graf import Workspace; ws = Workspace()
    st = torch.cuda.Stream()
    g = torch.empty(B, N, dtype=torch.complex64, device="cuda"); lo = torch.empty(B, dtype=torch.float64, device="cuda")
    with torch.cuda.stream(st):
        graf.af_loss_grad(s, M, spec, ws=ws, grad=g, loss_out=lo, stream=st)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(10):
                graf.af_loss_grad(s, M, spec, ws=ws, grad=g, loss_out=lo, stream=st)
        gr.replay(); st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            gr.replay()
        e1.record(st)
    st.synchronize()
    return e0.elapsed_time(e1) / (reps * 10) * 1e3

import sys as _s
KS = [int(x) for x in _s.argv[1].split(',')] if len(_s.argv) > 1 else [47, 48, 55, 56, 63, 64, 71, 72, 80]
BS = [int(x) for x in _s.argv[2].split(',')] if len(_s.argv) > 2 else [148, 222, 240, 256, 296, 444, 592]
for kmax in KS:
    print(f"B=256 N=256 k_max={kmax:3d}: {t_of(256, 256, 256, kmax):7.2f} us", flush=True)
for B in BS:
    print(f"B={B:3d} k_max=64: {t_of(B, 256, 256, 64):7.2f} us", flush=True)
