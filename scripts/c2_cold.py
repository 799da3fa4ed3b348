"""c2 step time warm vs after an L2 flush (256 MiB memset), one call per graph replay,
to size the cold-start share of the fused-ISL kernel.  Usage: python scripts/c2_cold.py"""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22935_b200 as graf
from paper_2506_22935_b200.graf import Workspace

B, N, M = 256, 256, 256
s = torch.polar(torch.ones(B, N, device="cuda"), torch.rand(B, N, device="cuda") * 6.2832).to(torch.complex64)
spec = graf.LossSpec(k_max=64, d_max=32, lambda_isl=1.0)
ws, st = Workspace(), torch.cuda.Stream()
g = torch.empty(B, N, dtype=torch.complex64, device="cuda"); lo = torch.empty(B, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with torch.cuda.stream(st):
    graf.af_loss_grad(s, M, spec, ws=ws, grad=g, loss_out=lo, stream=st)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        graf.af_loss_grad(s, M, spec, ws=ws, grad=g, loss_out=lo, stream=st)
    for mode in ("warm", "flushed", "flushed+s-touch", "warm"):
        ts = []
        for i in range(40):
            if mode != "warm":
                flush.fill_(i & 255)
                if mode == "flushed+s-touch":
                    s.add_(0)          # s back in L2, twiddles / code still cold
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st); gr.replay(); e1.record(st)
            st.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{mode:18s} median {ts[len(ts)//2]:6.2f} us  min {ts[0]:6.2f}", flush=True)
