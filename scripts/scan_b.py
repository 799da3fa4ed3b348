"""Development scan: step time of the c2 shape vs batch size (fixed-overhead probe)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_22935_b200 as graf
from graf_inputs import CONFIGS, config_waveforms

cfg = CONFIGS[2]
spec = graf.LossSpec.from_dict(cfg["loss"])
N = M = 256
st = torch.cuda.Stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for B in [1, 8, 32, 74, 148, 256, 512, 1024, 2048]:
    s = torch.from_numpy(config_waveforms(2, batch=B, start=0)).cuda() if B <= 256 else \
        torch.from_numpy(config_waveforms(2, batch=256, start=0)).cuda().repeat(B // 256, 1)
    ws = graf.graf.Workspace()
    grad = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    lo = torch.empty((B,), dtype=torch.float64, device="cuda")
    def call():
        graf.af_loss_grad(s, M, spec, ws=ws, grad=grad, loss_out=lo, stream=st)
    with torch.cuda.stream(st):
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        call()
    ts = []
    with torch.cuda.stream(st):
        for i in range(40):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st); g.replay(); b.record(st); b.synchronize()
            if i >= 5:
                ts.append(a.elapsed_time(b) * 1000)
    ts.sort()
    print(json.dumps({"B": B, "us_median": ts[len(ts) // 2], "us_min": ts[0], "launches": graf.lib().graf_last_launch_count()}))
