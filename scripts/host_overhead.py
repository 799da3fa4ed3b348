import sys, time, os
sys.path.insert(0, "/root/repo")
import torch, cProfile, pstats
import paper_2506_22935_b200 as graf
from graf_inputs import CONFIGS, config_waveforms
cfg = CONFIGS[2]
spec = graf.LossSpec.from_dict(cfg["loss"])
s = torch.from_numpy(config_waveforms(2)).cuda()
ws = graf.graf.Workspace()
grad = torch.empty((256, 256), dtype=torch.complex64, device="cuda")
lo = torch.empty(256, dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for _ in range(10):
    graf.af_loss_grad(s, 256, spec, ws=ws, grad=grad, loss_out=lo, stream=st)
torch.cuda.synchronize()
t = time.perf_counter()
n = 2000
for _ in range(n):
    graf.af_loss_grad(s, 256, spec, ws=ws, grad=grad, loss_out=lo, stream=st)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host us/call {(t1-t)/n*1e6:.1f}  total us/call incl drain {(t2-t)/n*1e6:.1f}")
pr = cProfile.Profile(); pr.enable()
for _ in range(500):
    graf.af_loss_grad(s, 256, spec, ws=ws, grad=grad, loss_out=lo, stream=st)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
