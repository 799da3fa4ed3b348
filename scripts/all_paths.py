"""Drive every kernel and launch path of libgraf.so once at small sizes and check
that every output is finite (a smoke run over all paths; the parity tests check values):

    python scripts/all_paths.py

Covers: forward (c64/abs/pow, raw/centred, windows, M = 64 .. 16384), fused ISL
with the cluster finalize, two-pass soft-PSL, the band cache, the full-plane
single pass and its guarded fallback, hard PSL, match loss, periodic mode,
cross-ambiguity, the generic adjoint, spectral variance (direct and FFT),
Adam, mainlobe width and combine_partials.  Prints one line per case.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_22935_b200 as graf                       # noqa: E402
from graf_inputs import SplitMix64, complex_gaussian, lfm, random_phase   # noqa: E402

dev = torch.device("cuda:0")


def cg(B, N, seed):
    return torch.from_numpy(np.stack([complex_gaussian(SplitMix64(seed * 100 + b), N) for b in range(B)])).to(dev)


def done(name, *ts):
    torch.cuda.synchronize()
    fin = all(bool(torch.isfinite(t if not t.is_complex() else torch.view_as_real(t)).all()) for t in ts
              if t is not None)
    print(f"{name:48s} ok finite={fin}", flush=True)


# ---- forward, every output kind and layout
for N, M in ((64, 64), (100, 256), (256, 256), (1000, 1024)):
    s = cg(2, N, N)
    for out in ("c64", "abs", "pow"):
        for layout in ("raw", "centered"):
            surf, _ = graf.af_forward(s, M, out=out, layout=layout, normalize_output=(out == "abs"))
            done(f"forward N={N} M={M} {out} {layout}", surf)
    surf, _ = graf.af_forward(s, M, out="c64", k_begin=-7, k_end=N // 3)
    done(f"forward window N={N} M={M}", surf)
for N, M, kb, ke in ((4096, 8192, -5, 5), (16384, 16384, 16380, 16384)):
    s = cg(1, N, 7)
    surf, _ = graf.af_forward(s, M, out="c64", layout="raw", k_begin=kb, k_end=ke)
    done(f"forward large N={N} M={M}", surf)

# ---- fused losses
S = graf.LossSpec
s = cg(3, 256, 11)
cases = {
    "ISL fused (cluster finalize)": S(k_max=64, d_max=32, lambda_isl=1.0),
    "ISL + softPSL two-pass": S(k_max=64, d_max=32, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05),
    "softPSL full plane single pass": S(k_max=256, d_max=256, lambda_isl=1.0, lambda_psl=1.0),
    "hard PSL + ISL": S(k_max=40, d_max=20, lambda_isl=1.0, lambda_hpsl=1.0),
    "raw ISL mainlobe 2x3": S(k_max=100, d_max=100, ml_k=2, ml_d=3, lambda_isl=0.5, normalize=0),
}
for name, spec in cases.items():
    lo, g, _ = graf.af_loss_grad(s, 256, spec)
    done(name, lo, g)
    lo, g, surf = graf.af_loss_grad(s, 256, spec, out="pow", k_begin=-30, k_end=30)
    done(name + " + surface", lo, g, surf)
    lo, g, _ = graf.af_loss_grad(s, 256, spec, periodic=True)
    done(name + " periodic", lo, g)

wk = torch.ones(2 * 256 - 1, device=dev)
wd = torch.linspace(0.5, 1.5, 256, device=dev)
wd = 0.5 * (wd + wd.flip(0).roll(1))
lo, g, _ = graf.af_loss_grad(s, 256, S(k_max=64, d_max=32, lambda_isl=1.0, w_k=wk, w_d=wd))
done("weighted ISL", lo, g)

# band cache: narrow Doppler band at M >= 4 * band
s2 = cg(2, 512, 13)
lo, g, _ = graf.af_loss_grad(s2, 2048, S(k_max=64, d_max=64, lambda_isl=1.0, lambda_psl=1.0))
done("band cache N=512 M=2048", lo, g)
s3 = cg(1, 4096, 17)
lo, g, _ = graf.af_loss_grad(s3, 8192, S(k_max=16, d_max=16, lambda_isl=1.0, lambda_psl=1.0))
done("band cache N=4096 M=8192", lo, g)

# full-plane single pass with the guarded fallback (LFM ridge, small T)
sl = torch.from_numpy(np.stack([lfm(256, 1.0), random_phase(SplitMix64(5), 256)])).to(dev)
lo, g, _ = graf.af_loss_grad(sl, 256, S(k_max=256, d_max=256, lambda_isl=0.0, lambda_psl=1.0, temperature=0.001))
done("single pass + guarded fallback", lo, g)

# M = 16384 split path, few rows via sharding
s5 = cg(1, 16384, 19)
spec5 = S(k_max=16384, d_max=16384, lambda_isl=1.0, lambda_psl=1.0)
_, part = graf.af_forward(s5, 16384, out=None, loss=spec5, shard=(3, 2048))
glob = graf.combine_partials(spec5, part[None])
lo, g, _ = graf.af_loss_grad(s5, 16384, spec5, global_partials=glob, shard=(3, 2048))
done("M=16384 sharded loss", lo, g)

# match loss
tgt = torch.rand(2 * 256 - 1, 256, device=dev)
lo, g, _ = graf.af_loss_grad(s, 256, S(k_max=255, d_max=128, lambda_isl=0.0, lambda_match=1.0, target=tgt),
                             k_begin=-255, k_end=256)
done("match loss", lo, g)

# generic adjoint
dA = cg(3, 20 * 256, 23).reshape(3, 20, 256)
g = graf.af_backward(s, 256, dA, k_begin=-10, k_end=10)
done("backward", g)
g = graf.af_backward(s, 256, dA, k_begin=-10, k_end=10, layout="raw", periodic=True)
done("backward periodic", g)

# cross-ambiguity
t = cg(3, 256, 29)
surf, part = graf.xaf_forward(s, t, 256, out="c64", loss=S(k_max=64, d_max=32))
done("xaf forward", surf, part)
lo, g1, g2, _ = graf.xaf_loss_grad(s, t, 256, S(k_max=64, d_max=32, lambda_isl=1.0, lambda_psl=1.0))
done("xaf loss_grad", lo, g1, g2)
dX = cg(3, 9 * 256, 31).reshape(3, 9, 256)
g1, g2 = graf.xaf_backward(s, t, 256, dX, k_begin=-4, k_end=5)
done("xaf backward", g1, g2)

# section 7: spectral variance, Adam, LPI optimizer, mainlobe width
for N in (16, 256):
    sv = cg(2, N, 37)
    lo, g = graf.spectral_variance(sv, weight=2.0)
    done(f"spectral variance N={N}", lo, g)
th = torch.rand(2, 64, device=dev) * 6.28
opt = graf.LpiOptimizer(th, [0.1, 1.0], per_graph=4)
lo = opt.run(9)
done("LpiOptimizer (graph replay)", lo, opt.theta)
lo, g = graf.mainlobe_width(s, gamma=0.3)
done("mainlobe width", lo, g)
lo, g = graf.mainlobe_width(s, gamma=0.3, periodic=True)
done("mainlobe width periodic", lo, g)
parts = torch.stack([graf.af_forward(s, 256, out=None, loss=cases["ISL + softPSL two-pass"], shard=(r, 3))[1]
                     for r in range(3)])
done("combine_partials", graf.combine_partials(cases["ISL + softPSL two-pass"], parts))
print("ALL PATHS DONE", flush=True)
