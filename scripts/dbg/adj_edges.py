import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2506_22935_b200 as graf
from oracle import graf_oracle as O
from graf_inputs import SplitMix64, complex_gaussian, random_phase
def cg(B, N, seed):
    return np.stack([complex_gaussian(SplitMix64(seed * 1000 + b), N) for b in range(B)])
for (N, M, kb, ke) in [(1000, 16384, -999, -900), (1000, 16384, -50, 50), (1000, 16384, 900, 1000),
                       (3000, 16384, -2999, -2900), (1000, 8192, -999, -900), (4000, 8192, -3999, -3900),
                       (16384, 16384, -16383, -16373), (16384, 16384, 16373, 16384)]:
    s = cg(1, N, 5)
    rows = np.arange(kb, ke)
    dA = cg(1, len(rows) * M, 6).reshape(1, len(rows), M)
    g = graf.af_backward(torch.from_numpy(s).cuda(), M, torch.from_numpy(dA).cuda(), k_begin=kb, k_end=ke, layout="raw").cpu().numpy()
    ref = O.adjoint(s[0], M, dA[0].astype(np.complex128), rows)
    e = np.abs(g[0] - ref).max() / np.abs(ref).max()
    # forward rows too
    A, _ = graf.af_forward(torch.from_numpy(s).cuda(), M, out="c64", layout="raw", k_begin=kb, k_end=ke)
    Aref = O.ambiguity(s[0], M, rows=rows)
    ea = np.abs(A.cpu().numpy()[0] - Aref).max() / O.energy(s[0])
    bad = np.where(np.abs(g[0] - ref) > 1e-4 * np.abs(ref).max())[0]
    print(N, M, kb, ke, "adj rel", e, "fwd rel/E", ea, "bad idx", bad[:10], len(bad), flush=True)
