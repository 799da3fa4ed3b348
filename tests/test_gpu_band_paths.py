"""GPU parity of the narrow-band and zero-padded specialisations against
the float64 oracle.  They are: the band-edge epilogues, the band cache, the
band-edge inverse FFT, the pruned pass-1 forward FFT (loss band |d| <= d_max < M/E),
and the half-slot lag product and correlation (2N <= M).  The loss kinds are ISL-only
fused, soft-PSL two-pass (with and without the band cache), match and hard PSL.  The
sizes are M = 2048, 4096, 8192 (M >= 2048 compiles these paths), with N = M/2, N < M/2
odd, and N > M/2, so each path is taken and its guard checked.  Tolerances as in
test_gpu_parity.py (reading R18).
"""
import numpy as np
import pytest
import torch

from graf_inputs import SplitMix64, complex_gaussian
from oracle import graf_oracle as O

from gradtol import grad_tol

pytestmark = pytest.mark.gpu

graf = pytest.importorskip("paper_2506_22935_b200")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def cg(B, N, seed):
    return np.stack([complex_gaussian(SplitMix64(seed * 1000 + b), N) for b in range(B)])


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SHAPES = [(1024, 2048), (777, 2048), (1500, 2048), (2048, 4096), (1001, 4096), (600, 8192)]
BANDS = [
    # ISL only (one fused pass), band below M/E
    dict(k_max=40, d_max=20, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    # weighted-free ISL + soft-PSL (two passes, band cache), band = M/E - 1 (the edge)
    dict(k_max=60, d_max=None, ml_k=1, ml_d=1, lambda_isl=0.5, lambda_psl=1.0, temperature=0.05, normalize=1),
    # soft-PSL with a band of exactly M/E bins: the edge paths must NOT be taken
    dict(k_max=30, d_max="T", ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.5, temperature=0.05, normalize=1),
]


def spec_for(d, M):
    d = dict(d)
    T = M // 16          # E = 16 for M = 2048 ... 8192
    if d["d_max"] is None:
        d["d_max"] = T - 1
    elif d["d_max"] == "T":
        d["d_max"] = T
    return d


@pytest.mark.parametrize("si", range(len(BANDS)))
@pytest.mark.parametrize("N,M", SHAPES)
def test_band_paths_loss_grad(si, N, M):
    d = spec_for(BANDS[si], M)
    s = cg(2, N, N + si)
    loss, g, _ = graf.af_loss_grad(dev(s), M, graf.LossSpec.from_dict(d))
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(d)
    for b in range(2):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b], L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol, (b, np.abs(g[b] - g_ref).max(), tol)


@pytest.mark.parametrize("N,M", [(1024, 2048), (900, 4096)])
def test_band_paths_forward_partials_and_sharding(N, M):
    # pass-1 statistics of the band-edge forward (pruned FFT) combine across delay shards
    d = spec_for(BANDS[1], M)
    spec = graf.LossSpec.from_dict(d)
    s = cg(2, N, 3)
    ds = dev(s)
    L1, g1, _ = graf.af_loss_grad(ds, M, spec)
    G = 3
    parts = torch.stack([graf.af_forward(ds, M, out=None, loss=spec, shard=(r, G))[1] for r in range(G)])
    glob = graf.combine_partials(spec, parts)
    gsum = sum(graf.af_loss_grad(ds, M, spec, global_partials=glob, shard=(r, G))[1] for r in range(G))
    assert (gsum - g1).abs().max().item() <= 1e-4 * g1.abs().max().item()


@pytest.mark.parametrize("N,M", [(1024, 2048), (1001, 4096)])
def test_band_paths_match_loss(N, M):
    B = 2
    s = cg(B, N, N + 11)
    kb, ke = -(N - 1), N
    r = SplitMix64(N)
    tgt = (r.uniform((ke - kb) * M) * 0.01).reshape(ke - kb, M).astype(np.float32)
    d = dict(k_max=25, d_max=M // 16 - 2, ml_k=0, ml_d=1, lambda_isl=0.3, lambda_psl=0.0, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_match = 2.0
    spec.target = dev(tgt)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, k_begin=kb, k_end=ke)
    ospec = O.LossSpec.from_dict(d)
    for b in range(B):
        Lm, gm = O.match_loss_and_grad(s[b], M, ospec, tgt.astype(np.float64), kb, "centered", False)
        Li, gi, t = O.loss_and_grad(s[b], M, ospec)
        L_ref, g_ref = Li + 2.0 * Lm, gi + 2.0 * gm
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= grad_tol(g_ref, t["sigma_g"])


@pytest.mark.parametrize("N,M", [(1024, 2048), (700, 4096)])
def test_band_paths_hard_psl(N, M):
    d = dict(k_max=30, d_max=M // 16 - 1, ml_k=0, ml_d=1, lambda_isl=0.0, lambda_psl=0.0, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_hpsl = 1.0
    s = cg(2, N, 17)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec)
    ospec = O.LossSpec.from_dict(d)
    for b in range(2):
        psl, gref, cell = O.hard_psl_and_grad(s[b], M, ospec, False)
        assert abs(loss[b].item() - psl) <= 1e-4 * abs(psl), (b, cell)
        E = O.energy(s[b])
        sig = 2 * psl / E * np.abs(s[b]).max()
        assert np.abs(g[b].cpu().numpy() - gref).max() <= 1e-4 * max(np.abs(gref).max(), sig), (b, cell)
