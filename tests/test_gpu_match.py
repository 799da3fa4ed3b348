"""GPU parity of the match loss ||x - x_target||^2 over the sidelobe region
(reading R24) against the float64 oracle."""
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


def window(N, periodic):
    return (0, N) if periodic else (-(N - 1), N)


@pytest.mark.parametrize("N,M,periodic", [(16, 16, False), (64, 64, False), (200, 256, False), (64, 64, True),
                                          (256, 256, True)])
@pytest.mark.parametrize("layout", ["centered", "raw"])
@pytest.mark.parametrize("per_waveform", [False, True])
def test_match_loss_and_grad(N, M, periodic, layout, per_waveform):
    B = 2
    s = cg(B, N, N + 3)
    kb, ke = window(N, periodic)
    rows = ke - kb
    r = SplitMix64(N)
    if per_waveform:
        tgt = (r.uniform(B * rows * M) * 0.05).reshape(B, rows, M).astype(np.float32)
    else:
        tgt = (r.uniform(rows * M) * 0.05).reshape(rows, M).astype(np.float32)
    d = dict(k_max=min(N - 1, 20), d_max=min(M // 2, 24), ml_k=0, ml_d=1, lambda_isl=0.3, lambda_psl=0.0,
             normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_match = 2.0
    spec.target = dev(tgt)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, layout=layout, k_begin=kb, k_end=ke, periodic=periodic)
    ospec = O.LossSpec.from_dict(d)
    for b in range(B):
        tb = tgt[b] if per_waveform else tgt
        Lm, gm = O.match_loss_and_grad(s[b], M, ospec, tb.astype(np.float64), kb, layout, periodic)
        Li, gi, t = O.loss_and_grad(s[b], M, ospec, periodic=periodic)
        L_ref, g_ref = Li + 2.0 * Lm, gi + 2.0 * gm
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b].item(), L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= grad_tol(g_ref, t["sigma_g"])


def test_match_own_surface_is_stationary():
    N = M = 128
    s = cg(1, N, 9)
    surf, _ = graf.af_forward(dev(s), M, out="pow", layout="centered", normalize_output=True)
    spec = graf.LossSpec(k_max=N, d_max=M, lambda_isl=0.0, normalize=1)
    spec.lambda_match = 1.0
    spec.target = surf[0].contiguous()
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, layout="centered")
    assert loss.item() < 1e-9
    assert g.abs().max().item() < 1e-5 * np.abs(s).max()


def test_match_with_hard_psl():
    N, M = 96, 128
    s = cg(2, N, 4)
    kb, ke = window(N, False)
    tgt = (SplitMix64(3).uniform((ke - kb) * M) * 0.02).reshape(ke - kb, M).astype(np.float32)
    d = dict(k_max=30, d_max=40, ml_k=0, ml_d=1, lambda_isl=0.0, lambda_psl=0.0, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_match, spec.lambda_hpsl, spec.target = 1.5, 1.0, dev(tgt)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, layout="centered")
    ospec = O.LossSpec.from_dict(d)
    for b in range(2):
        Lm, gm = O.match_loss_and_grad(s[b], M, ospec, tgt.astype(np.float64), kb, "centered")
        psl, gp, _ = O.hard_psl_and_grad(s[b], M, ospec)
        L_ref, g_ref = 1.5 * Lm + psl, 1.5 * gm + gp
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= 1e-4 * np.abs(g_ref).max() * 2


def test_match_argument_checks():
    s = dev(cg(1, 32, 1))
    spec = graf.LossSpec(k_max=10, d_max=10, lambda_psl=1.0)
    spec.lambda_match, spec.target = 1.0, torch.zeros((63, 32), device="cuda")
    with pytest.raises(graf.GrafError):
        graf.af_loss_grad(s, 32, spec)                       # with soft-PSL: unsupported in v1
    spec.lambda_psl = 0.0
    with pytest.raises(graf.GrafError):
        graf.af_loss_grad(s, 32, spec, k_begin=-5, k_end=5)  # window misses delays of the region


# ------------------------------------------------------------------ mainlobe width
@pytest.mark.parametrize("N,periodic", [(1, False), (8, False), (37, False), (256, False), (64, True), (256, True),
                                        (2048, False)])
def test_mainlobe_width(N, periodic):
    s = cg(2, N, N + 11)
    for b_gamma in (0.5, 5.0):
        E = np.array([O.energy(x) for x in s])
        gam = float(b_gamma / E.mean() ** 2)
        loss, g = graf.mainlobe_width(dev(s), gam, weight=0.7, periodic=periodic)
        for b in range(2):
            W, gref = O.mainlobe_width_and_grad(s[b], gam, periodic)
            assert abs(loss[b].item() - 0.7 * W) <= 1e-4 * max(abs(0.7 * W), 1e-12) + 1e-9
            sc = max(np.abs(gref).max(), 1e-30)
            assert np.abs(g[b].cpu().numpy() - 0.7 * gref).max() <= 1e-4 * 0.7 * sc + 1e-12
