"""GPU parity of the cross-ambiguity X = sum s1[n] conj(s2[n-k]) W^{mn} (
SURVEY.md §8(f) NEXT-4; reading R25) against the float64 oracle."""
import numpy as np
import pytest
import torch

from graf_inputs import SplitMix64, complex_gaussian
from oracle import graf_oracle as O

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


@pytest.mark.parametrize("N,M", [(1, 2), (7, 8), (33, 64), (100, 128), (256, 256), (1000, 1024), (2048, 4096)])
@pytest.mark.parametrize("kind", ["c64", "abs"])
def test_cross_surface(N, M, kind):
    s1, s2 = cg(2, N, N), cg(2, N, N + 1)
    surf, _ = graf.xaf_forward(dev(s1), dev(s2), M, out=kind, layout="centered")
    got = surf.cpu().numpy()
    for b in range(2):
        X = np.roll(O.cross_ambiguity(s1[b], s2[b], M), M // 2, axis=1)
        ref = X if kind == "c64" else np.abs(X)
        scale = np.sqrt(O.energy(s1[b]) * O.energy(s2[b]))
        assert np.abs(got[b] - ref).max() <= 1e-5 * scale, (N, M, b)


SPECS = [
    dict(k_max=5, d_max=4, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=20, d_max=16, ml_k=0, ml_d=1, lambda_isl=0.5, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=3, d_max=5, ml_k=1, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=0),
]


@pytest.mark.parametrize("si", range(len(SPECS)))
@pytest.mark.parametrize("N,M", [(16, 16), (60, 64), (256, 256), (500, 512)])
def test_cross_loss_and_both_gradients(si, N, M):
    s1, s2 = cg(3, N, 10 + si), cg(3, N, 20 + si)
    spec = graf.LossSpec.from_dict(SPECS[si])
    loss, g1, g2, _ = graf.xaf_loss_grad(dev(s1), dev(s2), M, spec)
    ospec = O.LossSpec.from_dict(SPECS[si])
    for b in range(3):
        L, r1, r2 = O.cross_loss_and_grad(s1[b], s2[b], M, ospec)
        assert abs(loss[b].item() - L) <= 1e-4 * abs(L)
        gm = max(np.abs(r1).max(), np.abs(r2).max())
        if ospec.normalize:   # the cancelling normalisation terms set the scale (reading R18)
            E1, E2 = O.energy(s1[b]), O.energy(s2[b])
            gm = max(gm, L / np.sqrt(E1 * E2) * max(np.abs(s1[b]).max(), np.abs(s2[b]).max()))
        assert np.abs(g1[b].cpu().numpy() - r1).max() <= 1e-4 * gm
        assert np.abs(g2[b].cpu().numpy() - r2).max() <= 1e-4 * gm


def test_cross_with_itself_is_auto():
    N = M = 128
    s = dev(cg(2, N, 3))
    spec = graf.LossSpec(k_max=30, d_max=20, ml_k=0, ml_d=1, lambda_isl=1.0)
    la, ga, _ = graf.af_loss_grad(s, M, spec)
    lx, g1, g2, _ = graf.xaf_loss_grad(s, s, M, spec)
    assert torch.allclose(lx, la, rtol=1e-5)
    assert (g1 + g2 - ga).abs().max().item() <= 1e-4 * ga.abs().max().item()


@pytest.mark.parametrize("N,M,window", [(16, 16, None), (60, 64, (-7, 12)), (256, 512, (-100, 50))])
def test_cross_backward(N, M, window):
    B = 2
    s1, s2 = cg(B, N, N + 2), cg(B, N, N + 3)
    kb, ke = window if window else (-(N - 1), N)
    rows = np.arange(kb, ke)
    dA = cg(B, len(rows) * M, N + 4).reshape(B, len(rows), M)
    g1, g2 = graf.xaf_backward(dev(s1), dev(s2), M, dev(dA), k_begin=kb, k_end=ke, layout="raw")
    for b in range(B):
        r1, r2 = O.cross_adjoint(s1[b], s2[b], M, dA[b].astype(np.complex128), rows)
        sc = max(np.abs(r1).max(), np.abs(r2).max())
        assert np.abs(g1[b].cpu().numpy() - r1).max() <= 1e-4 * sc
        assert np.abs(g2[b].cpu().numpy() - r2).max() <= 1e-4 * sc


def test_cross_limits():
    s = dev(cg(1, 16, 1))
    with pytest.raises(graf.GrafError):
        graf.xaf_forward(s, s, 8192, out="c64")       # M > 4096: v1 limit
