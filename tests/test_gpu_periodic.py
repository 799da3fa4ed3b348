"""GPU parity of the periodic mode (graf_af_desc.periodic = 1): the paper's own
circular surface, Eq. 2 / Algorithm 1 (L239-256) with the FFT's
e^{-j} (reading R2), its losses and adjoint, against
the float64 oracle (oracle/graf_oracle.py, periodic=True) on the same seeded
inputs.  Tolerances as in test_gpu_parity.py (reading R18).
"""
import numpy as np
import pytest
import torch

from graf_inputs import SplitMix64, complex_gaussian, frank, random_phase
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


# ------------------------------------------------------------------ surface
@pytest.mark.parametrize("N", [2, 4, 16, 64, 256, 1024])
@pytest.mark.parametrize("kind", ["c64", "abs", "pow"])
def test_periodic_surface_full(N, kind):
    s = cg(2, N, N)
    for layout in ("raw", "centered"):
        surf, _ = graf.af_forward(dev(s), N, out=kind, layout=layout, periodic=True)
        got = surf.cpu().numpy()
        for b in range(2):
            ref = O.surface(s[b], N, kind, layout, periodic=True)
            scale = O.energy(s[b]) ** (2 if kind == "pow" else 1)
            assert np.abs(got[b] - ref).max() <= 1e-5 * scale, (N, kind, layout, b)


@pytest.mark.parametrize("N,window", [(16, (-8, 8)), (64, (-5, 9)), (64, (40, 64)), (256, (-128, 128)),
                                      (256, (-255, -200)), (1024, (-512, 512))])
def test_periodic_surface_windows(N, window):
    s = cg(1, N, 3 * N)
    kb, ke = window
    surf, _ = graf.af_forward(dev(s), N, out="c64", layout="centered", k_begin=kb, k_end=ke, periodic=True)
    ref = O.surface(s[0], N, "c64", "centered", k_begin=kb, k_end=ke, periodic=True)
    assert np.abs(surf.cpu().numpy()[0] - ref).max() <= 1e-5 * O.energy(s[0])


@pytest.mark.parametrize("N", [64, 256])
def test_algorithm1_exactly(N):
    # Alg. 1 in plain torch (float64, CPU): S = circshift rows, R = s * conj(S),
    # X = FFT(R, dim=1), chi = |X|^2, fftshift over both axes.  The device call:
    # periodic pow surface over delays [-N/2, N/2) with centred Doppler.
    s = cg(1, N, 5)[0]
    st = torch.from_numpy(s)
    S = torch.stack([torch.roll(st, k) for k in range(N)])          # S[k, n] = s[(n - k) mod N]
    X = torch.fft.fft(st[None, :] * torch.conj(S), dim=1)
    chi = torch.fft.fftshift((X * torch.conj(X)).real).numpy()
    surf, _ = graf.af_forward(dev(s[None]), N, out="pow", layout="centered", k_begin=-N // 2, k_end=N // 2,
                              periodic=True)
    assert np.abs(surf.cpu().numpy()[0] - chi).max() <= 1e-5 * O.energy(s) ** 2


def test_periodic_frank_perfect_acf():
    N = 256
    s = frank(N)[None].astype(np.complex64)
    surf, _ = graf.af_forward(dev(s), N, out="abs", layout="raw", periodic=True)
    z = surf.cpu().numpy()[0, :, 0]                                   # zero-Doppler cut
    assert abs(z[0] - N) < 1e-4 * N and np.abs(z[1:]).max() < 1e-4 * N


def test_periodic_large_sampled_rows():
    N = 16384      # M = 16384: zero-padded global copy of s (periodic copy on the left)
    s = cg(1, N, 9)
    rows = [(-3, 3), (8190, 8194), (16380, 16384)]
    E = O.energy(s[0])
    for kb, ke in rows:
        surf, _ = graf.af_forward(dev(s), N, out="c64", layout="raw", k_begin=kb, k_end=ke, periodic=True)
        ref = O.surface(s[0], N, "c64", "raw", k_begin=kb, k_end=ke, periodic=True)
        assert np.abs(surf.cpu().numpy()[0] - ref).max() <= 1e-5 * E


# ------------------------------------------------------------------ loss and gradient
PSPECS = [
    dict(k_max=5, d_max=4, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=7, d_max=16, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=3, d_max=5, ml_k=1, ml_d=0, lambda_isl=0.5, lambda_psl=0.0, normalize=0),
    dict(k_max=64, d_max=32, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=10000, d_max=10000, ml_k=2, ml_d=3, lambda_isl=0.3, lambda_psl=0.7, temperature=0.01, normalize=1),
]


def check(s, spec_d, **kw):
    N = s.shape[1]
    spec = graf.LossSpec.from_dict(spec_d)
    loss, g, surf = graf.af_loss_grad(dev(s), N, spec, periodic=True, **kw)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(spec_d)
    for b in range(s.shape[0]):
        L_ref, g_ref, t = O.loss_and_grad(s[b], N, ospec, periodic=True)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b], L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol, (b, np.abs(g[b] - g_ref).max(), tol)
    return loss, g, surf


@pytest.mark.parametrize("si", range(len(PSPECS)))
@pytest.mark.parametrize("N", [16, 64, 256, 512])
def test_periodic_loss_grad(si, N):
    check(cg(3, N, 40 + si), PSPECS[si])


def test_periodic_paper_workload_n256():
    # the paper's §7 setting: N = 256 random-phase codes, periodic surface
    N = 256
    s = np.stack([random_phase(SplitMix64(b), N) for b in range(4)])
    check(s, dict(k_max=N, d_max=N, ml_k=0, ml_d=0, lambda_isl=0.0, lambda_psl=1.0, temperature=0.01, normalize=1))
    check(s, dict(k_max=40, d_max=20, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=0.0, normalize=1), out="pow",
          layout="centered", k_begin=-N // 2, k_end=N // 2)


def test_periodic_full_plane_closed_forms():
    N = 128
    s = cg(2, N, 77)
    loss, g, _ = graf.af_loss_grad(dev(s), N, graf.LossSpec(k_max=N, d_max=N, lambda_isl=1.0, normalize=1),
                                   periodic=True)
    assert np.abs(loss.cpu().numpy() - (N - 1)).max() < 1e-4 * N
    raw = graf.LossSpec(k_max=N, d_max=N, lambda_isl=1.0, normalize=0)
    loss, g, _ = graf.af_loss_grad(dev(s), N, raw, periodic=True)
    for b in range(2):
        E = O.energy(s[b])
        np.testing.assert_allclose(g[b].cpu().numpy(), 2 * (N - 1) * E * s[b], atol=1e-4 * 2 * (N - 1) * E)


def test_periodic_sharding_algebra():
    N = 128
    s = cg(2, N, 91)
    spec = graf.LossSpec.from_dict(PSPECS[1])
    ds = dev(s)
    L1, g1, _ = graf.af_loss_grad(ds, N, spec, periodic=True)
    for G in (2, 3):
        parts = torch.stack([graf.af_forward(ds, N, out=None, loss=spec, shard=(r, G), periodic=True)[1]
                             for r in range(G)])
        glob = graf.combine_partials(spec, parts)
        gsum = torch.zeros_like(g1)
        for r in range(G):
            Lr, gr, _ = graf.af_loss_grad(ds, N, spec, global_partials=glob, shard=(r, G), periodic=True)
            assert torch.allclose(Lr, L1, rtol=1e-6)
            gsum += gr
        assert (gsum - g1).abs().max().item() <= 1e-4 * g1.abs().max().item() + 1e-12


# ------------------------------------------------------------------ generic adjoint
@pytest.mark.parametrize("N,window", [(16, None), (64, (-7, 12)), (256, (-128, 128)), (1024, (900, 1024))])
@pytest.mark.parametrize("layout", ["raw", "centered"])
def test_periodic_backward(N, window, layout):
    B = 2
    s = cg(B, N, N + 5)
    kb, ke = window if window else (0, N)
    rows = np.arange(kb, ke)
    dA = cg(B, len(rows) * N, N + 6).reshape(B, len(rows), N)
    g = graf.af_backward(dev(s), N, dev(dA), k_begin=kb, k_end=ke, layout=layout, periodic=True).cpu().numpy()
    for b in range(B):
        G = dA[b] if layout == "raw" else np.roll(dA[b], -(N // 2), axis=1)
        ref = O.adjoint(s[b], N, G.astype(np.complex128), rows, periodic=True)
        assert np.abs(g[b] - ref).max() <= 1e-4 * np.abs(ref).max()


def test_periodic_requires_m_equal_n():
    s = dev(cg(1, 16, 1))
    with pytest.raises(graf.GrafError):
        graf.af_forward(s, 32, out="c64", periodic=True)
