"""Seeded random sweep of the parameter space against the float64 oracle: random
(B, N, M), delay windows, Doppler layouts, masks, mainlobes, loss weights and
temperatures, aperiodic and periodic (Eqs. 8-15, 19-20).
Each case is drawn from a SplitMix64 stream keyed by its index, so a failure is
reproduced by its id alone.  Tolerances as in test_gpu_parity.py (reading R18).
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


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def randint(r, lo, hi):
    """uniform integer in [lo, hi]"""
    return lo + int(r.uniform(1)[0] * (hi - lo + 1)) % (hi - lo + 1)


def draw_shape(r):
    periodic = r.uniform(1)[0] < 0.25
    if periodic:
        N = 1 << randint(r, 1, 10)
        return N, N, True
    N = randint(r, 1, 700)
    M0 = 1 << max(1, int(np.ceil(np.log2(max(N, 2)))))
    M = min(M0 << randint(r, 0, 2), 4096)
    return N, M, False


def draw_spec(r, N, M):
    ml_k, ml_d = randint(r, 0, 2), randint(r, 0, 2)
    ml_k = min(ml_k, N - 1)
    ml_d = min(ml_d, M // 2 - 1)
    k_max = randint(r, ml_k, N)
    d_max = randint(r, ml_d + 1, M // 2)          # the region keeps cells (0, +-d_max) at least
    lam_psl = [0.0, 0.0, 1.0, 0.5][randint(r, 0, 3)]
    lam_isl = 1.0 if lam_psl == 0.0 else [0.0, 0.3, 1.0][randint(r, 0, 2)]
    T = [0.02, 0.05, 0.1][randint(r, 0, 2)]
    normalize = 1 if (lam_psl > 0 or r.uniform(1)[0] < 0.7) else 0
    return dict(k_max=k_max, d_max=d_max, ml_k=ml_k, ml_d=ml_d, lambda_isl=lam_isl, lambda_psl=lam_psl,
                temperature=T, normalize=normalize)


@pytest.mark.parametrize("case", range(128))
def test_fuzz_loss_grad(case):
    r = SplitMix64(0xF0220000 + case)
    N, M, periodic = draw_shape(r)
    B = randint(r, 1, 3)
    spec = draw_spec(r, N, M)
    s = np.stack([complex_gaussian(SplitMix64(case * 100 + b), N) for b in range(B)])
    want_surface = r.uniform(1)[0] < 0.3
    kw = dict(periodic=periodic)
    if want_surface:
        kb = randint(r, -(N - 1), N - 1)
        ke = randint(r, kb + 1, min(N, kb + N) if periodic else N)   # periodic: at most N distinct delays
        kw.update(out="c64", layout=["raw", "centered"][randint(r, 0, 1)], k_begin=kb, k_end=ke)
    loss, g, surf = graf.af_loss_grad(dev(s), M, graf.LossSpec.from_dict(spec), **kw)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(spec)
    for b in range(B):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec, periodic=periodic)
        ctx = (case, N, M, periodic, spec, b)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref) + 1e-30, (ctx, loss[b], L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol + 1e-30, (ctx, np.abs(g[b] - g_ref).max(), tol)
        if want_surface:
            ref = O.surface(s[b], M, "c64", kw["layout"], k_begin=kw["k_begin"], k_end=kw["k_end"],
                            periodic=periodic)
            assert np.abs(surf[b].cpu().numpy() - ref).max() <= 1e-5 * O.energy(s[b]), ctx


@pytest.mark.parametrize("case", range(48))
def test_fuzz_backward(case):
    r = SplitMix64(0xBAC40000 + case)
    N, M, periodic = draw_shape(r)
    kb = randint(r, -(N - 1), N - 1)
    ke = randint(r, kb + 1, min(N, kb + 64, kb + N if periodic else N))
    layout = ["raw", "centered"][randint(r, 0, 1)]
    s = complex_gaussian(SplitMix64(case + 7), N)[None]
    rows = np.arange(kb, ke)
    dA = complex_gaussian(SplitMix64(case + 9), len(rows) * M).reshape(1, len(rows), M)
    g = graf.af_backward(dev(s), M, dev(dA), k_begin=kb, k_end=ke, layout=layout,
                         periodic=periodic).cpu().numpy()[0]
    G = dA[0] if layout == "raw" else np.roll(dA[0], -(M // 2), axis=1)
    ref = O.adjoint(s[0], M, G.astype(np.complex128), rows, periodic=periodic)
    assert np.abs(g - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-30), (case, N, M, periodic, kb, ke, layout)


@pytest.mark.parametrize("case", range(32))
def test_fuzz_large_m_narrow_band(case):
    # M = 2048 ... 8192 (the sizes that compile the band-edge and zero-padded paths), N up
    # to M, loss bands mostly narrower than M/16 bins, every loss kind of the fused kernels
    r = SplitMix64(0xBA4D0000 + case)
    M = 2048 << randint(r, 0, 2)
    N = randint(r, 2, min(M, 1200))
    T = M // 16
    d_max = randint(r, 0, T - 1) if r.uniform(1)[0] < 0.7 else randint(r, T, M // 2)
    ml_d = min(randint(r, 0, 2), d_max)
    if d_max == ml_d:
        ml_d = max(0, d_max - 1)
    k_max = randint(r, 1, min(N - 1, 200)) if N > 1 else 1
    lam_psl = [0.0, 1.0][randint(r, 0, 1)]
    spec = dict(k_max=k_max, d_max=d_max, ml_k=0, ml_d=ml_d, lambda_isl=1.0, lambda_psl=lam_psl,
                temperature=[0.02, 0.05][randint(r, 0, 1)], normalize=1)
    s = np.stack([complex_gaussian(SplitMix64(case * 77 + b), N) for b in range(2)])
    loss, g, _ = graf.af_loss_grad(dev(s), M, graf.LossSpec.from_dict(spec))
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(spec)
    for b in range(2):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        ctx = (case, N, M, spec, b)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref) + 1e-30, (ctx, loss[b], L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol + 1e-30, (ctx, np.abs(g[b] - g_ref).max(), tol)


@pytest.mark.parametrize("case", range(32))
def test_fuzz_tmem_sizes(case):
    """M = 8192 and 16384 (the tensor-memory accumulator kernels; M = 8192 with the unpadded
    staged s): random N <= 1100, full or partial delay extents, mainlobe blocks, ISL / soft-PSL
    / both, raw or normalised, surfaces on random windows, and the backward on a random
    window, against the oracle (plain-relative gradient gate)."""
    r = SplitMix64(0x7E3E0000 + case)
    M = [8192, 16384][randint(r, 0, 1)]
    N = randint(r, 2, 1100)
    full = r.uniform(1)[0] < 0.4
    ml_k, ml_d = randint(r, 0, 2), randint(r, 0, 2)
    ml_k = min(ml_k, N - 1)
    k_max = N - 1 if full else randint(r, max(ml_k, 1), N - 1)
    d_max = M // 2 if full else randint(r, ml_d + 1, 600)
    lam_psl = [0.0, 1.0, 0.5][randint(r, 0, 2)]
    lam_isl = 1.0 if lam_psl == 0.0 else [0.0, 1.0][randint(r, 0, 1)]
    normalize = 1 if (lam_psl > 0 or r.uniform(1)[0] < 0.7) else 0
    spec = dict(k_max=k_max, d_max=d_max, ml_k=ml_k, ml_d=ml_d, lambda_isl=lam_isl, lambda_psl=lam_psl,
                temperature=[0.02, 0.05][randint(r, 0, 1)], normalize=normalize)
    B = randint(r, 1, 2)
    s = np.stack([complex_gaussian(SplitMix64(case * 131 + b), N) for b in range(B)])
    kb = randint(r, -(N - 1), N - 1)
    ke = randint(r, kb + 1, min(N, kb + 24))
    kw = dict(out="c64", layout=["raw", "centered"][randint(r, 0, 1)], k_begin=kb, k_end=ke) \
        if r.uniform(1)[0] < 0.4 else {}
    loss, g, surf = graf.af_loss_grad(dev(s), M, graf.LossSpec.from_dict(spec), **kw)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(spec)
    for b in range(B):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        ctx = (case, N, M, spec, b)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref) + 1e-30, (ctx, loss[b], L_ref)
        assert np.abs(g[b] - g_ref).max() <= grad_tol(g_ref, t["sigma_g"]) + 1e-30, (ctx, np.abs(g[b] - g_ref).max())
        if kw:
            ref = O.surface(s[b], M, "c64", kw["layout"], k_begin=kb, k_end=ke)
            assert np.abs(surf[b].cpu().numpy() - ref).max() <= 1e-5 * O.energy(s[b]), ctx
    rows = np.arange(kb, ke)
    dA = complex_gaussian(SplitMix64(case + 11), len(rows) * M).reshape(1, len(rows), M)
    gb = graf.af_backward(dev(s[:1]), M, dev(dA), k_begin=kb, k_end=ke, layout="raw").cpu().numpy()[0]
    ref = O.adjoint(s[0], M, dA[0].astype(np.complex128), rows)
    assert np.abs(gb - ref).max() <= 1e-4 * np.abs(ref).max(), (case, N, M, kb, ke)
