"""Pins for the float64 oracle against what the paper and the mathematics fix
(task rule ③).  None of these re-types the oracle's own formula: each checks a
closed form, an invariant, an independent library routine (numpy.fft, torch
autograd), the paper's periodic Eq. 2 through the fold identity, or central
finite differences.  Golden values with citations live in tests/golden/.
"""
import json
import os

import numpy as np
import pytest
import torch

from graf_inputs import (SplitMix64, barker13, complex_gaussian, frank, lfm, p4,
                         random_phase, waveform, lfm_beta)
from oracle import graf_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rs(n, seed=0):
    return complex_gaussian(SplitMix64(seed), n).astype(np.complex128)


def full(s, M):
    n = len(s)
    return np.arange(-(n - 1), n), O.ambiguity(s, M)


def row(rows, k):
    return int(np.where(rows == k)[0][0])


# ---------------------------------------------------------------- conventions
@pytest.mark.parametrize("n,M", [(2, 2), (3, 4), (5, 8), (7, 16)])
def test_single_term_rows_fix_sign_and_delay(n, M):
    # k = N-1 keeps only n = N-1: A = s[N-1] conj(s[0]) e^{-j2pi m (N-1)/M};
    # k = -(N-1) keeps only n = 0: A = s[0] conj(s[N-1]) (north-star formula).
    s = rs(n, 1)
    rows, A = full(s, M)
    m = np.arange(M)
    np.testing.assert_allclose(A[row(rows, n - 1)],
                               s[-1] * np.conj(s[0]) * np.exp(-2j * np.pi * m * (n - 1) / M), atol=1e-14)
    np.testing.assert_allclose(A[row(rows, -(n - 1))], s[0] * np.conj(s[-1]) * np.ones(M), atol=1e-14)


def test_impulse():
    # S:L232 transferred: impulse -> A[0, m] = |s0|^2 for all m, zero elsewhere.
    s = np.array([2.0 + 1j, 0, 0, 0])
    rows, A = full(s, 8)
    assert np.allclose(A[row(rows, 0)], 5.0)
    A2 = A.copy(); A2[row(rows, 0)] = 0
    assert np.abs(A2).max() == 0


@pytest.mark.parametrize("n,M", [(13, 16), (32, 32), (20, 64), (64, 64)])
def test_matches_numpy_fft_of_lag_rows(n, M):
    # independent library routine: numpy's FFT of each zero-padded lag row.
    s = rs(n, 2)
    rows, A = full(s, M)
    for i, k in enumerate(rows):
        r = np.zeros(M, complex)
        for t in range(n):
            if 0 <= t - k < n:
                r[t % M] += s[t] * np.conj(s[t - k])
        np.testing.assert_allclose(A[i], np.fft.fft(r), atol=1e-12 * n)


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("n,M", [(16, 16), (16, 32), (13, 16), (50, 64)])
def test_origin_energy_volume_parseval_symmetry(n, M):
    s = rs(n, 3)
    E = O.energy(s)
    rows, A = full(s, M)
    assert abs(A[row(rows, 0), 0] - E) < 1e-12 * E                 # A[0,0] = E
    assert np.abs(A).max() <= E * (1 + 1e-12)                       # Cauchy-Schwarz
    np.testing.assert_allclose(np.sum(np.abs(A) ** 2), M * E ** 2, rtol=1e-12)   # volume
    for i, k in enumerate(rows):                                     # row Parseval
        lo, hi = max(0, k), min(n, n + k)
        rhs = M * np.sum(np.abs(s[lo:hi]) ** 2 * np.abs(s[lo - k:hi - k]) ** 2)
        np.testing.assert_allclose(np.sum(np.abs(A[i]) ** 2), rhs, rtol=1e-11, atol=1e-11 * E * E)
    m = np.arange(M)
    for i, k in enumerate(rows):                                     # symmetry
        j = row(rows, -k)
        np.testing.assert_allclose(np.abs(A[j][(-m) % M]), np.abs(A[i]), atol=1e-12 * E)
        np.testing.assert_allclose(A[j], np.exp(2j * np.pi * m * k / M) * np.conj(A[i][(-m) % M]),
                                   atol=1e-12 * E)


@pytest.mark.parametrize("n,M", [(8, 8), (8, 16), (17, 32)])
def test_constant_pulse_dirichlet(n, M):
    s = np.ones(n)
    rows, A = full(s, M)
    m = np.arange(1, M)
    for i, k in enumerate(rows):
        L = n - abs(k)
        assert abs(abs(A[i, 0]) - L) < 1e-12                        # |A[k,0]| = N-|k|
        np.testing.assert_allclose(np.abs(A[i, 1:]), np.abs(np.sin(np.pi * m * L / M) / np.sin(np.pi * m / M)),
                                   atol=1e-11)


def test_barker13_zero_doppler():
    with open(os.path.join(GOLDEN, "barker13.json")) as f:
        gold = json.load(f)
    s = barker13().astype(complex)
    rows, A = full(s, 16)
    cut = np.abs(A[:, 0])
    for i, k in enumerate(rows):
        assert abs(cut[i] - gold["aperiodic_zero_doppler_abs"][str(abs(int(k)))]) < 1e-12
    assert abs(cut.max() - 13) < 1e-12
    assert abs(np.sort(cut)[-2] - gold["max_sidelobe"]) < 1e-12


@pytest.mark.parametrize("n,M,beta", [(64, 64, 0.7), (64, 128, 1.9), (101, 128, 1.3)])
def test_lfm_closed_form(n, M, beta):
    s = lfm(n, beta).astype(complex)           # complex64-rounded input, promoted
    rows, A = full(s, M)
    # closed form uses the EXACT chirp; compare against |A| of the rounded input
    # through a tolerance covering the complex64 input rounding (~6e-8 * N).
    m = np.arange(M)
    for i, k in enumerate(rows):
        L = n - abs(k)
        f = beta * k / n - m / M
        with np.errstate(invalid="ignore", divide="ignore"):
            ref = np.abs(np.sin(np.pi * L * f) / np.sin(np.pi * f))
        ref = np.where(np.abs(np.sin(np.pi * f)) < 1e-15, L, ref)
        np.testing.assert_allclose(np.abs(A[i]), ref, atol=2e-6 * n)


def test_lfm_closed_form_c3_rows():
    # c3-size LFM waveform (N = M = 1024), a handful of full rows.
    s = waveform(3, 0).astype(complex)
    beta = lfm_beta(3, 0)
    n = M = 1024
    rows = np.array([-1023, -300, -1, 0, 1, 77, 512, 1023])
    A = O.ambiguity(s, M, rows)
    m = np.arange(M)
    for i, k in enumerate(rows):
        L = n - abs(k)
        f = beta * k / n - m / M
        with np.errstate(invalid="ignore", divide="ignore"):
            ref = np.abs(np.sin(np.pi * L * f) / np.sin(np.pi * f))
        ref = np.where(np.abs(np.sin(np.pi * f)) < 1e-15, L, ref)
        np.testing.assert_allclose(np.abs(A[i]), ref, atol=2e-6 * n)


@pytest.mark.parametrize("code", ["frank", "p4"])
def test_perfect_periodic_acf_via_fold(code):
    n = 64
    s = (frank(n) if code == "frank" else p4(n)).astype(complex)
    rows, A = full(s, n)
    for k in range(1, n):
        per = A[row(rows, k), 0] + A[row(rows, k - n), 0]          # fold identity
        assert abs(per) < 1e-5                                       # complex64 input rounding


@pytest.mark.parametrize("n", [4, 9, 16])
def test_fold_identity_equals_paper_eq2(n):
    # Paper Eq. 2 (periodic, e^{+j}) = aperiodic fold at mirrored Doppler.
    s = rs(n, 4)
    rows, A = full(s, n)
    X = O.periodic_ambiguity(s)
    m = np.arange(n)
    for k in range(n):
        fold = A[row(rows, k)] + (A[row(rows, k - n)] if k > 0 else 0)
        np.testing.assert_allclose(X[k], fold[(-m) % n], atol=1e-12 * O.energy(s))
    # SPEC S:L233 example on the periodic surface: all-ones N=4 -> chi[k,0] = 16
    X1 = O.periodic_ambiguity(np.ones(4))
    assert np.allclose(np.abs(X1[:, 0]) ** 2, 16)


def test_surface_layout_and_kinds():
    s = rs(6, 5)
    M = 8
    A = O.surface(s, M, "c64", "raw")
    C = O.surface(s, M, "c64", "centered")
    # centred column j holds Doppler d = j - M/2, i.e. raw bin (j - M/2) mod M
    for j in range(M):
        np.testing.assert_array_equal(C[:, j], A[:, (j - M // 2) % M])
    assert np.allclose(O.surface(s, M, "abs", "raw"), np.abs(A))
    assert np.allclose(O.surface(s, M, "pow", "raw"), np.abs(A) ** 2)
    assert np.allclose(O.surface(s, M, "c64", "raw", normalize_output=True)[5, 0], 1.0)  # A[0,0]/E
    w = O.surface(s, M, "c64", "raw", k_begin=-2, k_end=3)
    np.testing.assert_array_equal(w, A[3:8])


# ---------------------------------------------------------------- regions and losses
def test_region_cell_counts_match_configs():
    # |Omega_s| per waveform, SURVEY.md §8(a) table
    exp = {1: 8127, 2: 8384, 4: 525822}
    from graf_inputs import CONFIGS
    for c, cnt in exp.items():
        cfg = CONFIGS[c]
        spec = O.LossSpec.from_dict(cfg["loss"])
        if c == 4:
            spec.ml_d = 1
        rows, bins, mask, w = O.region(cfg["N"], cfg["M"], spec)
        assert int(mask.sum()) == cnt
    rows, bins, mask, _ = O.region(16384, 16384, O.LossSpec(k_max=16383, d_max=8192))
    assert len(rows) * len(bins) - 1 == 536854527 and mask.size - mask.sum() == 1


@pytest.mark.parametrize("n,M", [(16, 16), (12, 32), (64, 64)])
def test_full_plane_normalized_isl_is_M_minus_1_with_zero_grad(n, M):
    s = rs(n, 6)
    spec = O.LossSpec(k_max=n, d_max=M, lambda_isl=1.0, normalize=1)
    L, g, t = O.loss_and_grad(s, M, spec)
    assert abs(L - (M - 1)) < 1e-10 * M
    assert np.abs(g).max() < 1e-11 * M


@pytest.mark.parametrize("n,M", [(16, 16), (12, 32)])
def test_raw_full_plane_isl_closed_form_grad(n, M):
    s = rs(n, 7)
    E = O.energy(s)
    spec = O.LossSpec(k_max=n, d_max=M, lambda_isl=1.0, normalize=0)
    L, g, _ = O.loss_and_grad(s, M, spec)
    assert abs(L - (M - 1) * E ** 2) < 1e-11 * M * E ** 2
    np.testing.assert_allclose(g, 2 * (M - 1) * E * s, atol=1e-10 * M * E)


def test_softpsl_bounds_and_zero_temperature_limit():
    s = rs(24, 8)
    M = 32
    spec = O.LossSpec(k_max=10, d_max=6, ml_k=0, ml_d=0, lambda_isl=0, lambda_psl=1, temperature=0.01)
    t = O.loss_terms(s, M, spec)
    xmax = t["x"][t["mask"]].max()
    assert xmax <= t["lse"] <= xmax + 0.01 * np.log(t["count"]) + 1e-15
    spec.temperature = 1e-6
    assert abs(O.loss(s, M, spec) - xmax) < 1e-6 * np.log(t["count"]) + 1e-15


# ---------------------------------------------------------------- gradient
SPECS = [
    dict(k_max=5, d_max=4, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=7, d_max=16, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=3, d_max=5, ml_k=1, ml_d=0, lambda_isl=0.5, lambda_psl=0.0, normalize=0),
    dict(k_max=8, d_max=8, ml_k=0, ml_d=0, lambda_isl=0.0, lambda_psl=1.0, temperature=0.02, normalize=0),
]


def weights_for(spec, n, M, seed):
    r = SplitMix64(seed)
    wk = 0.5 + r.uniform(2 * n - 1)
    wd = 0.5 + r.uniform(M)
    return wk, wd


@pytest.mark.parametrize("si", range(len(SPECS)))
@pytest.mark.parametrize("weighted", [False, True])
def test_gradient_central_differences(si, weighted):
    n, M = 9, 16
    s = rs(n, 10 + si)
    spec = O.LossSpec(**SPECS[si])
    if weighted:
        spec.w_k, spec.w_d = weights_for(spec, n, M, 99)
    L, g, _ = O.loss_and_grad(s, M, spec)
    eps = 1e-6
    fd = np.zeros(n, complex)
    for p in range(n):
        for part, unit in ((0, 1.0), (1, 1j)):
            sp = s.copy(); sp[p] += eps * unit
            sm = s.copy(); sm[p] -= eps * unit
            d = (O.loss(sp, M, spec) - O.loss(sm, M, spec)) / (2 * eps)
            if part == 0:
                fd[p] += d
            else:
                fd[p] += 1j * d
    # dL/dRe = 2 Re g, dL/dIm = 2 Im g
    np.testing.assert_allclose(2 * g, fd, atol=1e-7 * max(1.0, np.abs(fd).max()))


def _torch_loss(st, M, spec, n):
    """Independent formulation: torch FFT of zero-padded lag rows + masks built here."""
    K = min(spec["k_max"], n - 1)
    rows = []
    for k in range(-K, K + 1):
        lo, hi = max(0, k), min(n, n + k)
        r = torch.zeros(M, dtype=torch.complex128)
        if lo < hi:
            r = torch.cat([torch.zeros(lo, dtype=torch.complex128), st[lo:hi] * torch.conj(st[lo - k:hi - k]),
                           torch.zeros(M - hi, dtype=torch.complex128)])
        rows.append(r)
    A = torch.fft.fft(torch.stack(rows), dim=1)
    chi = A.real ** 2 + A.imag ** 2
    E = torch.sum(st.real ** 2 + st.imag ** 2)
    x = chi / E ** 2 if spec["normalize"] else chi
    kk = torch.arange(-K, K + 1)[:, None]
    mm = torch.arange(M)[None, :]
    d = torch.where(mm < M // 2, mm, mm - M)
    mask = (d.abs() <= spec["d_max"]) & ~((kk.abs() <= spec["ml_k"]) & (d.abs() <= spec["ml_d"]))
    S = torch.sum(chi[mask])
    isl = S / E ** 2 if spec["normalize"] else S
    T = spec.get("temperature", 0.01)
    lse = T * torch.logsumexp(x[mask] / T, dim=0)
    return spec["lambda_isl"] * isl + spec["lambda_psl"] * lse


@pytest.mark.parametrize("si", range(len(SPECS)))
def test_gradient_matches_torch_autograd(si):
    n, M = 20, 32
    s = rs(n, 20 + si)
    spec = SPECS[si]
    L, g, _ = O.loss_and_grad(s, M, O.LossSpec(**spec))
    st = torch.tensor(s, dtype=torch.complex128, requires_grad=True)
    Lt = _torch_loss(st, M, spec, n)
    Lt.backward()
    assert abs(Lt.item() - L) < 1e-10 * max(1, abs(L))
    # torch's complex grad convention: z.grad = 2 dL/dz*  (SURVEY finding 7)
    np.testing.assert_allclose(st.grad.numpy(), 2 * g, atol=1e-10 * max(1, np.abs(g).max()))


@pytest.mark.parametrize("si", range(len(SPECS)))
def test_gradient_invariants(si):
    n, M = 24, 32
    s = rs(n, 30 + si)
    spec = O.LossSpec(**SPECS[si])
    L, g, _ = O.loss_and_grad(s, M, spec)
    sc = max(1.0, np.abs(g).max() * np.abs(s).max() * n)
    assert abs(np.vdot(g, s).imag) < 1e-11 * sc                              # global phase
    assert abs(np.sum(np.arange(n) * np.conj(g) * s).imag) < 1e-11 * sc * n  # Doppler shift
    if spec.normalize:
        assert abs(np.vdot(g, s).real) < 1e-11 * sc                         # scale invariance S:L390
    elif spec.lambda_psl == 0:
        assert abs(np.vdot(g, s).real - 2 * L) < 1e-10 * max(1, abs(L))      # Euler, degree 4


def test_adjoint_inner_product_identity():
    # A is sesquilinear, so (A(s+d) - A(s-d))/2 is its exact linearisation:
    # Re<G, dA> = Re<adjoint(G), d>.
    n, M = 11, 16
    s = rs(n, 40)
    dlt = rs(n, 41)
    rows = np.arange(-(n - 1), n)
    G = rs(len(rows) * M, 42).reshape(len(rows), M)
    lin = (O.ambiguity(s + dlt, M) - O.ambiguity(s - dlt, M)) / 2
    lhs = np.vdot(G, lin).real
    rhs = np.vdot(O.adjoint(s, M, G, rows), dlt).real
    assert abs(lhs - rhs) < 1e-11 * max(1, abs(lhs))


def test_chunked_equals_one_shot():
    n, M = 40, 64
    s = rs(n, 50)
    spec = O.LossSpec(k_max=n, d_max=M, lambda_isl=1.0, lambda_psl=1.0, temperature=0.01, normalize=1)
    L1, g1, t1 = O.loss_and_grad(s, M, spec)
    L2, g2, t2 = O.loss_and_grad_chunked(s, M, spec, chunk_rows=7, chunk_bins=13)
    assert abs(L1 - L2) < 1e-12 * abs(L1)
    np.testing.assert_allclose(g1, g2, atol=1e-13 * max(1, np.abs(g1).max()) + 1e-15)


# ---------------------------------------------------------------- periodic (the paper's Alg. 1)
# The circular surface of Eq. 2 / Alg. 1, pinned to the
# independent aperiodic path (fold identity), to Eq. 2 as printed (mirrored
# Doppler, reading R2), and by the periodic closed forms / invariants.
PSPECS = [
    dict(k_max=2, d_max=3, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=4, d_max=4, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=3, d_max=2, ml_k=1, ml_d=0, lambda_isl=0.5, lambda_psl=0.0, normalize=0),
]


@pytest.mark.parametrize("n", [4, 8, 16])
def test_periodic_surface_is_fold_and_mirrored_eq2(n):
    s = rs(n, 60)
    rows, A = full(s, n)
    P = O.ambiguity(s, n, rows=np.arange(n), periodic=True)
    X = O.periodic_ambiguity(s)
    m = np.arange(n)
    for k in range(n):
        fold = A[row(rows, k)] + (A[row(rows, k - n)] if k > 0 else 0)
        np.testing.assert_allclose(P[k], fold, atol=1e-12 * O.energy(s))
        np.testing.assert_allclose(P[k], X[k, (-m) % n], atol=1e-12 * O.energy(s))
    # negative delays are the residues: row -k == row N-k
    Pn = O.ambiguity(s, n, rows=np.arange(-(n - 1), 0), periodic=True)
    np.testing.assert_allclose(Pn, P[1:], atol=1e-12 * O.energy(s))
    # volume: sum |A_per|^2 = N E^2
    assert abs(np.sum(np.abs(P) ** 2) - n * O.energy(s) ** 2) < 1e-10 * n * O.energy(s) ** 2


@pytest.mark.parametrize("code", ["frank", "p4"])
def test_periodic_perfect_acf(code):
    n = 64
    s = (frank(n) if code == "frank" else p4(n)).astype(complex)
    P = O.ambiguity(s, n, rows=np.arange(n), bins=np.array([0]), periodic=True)
    assert abs(P[0, 0] - n) < 1e-5 and np.abs(P[1:, 0]).max() < 1e-5


@pytest.mark.parametrize("n", [8, 9, 16])
def test_periodic_full_plane_closed_forms(n):
    s = rs(n, 61)
    E = O.energy(s)
    spec = O.LossSpec(k_max=n, d_max=n, lambda_isl=1.0, normalize=1)
    L, g, t = O.loss_and_grad(s, n, spec, periodic=True)
    assert t["count"] == n * n - 1
    assert abs(L - (n - 1)) < 1e-10 * n and np.abs(g).max() < 1e-11 * n
    spec.normalize = 0
    L, g, _ = O.loss_and_grad(s, n, spec, periodic=True)
    assert abs(L - (n - 1) * E ** 2) < 1e-11 * n * E ** 2
    np.testing.assert_allclose(g, 2 * (n - 1) * E * s, atol=1e-10 * n * E)


@pytest.mark.parametrize("si", range(len(PSPECS)))
@pytest.mark.parametrize("n", [8, 9])
def test_periodic_gradient_central_differences(si, n):
    s = rs(n, 70 + si)
    spec = O.LossSpec(**PSPECS[si])
    L, g, _ = O.loss_and_grad(s, n, spec, periodic=True)
    eps = 1e-6
    fd = np.zeros(n, complex)
    for p in range(n):
        for unit in (1.0, 1j):
            sp = s.copy(); sp[p] += eps * unit
            sm = s.copy(); sm[p] -= eps * unit
            d = (O.loss(sp, n, spec, periodic=True) - O.loss(sm, n, spec, periodic=True)) / (2 * eps)
            fd[p] += d * (1.0 if unit == 1.0 else 1j)
    np.testing.assert_allclose(2 * g, fd, atol=1e-7 * max(1.0, np.abs(fd).max()))
    sc = max(1.0, np.abs(g).max() * np.abs(s).max() * n)
    assert abs(np.vdot(g, s).imag) < 1e-11 * sc
    if spec.normalize:
        assert abs(np.vdot(g, s).real) < 1e-11 * sc


def test_periodic_adjoint_inner_product_identity():
    n = 12
    s, dlt = rs(n, 80), rs(n, 81)
    rows = np.arange(-5, 7)
    G = rs(len(rows) * n, 82).reshape(len(rows), n)
    lin = (O.ambiguity(s + dlt, n, rows, periodic=True) - O.ambiguity(s - dlt, n, rows, periodic=True)) / 2
    lhs = np.vdot(G, lin).real
    rhs = np.vdot(O.adjoint(s, n, G, rows, periodic=True), dlt).real
    assert abs(lhs - rhs) < 1e-11 * max(1, abs(lhs))


# ---------------------------------------------------------------- the paper's §7 workload (NEXT-2)
def _fd(fun, x, eps=1e-6, complex_input=True):
    g = np.zeros(len(x), complex if complex_input else float)
    for p in range(len(x)):
        units = (1.0, 1j) if complex_input else (1.0,)
        for u in units:
            xp = x.copy(); xp[p] += eps * u
            xm = x.copy(); xm[p] -= eps * u
            g[p] += (fun(xp) - fun(xm)) / (2 * eps) * (1.0 if u == 1.0 else 1j)
    return g


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("normalize", [1, 0])
def test_hard_psl_value_and_subgradient(periodic, normalize):
    n = 8
    s = rs(n, 90 + normalize)
    spec = O.LossSpec(k_max=3, d_max=3, ml_k=0, ml_d=0, normalize=normalize)
    psl, g, (k, m) = O.hard_psl_and_grad(s, n, spec, periodic)
    t = O.loss_terms(s, n, spec, periodic)
    assert psl == t["x"][t["mask"]].max()                      # Eq. 19: the max over Omega_s
    # away from ties the max is differentiable: central differences of PSL
    fd = _fd(lambda z: O.hard_psl_and_grad(z, n, spec, periodic)[0], s)
    np.testing.assert_allclose(2 * g, fd, atol=1e-6 * max(1.0, np.abs(fd).max()))


def test_hard_psl_mirrored_tie_and_barker():
    # |A[-k,-m]| = |A[k,m]|: the max is attained twice; the subgradient of either cell is the same
    s = rs(10, 95)
    spec = O.LossSpec(k_max=9, d_max=8, normalize=1)
    psl, g, (k, m) = O.hard_psl_and_grad(s, 16, spec)
    assert k <= 0                                              # row-major first of the mirrored pair
    # Barker-13 zero-Doppler: max aperiodic sidelobe 1 -> PSL = 1/169 on the delay axis (golden)
    b = barker13().astype(complex)
    psl, _, (k, m) = O.hard_psl_and_grad(b, 16, O.LossSpec(k_max=12, d_max=0, normalize=1))
    assert abs(psl - 1 / 169) < 1e-15 and m == 0


def test_spectral_variance_closed_forms_and_gradient():
    n = 16
    # impulse: flat spectrum -> SV = 0 with zero gradient at the minimum
    d = np.zeros(n, complex); d[3] = 1.0
    sv, g = O.spectral_variance_and_grad(d)
    assert abs(sv) < 1e-30 and np.abs(g).max() < 1e-15
    # single tone: all power in one bin -> p = e_j, sum (p - 1/N)^2 = (N-1)/N, so the
    # population variance is (N-1)/N^2 and the unbiased one 1/N
    tone = np.exp(2j * np.pi * 5 * np.arange(n) / n)
    assert abs(O.spectral_variance_and_grad(tone)[0] - (n - 1) / n ** 2) < 1e-15
    assert abs(O.spectral_variance_and_grad(tone, ddof=1)[0] - 1.0 / n) < 1e-14
    # SPEC.md L331 worked example: all-ones N = 4 -> p = [1,0,0,0] -> 3/16 (population)
    assert abs(O.spectral_variance_and_grad(np.ones(4, complex))[0] - 0.1875) < 1e-16
    # matches numpy.fft + numpy's variance (both ddof) on random input; central differences
    s = rs(n, 96)
    S = np.fft.fft(s)
    p = np.abs(S) ** 2 / np.sum(np.abs(S) ** 2)
    for ddof in (0, 1):
        sv, g = O.spectral_variance_and_grad(s, ddof=ddof)
        assert abs(sv - np.var(p, ddof=ddof)) < 1e-15
        fd = _fd(lambda z: O.spectral_variance_and_grad(z, ddof=ddof)[0], s)
        np.testing.assert_allclose(2 * g, fd, atol=1e-7 * np.abs(fd).max())
        assert abs(np.vdot(g, s)) < 1e-12                       # scale- and phase-invariant


def test_adam_matches_torch_and_first_step():
    r = SplitMix64(97)
    th = r.uniform(12) * 6.0
    grads = [r.uniform(12) - 0.5 for _ in range(5)]
    p = torch.tensor(th, dtype=torch.float64, requires_grad=True)
    opt = torch.optim.Adam([p], lr=0.01)
    m = np.zeros(12); v = np.zeros(12); x = th.copy()
    for t, gr in enumerate(grads, start=1):
        opt.zero_grad(); p.grad = torch.tensor(gr); opt.step()
        x, m, v = O.adam_step(x, m, v, gr, t)
        np.testing.assert_allclose(x, p.detach().numpy(), rtol=0, atol=1e-14)
    x1, _, _ = O.adam_step(th, np.zeros(12), np.zeros(12), grads[0], 1)
    np.testing.assert_allclose(x1, th - 0.01 * np.sign(grads[0]), atol=1e-9)   # |step| = lr at t = 1


def test_lpi_phase_gradient_central_differences():
    n = 8
    th = SplitMix64(98).uniform(n) * 2 * np.pi
    spec = O.LossSpec(k_max=n, d_max=n, normalize=1)
    L, gth, parts = O.lpi_loss_and_grad(th, spec, lam=0.5)
    fd = _fd(lambda z: O.lpi_loss_and_grad(z, spec, lam=0.5)[0], th, complex_input=False)
    np.testing.assert_allclose(gth, fd.real, atol=1e-6 * max(1.0, np.abs(fd).max()))
    assert abs(L - (parts["psl"] + 0.5 * 2000.0 * parts["sv"])) < 1e-15 * max(1, L)


# ---------------------------------------------------------------- match loss (NEXT-3)
@pytest.mark.parametrize("periodic,layout", [(False, "centered"), (False, "raw"), (True, "centered")])
def test_match_loss_pins(periodic, layout):
    n, M = 8, 8
    s = rs(n, 120)
    spec = O.LossSpec(k_max=3, d_max=3, ml_k=0, ml_d=1, normalize=1)
    kb = 0 if periodic else -(n - 1)
    rows_w = n if periodic else 2 * n - 1
    surf = O.surface(s, M, "pow", layout, k_begin=kb, k_end=kb + rows_w, periodic=periodic) / O.energy(s) ** 2
    # target = the surface itself: zero loss, zero gradient
    L, g = O.match_loss_and_grad(s, M, spec, surf, kb, layout, periodic)
    assert L < 1e-28 and np.abs(g).max() < 1e-14
    # target = 0: L = sum over Omega of x^2 (cell count from the region)
    L0, _ = O.match_loss_and_grad(s, M, spec, np.zeros_like(surf), kb, layout, periodic)
    t = O.loss_terms(s, M, spec, periodic)
    assert abs(L0 - np.sum(t["x"][t["mask"]] ** 2)) < 1e-14 * max(1, L0)
    # central differences on a random target
    tgt = SplitMix64(121).uniform(surf.size).reshape(surf.shape) * 0.2
    L, g = O.match_loss_and_grad(s, M, spec, tgt, kb, layout, periodic)
    fd = _fd(lambda z: O.match_loss_and_grad(z, M, spec, tgt, kb, layout, periodic)[0], s)
    np.testing.assert_allclose(2 * g, fd, atol=1e-6 * max(1.0, np.abs(fd).max()))
    assert abs(np.vdot(g, s).imag) < 1e-10 * max(1, np.abs(g).max())


# ---------------------------------------------------------------- cross-ambiguity (NEXT-4)
def test_cross_reduces_to_auto_and_swap_identity():
    n, M = 9, 16
    s = rs(n, 130)
    rows = np.arange(-(n - 1), n)
    np.testing.assert_allclose(O.cross_ambiguity(s, s, M), O.ambiguity(s, M), atol=1e-13)
    spec = O.LossSpec(k_max=5, d_max=6, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=0.5, temperature=0.05,
                      normalize=1)
    L, g1, g2 = O.cross_loss_and_grad(s, s, M, spec)
    La, ga, _ = O.loss_and_grad(s, M, spec)
    assert abs(L - La) < 1e-13 * abs(La)
    np.testing.assert_allclose(g1 + g2, ga, atol=1e-12 * np.abs(ga).max())
    # X_21[-k, m] = W^{-mk} conj(X_12[k, -m]);  Cauchy-Schwarz |X| <= sqrt(E1 E2)
    s2 = rs(n, 131)
    X12 = O.cross_ambiguity(s, s2, M)
    X21 = O.cross_ambiguity(s2, s, M)
    m = np.arange(M)
    for i, k in enumerate(rows):
        ph = np.exp(2j * np.pi * ((m * k) % M) / M)
        np.testing.assert_allclose(X21[row(rows, -k)], ph * np.conj(X12[i, (-m) % M]), atol=1e-12)
    assert np.abs(X12).max() <= np.sqrt(O.energy(s) * O.energy(s2)) * (1 + 1e-12)


@pytest.mark.parametrize("normalize", [1, 0])
def test_cross_gradients_central_differences(normalize):
    n, M = 7, 8
    s1, s2 = rs(n, 132), rs(n, 133)
    spec = O.LossSpec(k_max=4, d_max=3, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.7, temperature=0.05 if
                      normalize else 2.0, normalize=normalize)
    L, g1, g2 = O.cross_loss_and_grad(s1, s2, M, spec)
    fd1 = _fd(lambda z: O.cross_loss_and_grad(z, s2, M, spec)[0], s1)
    fd2 = _fd(lambda z: O.cross_loss_and_grad(s1, z, M, spec)[0], s2)
    np.testing.assert_allclose(2 * g1, fd1, atol=1e-6 * max(1.0, np.abs(fd1).max()))
    np.testing.assert_allclose(2 * g2, fd2, atol=1e-6 * max(1.0, np.abs(fd2).max()))


def test_cross_adjoint_inner_product_identity():
    n, M = 10, 16
    s1, s2, d1, d2 = rs(n, 134), rs(n, 135), rs(n, 136), rs(n, 137)
    rows = np.arange(-(n - 1), n)
    G = rs(len(rows) * M, 138).reshape(len(rows), M)
    # X is bilinear in (s1, conj s2): the exact linearisation in (d1, d2)
    lin = (O.cross_ambiguity(s1 + d1, s2 + d2, M) - O.cross_ambiguity(s1 - d1, s2 - d2, M)) / 2
    g1, g2 = O.cross_adjoint(s1, s2, M, G, rows)
    assert abs(np.vdot(G, lin).real - (np.vdot(g1, d1).real + np.vdot(g2, d2).real)) < 1e-10


# ---------------------------------------------------------------- mainlobe width (NEXT-3)
@pytest.mark.parametrize("periodic", [False, True])
def test_mainlobe_width_pins(periodic):
    n = 8
    s = rs(n, 140)
    E = O.energy(s)
    W, g = O.mainlobe_width_and_grad(s, gamma=0.3 / E ** 2, periodic=periodic)
    fd = _fd(lambda z: O.mainlobe_width_and_grad(z, 0.3 / E ** 2, periodic)[0], s)
    np.testing.assert_allclose(2 * g, fd, atol=1e-7 * max(1.0, np.abs(fd).max()))
    # gamma -> infinity: the hard -3 dB count sum_{chi(tau,0) > E^2/2} |tau|
    rows = O.delay_rows(n, periodic=periodic)
    cut = np.abs(O.ambiguity(s, n, rows=rows, bins=np.array([0]), periodic=periodic)[:, 0]) ** 2
    hard = float(np.sum(np.abs(rows)[cut > 0.5 * E ** 2]))
    Wh, _ = O.mainlobe_width_and_grad(s, gamma=1e6 / E ** 2, periodic=periodic)
    assert abs(Wh - hard) < 1e-6
    # constant pulse: chi(tau,0) = (N-|tau|)^2 > N^2/2 iff |tau| < N(1 - 1/sqrt 2)
    one = np.ones(16, complex)
    Wc, gc = O.mainlobe_width_and_grad(one, gamma=1e3, periodic=False)
    t = np.arange(-15, 16)
    assert abs(Wc - float(np.sum(np.abs(t)[(16 - np.abs(t)) ** 2 > 128]))) < 1e-9


def test_c5_golden_pinned_by_invariants():
    """tests/golden/c5_w0_softpsl.npz (scripts/make_c5_golden.py, oracle only) against what
    the mathematics fixes at N = M = 16384: it was computed from config 5's waveform 0;
    full-plane normalised ISL = M - 1 (volume identity); max x <= softPSL <=
    max x + T log|Omega| (|Omega| = (2N-1)M - 1); and the gradient invariants of an
    |A|-based normalised loss: Im<g,s> = 0 (global phase), Re<g,s> = 0 (scale),
    Im sum_n n conj(g[n]) s[n] = 0 (linear phase = Doppler shift)."""
    import hashlib
    import os
    from graf_inputs import config_waveforms
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c5_w0_softpsl.npz"))
    s = config_waveforms(5, batch=1)[0]
    assert str(z["s_sha256"]) == hashlib.sha256(np.ascontiguousarray(s).tobytes()).hexdigest()
    N = M = 16384
    assert int(z["count"]) == (2 * N - 1) * M - 1
    assert abs(float(z["isl"]) - (M - 1)) < 1e-9 * M
    c, lse, T = float(z["c"]), float(z["lse"]), float(z["temperature"])
    assert c <= lse <= c + T * np.log(float(z["count"]))
    g = z["grad"]
    sd = s.astype(np.complex128)
    scale = np.sum(np.abs(g) * np.abs(sd))
    n = np.arange(N)
    assert abs(np.vdot(g, sd).imag) < 1e-12 * scale
    assert abs(np.vdot(g, sd).real) < 1e-11 * scale
    assert abs(np.sum(n * np.conj(g) * sd).imag) < 1e-12 * np.sum(n * np.abs(g) * np.abs(sd))
