"""GRAF ambiguity-function ORACLE (float64, CPU) — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import or run anything under `oracle/`.  The product
path (`paper_2506_22935_b200/`) never imports it and shares no code with it:
the only module both sides use is `graf_inputs` (seeded waveform draws, no AF
arithmetic).

What it computes (citations: P:Lnnn = /root/reference/PAPER.md line nnn,
S:Lnnn = SPEC.md line nnn; readings R# = DESIGN.md §2 / SURVEY.md §8(c)):

  A[k,m] = sum_n s[n] * conj(s[n-k]) * exp(-2j*pi*m*n/M),
           k in [-(N-1), N-1], m in [0, M)                     (north star;
           aperiodic form of Eq. 2 P:L121 / Eq. 7, reading R1-R4)

written out as the plain definition: the lag-product matrix R[k,n] =
s[n]*conj(s[n-k]) (Eqs. 8-10, aperiodic: zero outside 0<=n-k<N)
times the DFT matrix W[n,m] = exp(-2j*pi*((m*n) mod M)/M) (Eq. 11, P:L197-201,
the "FFT over the time axis" written as its defining sum; a matrix product is
the library primitive used for that sum).  There is NO FFT anywhere in this
file.  Phases are reduced on exact integers ((m*n) mod M) before the
exponential, so no phase error accumulates.

Losses and gradient follow SURVEY.md §8(c) steps 4-8:
  chi = |A|^2 (Eq. 12);  x = chi/E^2 if normalized (Eqs. 19-20 divide by
  chi(0,0) = E^2, reading R6) else chi
  S = sum_{Omega} w*chi;  LSE = c + T*log sum_{Omega} exp((x-c)/T), c = max x
  L = lambda_isl*(S/E^2 | S) + lambda_psl*LSE              (Eq. 23 weighting)
  f' = dL/dx = lambda_isl*w + lambda_psl*exp((x-LSE)/T) on Omega
  G = dL/dA* = f'*A/E^2 (normalized) | f'*A (raw)          (Eq. 14)
  H[k,n] = sum_m G[k,m]*exp(+2j*pi*m*n/M)                  ("IFFT (linear)", P:L230;
                                                             S:L143 op_fft_rows adjoint)
  g[p] = sum_k H[k,p]*s[p-k] + sum_k conj(H[k,p+k])*s[p+k]  (Eq. 15, "element-wise
         - (2/E^3)*(sum_{Omega} f'*chi)*s   [normalized only]  multiplication gradient" P:L231)

g is the Wirtinger cotangent dL/ds* (P:L219), so
dL/dRe s = 2*Re g and dL/dIm s = 2*Im g.

Parity pins: every function here is pinned by tests/test_oracle_pins.py against
closed forms, invariants, brute force, numpy.fft, central finite differences
and torch autograd (DESIGN.md §4 lists which pin covers which function).  No
function is "parity unpinned".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "LossSpec", "energy", "delay_rows", "centred_bins", "dft_matrix",
    "lag_products", "ambiguity", "region", "loss_terms", "loss",
    "loss_and_grad", "adjoint", "correlate", "surface", "loss_and_grad_chunked",
    "periodic_ambiguity", "hard_psl_and_grad", "spectral_variance_and_grad", "phase_grad",
    "adam_step", "lpi_loss_and_grad", "match_loss_and_grad", "cross_lag_products", "cross_ambiguity",
    "cross_correlate", "cross_adjoint", "cross_loss_and_grad", "mainlobe_width_and_grad",
]


# ---------------------------------------------------------------------------
# index conventions
# ---------------------------------------------------------------------------
def delay_rows(n: int, k_max: Optional[int] = None, periodic: bool = False) -> np.ndarray:
    """Delays k = -K..K with K = min(k_max, N-1) (north star: k in +-(N-1)).
    periodic (the paper's circular Eq. 2): the distinct residues k mod N
    with circular distance <= k_max, as k in (-N/2, N/2] (K = min(k_max, N//2))."""
    if periodic:
        K = n // 2 if k_max is None else min(k_max, n // 2)
        lo = -K + 1 if 2 * K == n else -K
        return np.arange(lo, K + 1)
    K = n - 1 if k_max is None else min(k_max, n - 1)
    return np.arange(-K, K + 1)


def centred(m: np.ndarray, M: int) -> np.ndarray:
    """Centred Doppler index d in [-M/2, M/2): d = m for m < M/2 else m - M
    (Alg. 1 step 5 fftshift; reading R5)."""
    m = np.asarray(m)
    return np.where(m < M // 2, m, m - M)


def centred_bins(M: int, d_max: Optional[int] = None) -> np.ndarray:
    """Raw Doppler bins m whose centred index satisfies |d| <= d_max."""
    m = np.arange(M)
    if d_max is None:
        return m
    return m[np.abs(centred(m, M)) <= d_max]


def energy(s: np.ndarray) -> float:
    """E = sum_n |s[n]|^2 (= chi(0,0)^(1/2))."""
    s = np.asarray(s, dtype=np.complex128)
    return float(np.sum(s.real ** 2 + s.imag ** 2))


# ---------------------------------------------------------------------------
# Step 3: the surface, as the plain definition (matrix form of the DFT sum)
# ---------------------------------------------------------------------------
def dft_matrix(n: int, M: int, bins: np.ndarray, sign: int = -1) -> np.ndarray:
    """W[n, j] = exp(sign*2j*pi*((bins[j]*n) mod M)/M), n = 0..N-1."""
    nn = np.arange(n, dtype=np.int64)[:, None]
    mm = np.asarray(bins, dtype=np.int64)[None, :]
    ph = (nn * mm) % M
    return np.exp(sign * 2j * np.pi * ph / M)


def lag_products(s: np.ndarray, rows: np.ndarray, periodic: bool = False) -> np.ndarray:
    """R[i, n] = s[n]*conj(s[n-k_i]) when 0 <= n-k_i < N, else 0 (Eqs. 8-10,
    aperiodic reading R1).  rows: integer delays k.
    periodic: R[i, n] = s[n]*conj(s[(n-k_i) mod N]) for every n (Eqs. 8-10 exactly as
    printed: the circulant shift matrix S[k,n] = s[(n-k) mod N])."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    if periodic:
        return np.stack([s * np.conj(s[(np.arange(n) - int(k)) % n]) for k in rows]) if len(rows) else \
            np.zeros((0, n), dtype=np.complex128)
    R = np.zeros((len(rows), n), dtype=np.complex128)
    for i, k in enumerate(rows):
        k = int(k)
        lo, hi = max(0, k), min(n, n + k)
        if lo < hi:
            R[i, lo:hi] = s[lo:hi] * np.conj(s[lo - k:hi - k])
    return R


def ambiguity(s: np.ndarray, M: int, rows: Optional[np.ndarray] = None,
              bins: Optional[np.ndarray] = None, periodic: bool = False) -> np.ndarray:
    """A[rows, bins] (complex128), direct O(N*|rows|*|bins|) evaluation.
    periodic: the circular lag products (the paper's Eq. 2 with the FFT's e^{-j},
    reading R2; M = N in the paper)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows = delay_rows(n, periodic=periodic) if rows is None else np.asarray(rows)
    bins = np.arange(M) if bins is None else np.asarray(bins)
    return lag_products(s, rows, periodic) @ dft_matrix(n, M, bins)


def surface(s: np.ndarray, M: int, kind: str = "c64", layout: str = "centered",
            normalize_output: bool = False, k_begin: Optional[int] = None,
            k_end: Optional[int] = None, periodic: bool = False) -> np.ndarray:
    """The forward-surface output the ABI writes: rows k_begin..k_end-1 (row
    index k - k_begin), Doppler raw m or centred j = d + M/2 (Alg. 1 step 5,
    P:L252).  kind: 'c64' -> A, 'abs' -> |A|, 'pow' -> |A|^2 (Alg. 1 step 4,
    P:L251).  normalize_output divides A by E (Eq. 17 analogue: max chi = E^2,
    P:L265-268, reading R6)."""
    n = len(s)
    if periodic:   # Alg. 1: rows k = 0..N-1, or any window of <= N delays
        kb = 0 if k_begin is None else k_begin
    else:
        kb = -(n - 1) if k_begin is None else k_begin
    ke = n if k_end is None else k_end
    A = ambiguity(s, M, rows=np.arange(kb, ke), periodic=periodic)
    if normalize_output:
        A = A / energy(s)
    if layout == "centered":
        A = np.roll(A, M // 2, axis=1)   # column j holds bin m = (j - M/2) mod M
    if kind == "c64":
        return A
    if kind == "abs":
        return np.abs(A)
    if kind == "pow":
        return np.abs(A) ** 2
    raise ValueError(kind)


# ---------------------------------------------------------------------------
# Loss region and losses (steps 4-5)
# ---------------------------------------------------------------------------
@dataclass
class LossSpec:
    """Sidelobe region Omega_s (never defined by the paper; reading R7):
    |k| <= k_max and |d| <= d_max, minus the mainlobe |k| <= ml_k and
    |d| <= ml_d.  Optional separable weights w_k[k+N-1], w_d[d+M/2] (R8)."""
    k_max: int
    d_max: int
    ml_k: int = 0
    ml_d: int = 0
    lambda_isl: float = 1.0
    lambda_psl: float = 0.0
    temperature: float = 0.01
    normalize: int = 1
    w_k: Optional[np.ndarray] = field(default=None, repr=False)
    w_d: Optional[np.ndarray] = field(default=None, repr=False)

    @classmethod
    def from_dict(cls, d: dict) -> "LossSpec":
        return cls(**{k: v for k, v in d.items() if k in cls.__dataclass_fields__})


def region(n: int, M: int, spec: LossSpec, periodic: bool = False):
    """rows (k), bins (m), mask [rows, bins] (bool), weights [rows, bins].
    periodic: rows are the residues with circular delay distance <= k_max."""
    rows = delay_rows(n, spec.k_max, periodic)
    bins = centred_bins(M, spec.d_max)
    d = centred(bins, M)
    mainlobe = (np.abs(rows)[:, None] <= spec.ml_k) & (np.abs(d)[None, :] <= spec.ml_d)
    mask = ~mainlobe
    wk = np.ones(len(rows)) if spec.w_k is None else np.asarray(spec.w_k, np.float64)[rows + n - 1]
    wd = np.ones(len(bins)) if spec.w_d is None else np.asarray(spec.w_d, np.float64)[d + M // 2]
    w = wk[:, None] * wd[None, :]
    return rows, bins, mask, w


def loss_terms(s: np.ndarray, M: int, spec: LossSpec, periodic: bool = False) -> dict:
    """All step 3-5 quantities for one waveform (dict of numpy values)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows, bins, mask, w = region(n, M, spec, periodic)
    if not mask.any():
        raise ValueError("empty sidelobe region (S:L302)")
    E = energy(s)
    A = ambiguity(s, M, rows, bins, periodic)
    chi = A.real ** 2 + A.imag ** 2
    x = chi / E ** 2 if spec.normalize else chi
    S = float(np.sum(w[mask] * chi[mask]))
    T = spec.temperature
    xm = x[mask]
    c = float(np.max(xm))
    Z = float(np.sum(np.exp((xm - c) / T)))
    lse = c + T * np.log(Z)
    isl = S / E ** 2 if spec.normalize else S
    L = spec.lambda_isl * isl + spec.lambda_psl * lse
    return dict(E=E, A=A, chi=chi, x=x, rows=rows, bins=bins, mask=mask, w=w,
                S=S, isl=isl, c=c, Z=Z, lse=lse, loss=L, count=int(mask.sum()))


def loss(s: np.ndarray, M: int, spec: LossSpec, periodic: bool = False) -> float:
    return loss_terms(s, M, spec, periodic)["loss"]


# ---------------------------------------------------------------------------
# Steps 6-8: the Wirtinger adjoint
# ---------------------------------------------------------------------------
def correlate(s: np.ndarray, H: np.ndarray, rows: np.ndarray, periodic: bool = False) -> np.ndarray:
    """Step 8 without the normalization term:
    g[p] = sum_k H[k,p]*s[p-k] + sum_k conj(H[k,p+k])*s[p+k], valid indices only
    (adjoint of R[k,n] = s[n]*conj(s[n-k]) w.r.t. s*, Eq. 15).
    periodic: every index taken mod N (adjoint of the circulant lag products)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    g = np.zeros(n, dtype=np.complex128)
    if periodic:
        idx = np.arange(n)
        for i, k in enumerate(rows):
            k = int(k)
            g += H[i] * s[(idx - k) % n]                      # term 1: p = n
            np.add.at(g, (idx - k) % n, np.conj(H[i]) * s)    # term 2: p = (n - k) mod N
        return g
    for i, k in enumerate(rows):
        k = int(k)
        lo, hi = max(0, k), min(n, n + k)      # valid n (= p for term 1)
        if lo >= hi:
            continue
        # term 1: p = n, uses s[p-k]
        g[lo:hi] += H[i, lo:hi] * s[lo - k:hi - k]
        # term 2: p = n - k, uses conj(H[k, p+k]) * s[p+k]
        g[lo - k:hi - k] += np.conj(H[i, lo:hi]) * s[lo:hi]
    return g


def adjoint(s: np.ndarray, M: int, G: np.ndarray, rows: np.ndarray,
            bins: Optional[np.ndarray] = None, periodic: bool = False) -> np.ndarray:
    """Generic backward (graf_af_backward): given G = dL/dA* on rows x bins,
    return dL/ds* = steps 7-8 (no normalization term: A itself does not
    depend on E)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    bins = np.arange(M) if bins is None else np.asarray(bins)
    H = np.asarray(G, dtype=np.complex128) @ dft_matrix(n, M, bins, sign=+1).T
    return correlate(s, H, rows, periodic)


def loss_and_grad(s: np.ndarray, M: int, spec: LossSpec, periodic: bool = False):
    """(L, g = dL/ds*, terms) for one waveform."""
    t = loss_terms(s, M, spec, periodic)
    s = np.asarray(s, dtype=np.complex128)
    E, A, chi, x, mask, w = t["E"], t["A"], t["chi"], t["x"], t["mask"], t["w"]
    T = spec.temperature
    fp = np.zeros_like(chi)
    fp[mask] = spec.lambda_isl * w[mask] + spec.lambda_psl * np.exp((x[mask] - t["lse"]) / T)
    G = fp * A / E ** 2 if spec.normalize else fp * A
    g = adjoint(s, M, G, t["rows"], t["bins"], periodic)
    if spec.normalize:
        g = g - (2.0 / E ** 3) * float(np.sum(fp[mask] * chi[mask])) * s
    t["fprime"] = fp
    t["sigma_g"] = (2.0 / E ** 3) * float(np.sum(np.abs(fp[mask]) * chi[mask])) * float(np.max(np.abs(s))) \
        if spec.normalize else 0.0
    return t["loss"], g, t


def loss_and_grad_chunked(s: np.ndarray, M: int, spec: LossSpec, chunk_rows: int = 512,
                          chunk_bins: int = 2048, threads_note: str = ""):
    """Same quantities as loss_and_grad, for waveforms whose full surface does
    not fit in memory (c5: 32767 x 16384 cells).  The row/bin chunking only
    regroups independent dot products and exact partial sums (S, max, Z are
    combined exactly); every A[k,m] is still the direct sum.  Two sweeps:
    (1) S, c, Z over Omega; (2) recompute A, f', H and the correlation."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows_all, bins, mask_all, w_all = region(n, M, spec)
    E = energy(s)
    T = spec.temperature
    S, c, Z, cnt = 0.0, -np.inf, 0.0, 0
    # the DFT-matrix blocks are the same for every row chunk: built once (same values)
    cache = {}

    def W(b0, sign=-1):
        key = (b0, sign)
        if key not in cache:
            cache[key] = dft_matrix(n, M, bins[b0:b0 + chunk_bins], sign=sign)
        return cache[key]

    # sweep 1
    for r0 in range(0, len(rows_all), chunk_rows):
        rows = rows_all[r0:r0 + chunk_rows]
        Rm = lag_products(s, rows)
        for b0 in range(0, len(bins), chunk_bins):
            A = Rm @ W(b0)
            chi = A.real ** 2 + A.imag ** 2
            x = chi / E ** 2 if spec.normalize else chi
            msk = mask_all[r0:r0 + chunk_rows, b0:b0 + chunk_bins]
            w = w_all[r0:r0 + chunk_rows, b0:b0 + chunk_bins]
            S += float(np.sum(w[msk] * chi[msk]))
            cnt += int(msk.sum())
            if msk.any():
                cm = float(np.max(x[msk]))
                if cm > c:
                    Z = Z * np.exp((c - cm) / T)
                    c = cm
                Z += float(np.sum(np.exp((x[msk] - c) / T)))
    lse = c + T * np.log(Z)
    isl = S / E ** 2 if spec.normalize else S
    L = spec.lambda_isl * isl + spec.lambda_psl * lse
    # sweep 2
    g = np.zeros(n, dtype=np.complex128)
    fchi = 0.0
    afchi = 0.0
    for r0 in range(0, len(rows_all), chunk_rows):
        rows = rows_all[r0:r0 + chunk_rows]
        Rm = lag_products(s, rows)
        H = np.zeros((len(rows), n), dtype=np.complex128)
        for b0 in range(0, len(bins), chunk_bins):
            A = Rm @ W(b0)
            chi = A.real ** 2 + A.imag ** 2
            x = chi / E ** 2 if spec.normalize else chi
            msk = mask_all[r0:r0 + chunk_rows, b0:b0 + chunk_bins]
            w = w_all[r0:r0 + chunk_rows, b0:b0 + chunk_bins]
            fp = np.where(msk, spec.lambda_isl * w + spec.lambda_psl * np.exp((x - lse) / T), 0.0)
            fchi += float(np.sum(fp * chi))
            afchi += float(np.sum(np.abs(fp) * chi))
            G = fp * A / E ** 2 if spec.normalize else fp * A
            H += G @ W(b0, +1).T
        g += correlate(s, H, rows)
    if spec.normalize:
        g = g - (2.0 / E ** 3) * fchi * s
    sigma_g = (2.0 / E ** 3) * afchi * float(np.max(np.abs(s))) if spec.normalize else 0.0
    return L, g, dict(E=E, S=S, isl=isl, c=c, Z=Z, lse=lse, loss=L, count=cnt, sigma_g=sigma_g)


# ---------------------------------------------------------------------------
# The paper's own periodic surface (Eq. 2), used by the fold-identity pin
# ---------------------------------------------------------------------------
def periodic_ambiguity(s: np.ndarray) -> np.ndarray:
    """X[k,m] = sum_n s[n]*conj(s[(n-k) mod N])*exp(+2j*pi*m*n/N), k,m in [0,N)
    — Eq. 2 inside the |.|^2 exactly as printed (periodic, e^{+j}, M = N)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    R = np.stack([s * np.conj(np.roll(s, k)) for k in range(n)])
    return R @ dft_matrix(n, n, np.arange(n), sign=+1)


# ---------------------------------------------------------------------------
# The paper's §7 workload: hard PSL with its argmax
# subgradient (Eq. 19), spectral variance, the Eq. 26
# loss L = PSL + lambda*alpha*SV on phase-coded waveforms
# s = exp(j*theta), and the Adam update.
# ---------------------------------------------------------------------------
def hard_psl_and_grad(s: np.ndarray, M: int, spec: LossSpec, periodic: bool = False):
    """PSL = max_{Omega_s} x (x = chi/E^2 normalized | chi raw) and its subgradient
    dPSL/ds* at the argmax cell (Eq. 19; ties -> lowest row-major index over
    (delay k ascending, raw Doppler bin m ascending), reading R23).  Returns
    (psl, g, (k, m))."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows, bins, mask, _ = region(n, M, spec, periodic)
    E = energy(s)
    A = ambiguity(s, M, rows, bins, periodic)
    chi = A.real ** 2 + A.imag ** 2
    x = chi / E ** 2 if spec.normalize else chi
    # row-major order over (k ascending, m ascending): sort the bins
    order = np.argsort(bins, kind="stable")
    xs = np.where(mask, x, -np.inf)[:, order]
    flat = int(np.argmax(xs))                     # first occurrence = lowest index
    i, jj = divmod(flat, len(bins))
    j = int(order[jj])
    psl = float(x[i, j])
    G = np.zeros_like(A)
    G[i, j] = A[i, j] / E ** 2 if spec.normalize else A[i, j]   # d x/d A* at the cell
    g = adjoint(s, M, G, rows, bins, periodic)
    if spec.normalize:
        g = g - (2.0 / E ** 3) * chi[i, j] * s
    return psl, g, (int(rows[i]), int(bins[j]))


def spectral_variance_and_grad(s: np.ndarray, ddof: int = 0):
    """SV = var{|F s|^2 / sum |F s|^2} over the N DFT bins, F = length-N DFT
    written as its matrix; and dSV/ds* (chain rule through p_j = |S_j|^2 / P).
    var = sum (p - mean p)^2 / (N - ddof): ddof = 0 is the population variance that
    SPEC.md L328 fixes (all-ones N = 4 -> 3/16; reading R22), ddof = 1 the
    unbiased estimator (PyTorch's var default)."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    F = dft_matrix(n, n, np.arange(n)).T          # S_j = sum_n s_n exp(-2 pi i j n / N)
    S = F @ s
    pw = S.real ** 2 + S.imag ** 2
    P = float(np.sum(pw))
    p = pw / P
    mean = float(np.mean(p))
    sv = float(np.sum((p - mean) ** 2) / (n - ddof))
    c = 2.0 * (p - mean) / (n - ddof)             # dSV/dp_j
    dS = (c - float(np.sum(c * p))) * S / P       # dSV/dS_j*
    g = np.conj(F).T @ dS                         # adjoint of S = F s
    return sv, g


def phase_grad(s: np.ndarray, g: np.ndarray) -> np.ndarray:
    """dL/dtheta for s = exp(j*theta) and g = dL/ds*: 2 Re(conj(g) * j s) = -2 Im(s conj(g))."""
    return -2.0 * np.imag(np.asarray(s) * np.conj(np.asarray(g)))


def adam_step(theta, m, v, grad, t: int, lr: float = 0.01, beta1: float = 0.9,
              beta2: float = 0.999, eps: float = 1e-8):
    """One Adam update (Kingma & Ba, Alg. 1; P:L425 'Adam optimizer with learning
    rate 0.01'), step t >= 1.  Returns (theta, m, v)."""
    m = beta1 * m + (1.0 - beta1) * grad
    v = beta2 * v + (1.0 - beta2) * grad * grad
    mh = m / (1.0 - beta1 ** t)
    vh = v / (1.0 - beta2 ** t)
    return theta - lr * mh / (np.sqrt(vh) + eps), m, v


def lpi_loss_and_grad(theta: np.ndarray, spec: LossSpec, lam: float, alpha: float = 2000.0,
                      periodic: bool = True):
    """Eq. 26: L = PSL + lam*alpha*SV on s = exp(j*theta) (M = N), and dL/dtheta."""
    theta = np.asarray(theta, dtype=np.float64)
    s = np.exp(1j * theta)
    n = s.shape[0]
    psl, gp, _ = hard_psl_and_grad(s, n, spec, periodic)
    sv, gs = spectral_variance_and_grad(s)
    L = psl + lam * alpha * sv
    return L, phase_grad(s, gp + lam * alpha * gs), dict(psl=psl, sv=sv)


# ---------------------------------------------------------------------------
# Match loss: L_match = ||x - x_target||_F^2 over the
# sidelobe region Omega_s (reading R24: the same region as ISL/PSL; x = chi/E^2
# normalized | chi raw), the target laid out like the surface window
# (rows k_begin..k_end-1, Doppler raw or centred).
# ---------------------------------------------------------------------------
def match_loss_and_grad(s: np.ndarray, M: int, spec: LossSpec, target: np.ndarray, k_begin: int,
                        layout: str = "centered", periodic: bool = False):
    """(L_match, g = dL_match/ds*) with f' = dL/dx = 2 (x - t) on Omega_s."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows, bins, mask, _ = region(n, M, spec, periodic)
    E = energy(s)
    A = ambiguity(s, M, rows, bins, periodic)
    chi = A.real ** 2 + A.imag ** 2
    x = chi / E ** 2 if spec.normalize else chi
    tgt = np.asarray(target, dtype=np.float64)
    ri = rows - k_begin
    if periodic:
        ri = ri % n if tgt.shape[0] == n else ri
    ci = (bins + M // 2) % M if layout == "centered" else bins
    t = tgt[ri[:, None], ci[None, :]]
    diff = np.where(mask, x - t, 0.0)
    L = float(np.sum(diff ** 2))
    fp = 2.0 * diff
    G = fp * A / E ** 2 if spec.normalize else fp * A
    g = adjoint(s, M, G, rows, bins, periodic)
    if spec.normalize:
        g = g - (2.0 / E ** 3) * float(np.sum(fp * chi)) * s
    return L, g


# ---------------------------------------------------------------------------
# Cross-ambiguity (P:L546 MIMO):
#   X[k,m] = sum_n s1[n] conj(s2[n-k]) exp(-2j pi m n / M)   (aperiodic, k in +-(N-1))
# normalised by E1*E2 (reading R25: |X| <= sqrt(E1 E2), equal to E^2 when s1 = s2).
# Losses over Omega_s as for the auto surface; no row folding (no symmetry).
# ---------------------------------------------------------------------------
def cross_lag_products(s1: np.ndarray, s2: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """R[i, n] = s1[n] conj(s2[n-k_i]) for 0 <= n-k_i < N, else 0."""
    s1 = np.asarray(s1, dtype=np.complex128)
    s2 = np.asarray(s2, dtype=np.complex128)
    n = s1.shape[0]
    R = np.zeros((len(rows), n), dtype=np.complex128)
    for i, k in enumerate(rows):
        k = int(k)
        lo, hi = max(0, k), min(n, n + k)
        if lo < hi:
            R[i, lo:hi] = s1[lo:hi] * np.conj(s2[lo - k:hi - k])
    return R


def cross_ambiguity(s1, s2, M: int, rows=None, bins=None) -> np.ndarray:
    n = len(s1)
    rows = delay_rows(n) if rows is None else np.asarray(rows)
    bins = np.arange(M) if bins is None else np.asarray(bins)
    return cross_lag_products(s1, s2, rows) @ dft_matrix(n, M, bins)


def cross_correlate(s1, s2, H: np.ndarray, rows: np.ndarray):
    """(g1, g2): g1[p] = sum_k H[k,p] s2[p-k] (dX*-side w.r.t. s1*), g2[p] = sum_k conj(H[k,p+k]) s1[p+k]."""
    s1 = np.asarray(s1, dtype=np.complex128)
    s2 = np.asarray(s2, dtype=np.complex128)
    n = s1.shape[0]
    g1 = np.zeros(n, dtype=np.complex128)
    g2 = np.zeros(n, dtype=np.complex128)
    for i, k in enumerate(rows):
        k = int(k)
        lo, hi = max(0, k), min(n, n + k)
        if lo >= hi:
            continue
        g1[lo:hi] += H[i, lo:hi] * s2[lo - k:hi - k]
        g2[lo - k:hi - k] += np.conj(H[i, lo:hi]) * s1[lo:hi]
    return g1, g2


def cross_adjoint(s1, s2, M: int, G: np.ndarray, rows: np.ndarray, bins=None):
    n = len(s1)
    bins = np.arange(M) if bins is None else np.asarray(bins)
    H = np.asarray(G, dtype=np.complex128) @ dft_matrix(n, M, bins, sign=+1).T
    return cross_correlate(s1, s2, H, rows)


def cross_loss_and_grad(s1, s2, M: int, spec: LossSpec):
    """(L, g1 = dL/ds1*, g2 = dL/ds2*) for L = lambda_isl ISL + lambda_psl softPSL on X."""
    s1 = np.asarray(s1, dtype=np.complex128)
    s2 = np.asarray(s2, dtype=np.complex128)
    n = s1.shape[0]
    rows, bins, mask, w = region(n, M, spec)
    E1, E2 = energy(s1), energy(s2)
    A = cross_ambiguity(s1, s2, M, rows, bins)
    chi = A.real ** 2 + A.imag ** 2
    x = chi / (E1 * E2) if spec.normalize else chi
    S = float(np.sum(w[mask] * chi[mask]))
    T = spec.temperature
    c = float(np.max(x[mask]))
    lse = c + T * np.log(float(np.sum(np.exp((x[mask] - c) / T))))
    L = spec.lambda_isl * (S / (E1 * E2) if spec.normalize else S) + spec.lambda_psl * lse
    fp = np.zeros_like(chi)
    fp[mask] = spec.lambda_isl * w[mask] + spec.lambda_psl * np.exp((x[mask] - lse) / T)
    G = fp * A / (E1 * E2) if spec.normalize else fp * A
    g1, g2 = cross_adjoint(s1, s2, M, G, rows, bins)
    if spec.normalize:
        F = float(np.sum(fp * chi))
        g1 = g1 - F / (E1 ** 2 * E2) * s1
        g2 = g2 - F / (E1 * E2 ** 2) * s2
    return L, g1, g2


# ---------------------------------------------------------------------------
# Mainlobe width: the -3 dB delay width through
# the differentiable sigmoid threshold
#   W = sum_tau |tau| * sigma(gamma * (chi(tau, 0) - 0.5 chi(0, 0)))
# over every delay of the zero-Doppler cut (aperiodic tau in +-(N-1), or the
# periodic residues in (-N/2, N/2]), chi raw (reading R26).
# ---------------------------------------------------------------------------
def mainlobe_width_and_grad(s: np.ndarray, gamma: float, periodic: bool = False):
    """(W, dW/ds*) with dW/dchi(tau,0) = |tau| gamma sigma'(u) and the chi(0,0) = E^2 term."""
    s = np.asarray(s, dtype=np.complex128)
    n = s.shape[0]
    rows = delay_rows(n, periodic=periodic)
    A = ambiguity(s, n if periodic else max(2, n), rows=rows, bins=np.array([0]), periodic=periodic)[:, 0]
    chi = A.real ** 2 + A.imag ** 2
    E = energy(s)
    u = gamma * (chi - 0.5 * E ** 2)
    sig = 0.5 * (1.0 + np.tanh(0.5 * u))                # logistic sigma, overflow-free
    W = float(np.sum(np.abs(rows) * sig))
    dsig = sig * (1.0 - sig)
    c = np.abs(rows) * gamma * dsig                     # dW/dchi(tau, 0)
    G = (c * A)[:, None]                                # dW/dA*(tau, 0) = c * A
    g = adjoint(s, n if periodic else max(2, n), G, rows, np.array([0]), periodic)
    g = g - 0.5 * float(np.sum(c)) * 2.0 * E * s        # through chi(0,0) = E^2: d(E^2)/ds* = 2 E s
    return W, g
