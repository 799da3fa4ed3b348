"""Config 3 at full scale: O(N)-per-row pins on ALL 1024 GPU surfaces (SURVEY.md §8(c)
"what pins each part").  The direct oracle costs 2e9 complex MACs per
waveform, so it runs on a subset elsewhere (test_gpu_parity.py); here every waveform of
the bench's full-surface call (|A| fp32, centred Doppler) is checked against what the
mathematics fixes at any size:

  * A[0,0] = E                                   (Cauchy-Schwarz maximum)
  * row Parseval  sum_m |A[k,m]|^2 = M sum_n |s[n]|^2 |s[n-k]|^2   (every row, every waveform)
  * volume        sum_{k,m} |A|^2 = M E^2        (M >= N)
  * symmetry      |A[-k,-m]| = |A[k,m]|
  * LFM third     |A[k,m]| = |sin(pi L f) / sin(pi f)|, f = beta k/N - m/M, L = N - |k|
                  (closed form of the chirp's lag products; sampled rows, all bins)
  * Frank/P4 third: perfect periodic autocorrelation through the fold identity
                  |A[k,0] + A[k-N,0]| = 0 for k = 1..N-1 (the paper's periodic Eq. 2 at
                  zero Doppler; complex surface of those waveforms)

Tolerances follow from the surface bound |dA| <= delta = 1e-5 E per cell (north star):
a sum of |A|^2 over a set C moves by at most 2 delta sum_C |A| + |C| delta^2.
"""
import numpy as np
import pytest
import torch

from graf_inputs import CONFIGS, config_waveforms, lfm_beta

pytestmark = pytest.mark.gpu

graf = pytest.importorskip("paper_2506_22935_b200")


@pytest.fixture(scope="module")
def c3():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS[3]
    s = config_waveforms(3)                          # all 1024 waveforms
    ds = torch.from_numpy(s).cuda()
    surf, _ = graf.af_forward(ds, cfg["M"], out="abs", layout="centered")   # [1024, 2047, 1024] fp32
    torch.cuda.synchronize()
    yield cfg, s, ds, surf
    del surf
    torch.cuda.empty_cache()


def test_c3_origin_is_energy_all_waveforms(c3):
    cfg, s, ds, surf = c3
    N, M = cfg["N"], cfg["M"]
    E = (ds.abs().double() ** 2).sum(1)
    a00 = surf[:, N - 1, M // 2].double()
    assert ((a00 - E).abs() <= 1e-5 * E).all()
    assert (surf.amax(dim=(1, 2)).double() <= E * (1 + 1e-5)).all()     # |A| <= E everywhere


def test_c3_row_parseval_and_volume_all_waveforms(c3):
    cfg, s, ds, surf = c3
    N, M = cfg["N"], cfg["M"]
    p = ds.abs().double() ** 2                                          # |s[n]|^2, [B, N]
    # sum_n |s[n]|^2 |s[n-k]|^2 for every k (delay row index k + N - 1): direct O(N^2) on device
    B = p.shape[0]
    rhs = torch.empty((B, 2 * N - 1), dtype=torch.float64, device="cuda")
    for k in range(-(N - 1), N):
        lo, hi = max(0, k), min(N, N + k)
        rhs[:, k + N - 1] = (p[:, lo:hi] * p[:, lo - k:hi - k]).sum(1)
    rhs = M * rhs
    E = p.sum(1)
    delta = 1e-5 * E[:, None]
    worst = 0.0
    for b0 in range(0, B, 128):
        a = surf[b0:b0 + 128].double()
        row = (a * a).sum(2)                                            # [b, 2N-1]
        bound = 2 * delta[b0:b0 + 128] * a.sum(2) + M * delta[b0:b0 + 128] ** 2
        err = (row - rhs[b0:b0 + 128]).abs()
        worst = max(worst, (err / bound).max().item())
        assert (err <= bound).all(), (b0, (err / bound).max().item())
        vol = row.sum(1)
        vb = (2 * delta[b0:b0 + 128, 0] * a.sum((1, 2)) + (2 * N - 1) * M * delta[b0:b0 + 128, 0] ** 2)
        assert ((vol - M * E[b0:b0 + 128] ** 2).abs() <= vb).all()
    print(f"PARITY c3 row Parseval worst err/bound {worst:.3e}")


def test_c3_mirror_symmetry_all_waveforms(c3):
    cfg, s, ds, surf = c3
    N, M = cfg["N"], cfg["M"]
    E = (ds.abs().double() ** 2).sum(1)
    for b0 in range(0, s.shape[0], 128):
        a = surf[b0:b0 + 128]
        # centred column j <-> d = j - M/2; -d -> column M - j (mod M) ; rows k <-> -k: flip
        mir = torch.roll(torch.flip(a, dims=(1, 2)), shifts=1, dims=2)
        diff = (a - mir).abs().amax(dim=(1, 2)).double()
        assert (diff <= 2e-5 * E[b0:b0 + 128]).all()


def test_c3_lfm_closed_form_sampled_rows(c3):
    cfg, s, ds, surf = c3
    N, M = cfg["N"], cfg["M"]
    rows = np.array([-(N - 1), -700, -257, -31, -2, -1, 0, 1, 2, 64, 333, 512, 1000, N - 1])
    m = np.arange(M)
    col = (m + M // 2) % M                        # centred column of raw bin m
    worst = 0.0
    for b in range(0, s.shape[0], 3):             # family 0: LFM
        beta = lfm_beta(3, b)
        E = float(np.sum(np.abs(s[b].astype(np.complex128)) ** 2))
        got = surf[b, torch.from_numpy(rows + N - 1).cuda()][:, torch.from_numpy(col).cuda()].double().cpu().numpy()
        for i, k in enumerate(rows):
            L = N - abs(int(k))
            f = beta * k / N - m / M
            sf = np.sin(np.pi * f)
            with np.errstate(divide="ignore", invalid="ignore"):
                ref = np.where(np.abs(sf) < 1e-12, float(L), np.abs(np.sin(np.pi * L * f) / sf))
            e = np.abs(got[i] - ref).max()
            worst = max(worst, e / E)
            assert e <= 1e-5 * E, (b, k, e)
    print(f"PARITY c3 LFM closed form worst err/E {worst:.3e}")


def test_c3_frank_p4_perfect_periodic_acf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cfg = CONFIGS[3]
    N, M = cfg["N"], cfg["M"]
    idx = np.arange(1, cfg["B"], 3)               # family 1: Frank / P4
    s = config_waveforms(3)[idx]
    worst = 0.0
    for b0 in range(0, len(idx), 64):
        ds = torch.from_numpy(s[b0:b0 + 64]).cuda()
        surf, _ = graf.af_forward(ds, M, out="c64", layout="raw")        # [b, 2N-1, M]
        z = surf[:, :, 0]                                                 # zero Doppler
        per = z[:, N:] + z[:, :N - 1]                                     # A[k,0] + A[k-N,0], k = 1..N-1
        E = (ds.abs().double() ** 2).sum(1)
        r = (per.abs().double().amax(1) / E)
        worst = max(worst, r.max().item())
        assert (r <= 1e-5).all()
        del surf
    print(f"PARITY c3 Frank/P4 periodic ACF worst |A_per|/E {worst:.3e}")
