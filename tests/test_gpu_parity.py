"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on
the same seeded inputs (task rule ③).

Tolerances (BASELINE.json north_star, SURVEY.md §8(c) reading R18):
  surface  max|A_gpu - A_ref| <= 1e-5 * E_b
  loss     |L_gpu - L_ref|    <= 1e-4 * |L_ref|
  gradient max|g_gpu - g_ref| <= 1e-4 * max|g_ref|   (tests/gradtol.py; sigma_g only when g == 0 exactly)
sigma_g = (2/E^3)|sum f' chi| max|s| is the size of the normalisation term that
cancels in normalised losses (0 in raw mode: plain relative error).
"""
import numpy as np
import pytest
import torch

from graf_inputs import CONFIGS, SplitMix64, complex_gaussian, config_waveforms, random_phase
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
SURF_CASES = [(1, 2), (1, 16), (3, 4), (5, 8), (13, 16), (7, 32), (64, 64), (37, 64), (100, 128),
              (256, 256), (200, 256), (300, 512), (512, 512), (1000, 1024), (1024, 1024)]


@pytest.mark.parametrize("N,M", SURF_CASES)
def test_surface_full_plane_c64(N, M):
    B = 3
    s = cg(B, N, N + M)
    surf, _ = graf.af_forward(dev(s), M, out="c64", layout="centered")
    got = surf.cpu().numpy()
    for b in range(B):
        ref = O.surface(s[b], M, "c64", "centered")
        assert np.abs(got[b] - ref).max() <= 1e-5 * O.energy(s[b])


@pytest.mark.parametrize("kind", ["abs", "pow", "c64"])
@pytest.mark.parametrize("layout", ["raw", "centered"])
@pytest.mark.parametrize("window", [None, (-5, 9), (3, 40), (-40, -2), (0, 1)])
@pytest.mark.parametrize("norm", [False, True])
def test_surface_kinds_layouts_windows(kind, layout, window, norm):
    N, M = 50, 64
    s = cg(2, N, 7)
    kb, ke = window if window else (None, None)
    surf, _ = graf.af_forward(dev(s), M, out=kind, layout=layout, k_begin=kb, k_end=ke, normalize_output=norm)
    got = surf.cpu().numpy()
    for b in range(2):
        E = O.energy(s[b])
        ref = O.surface(s[b], M, kind, layout, norm, kb, ke)
        scale = E if kind != "pow" else E * E
        if norm:
            scale = 1.0
        assert np.abs(got[b] - ref).max() <= 1e-5 * scale


@pytest.mark.parametrize("N,M", [(2048, 2048), (1500, 2048), (4096, 4096), (4096, 8192), (16384, 16384),
                                 (9000, 16384)])
def test_surface_large_sampled_rows(N, M):
    # full rows at sampled delays (the oracle computes one row in O(N*M))
    B = 1
    s = random_phase(SplitMix64(N), N)[None]
    rows = np.array([-(N - 1), -N // 3, -1, 0, 1, 2, N // 2 + 1, N - 2, N - 1])
    E = O.energy(s[0])
    for k in rows:
        surf, _ = graf.af_forward(dev(s), M, out="c64", layout="raw", k_begin=int(k), k_end=int(k) + 1)
        ref = O.ambiguity(s[0], M, rows=np.array([k]))
        assert np.abs(surf.cpu().numpy()[0] - ref).max() <= 1e-5 * E, k


def test_c3_surface_families_vs_oracle_subset():
    cfg = CONFIGS[3]
    s = config_waveforms(3, batch=6)
    surf, _ = graf.af_forward(dev(s), cfg["M"], out="abs", layout="centered")
    got = surf.cpu().numpy()
    for b in range(6):
        ref = O.surface(s[b], cfg["M"], "abs", "centered")
        assert np.abs(got[b] - ref).max() <= 1e-5 * O.energy(s[b])


# ------------------------------------------------------------------ loss and gradient
def check_loss_grad(s, M, spec_d, **kw):
    spec = graf.LossSpec.from_dict(spec_d)
    loss, g, surf = graf.af_loss_grad(dev(s), M, spec, **kw)
    loss = loss.cpu().numpy()
    g = g.cpu().numpy()
    ospec = O.LossSpec.from_dict(spec_d)
    for b in range(s.shape[0]):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b], L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        err = np.abs(g[b] - g_ref).max()
        assert err <= tol, (b, err, tol, np.abs(g_ref).max())
    return loss, g, surf


def test_c1_surface_isl_grad_normalized_and_raw():
    cfg = CONFIGS[1]
    s = config_waveforms(1)
    loss, g, surf = check_loss_grad(s, cfg["M"], cfg["loss"], out="c64", layout="centered")
    assert abs(loss[0] - 63) < 1e-4 * 63            # volume identity: ISL = M - 1
    ref = O.surface(s[0], cfg["M"], "c64", "centered")
    assert np.abs(surf.cpu().numpy()[0] - ref).max() <= 1e-5 * O.energy(s[0])
    raw = dict(cfg["loss"], normalize=0)
    loss, g, _ = check_loss_grad(s, cfg["M"], raw, out="c64", layout="centered")
    E = O.energy(s[0])
    np.testing.assert_allclose(g[0], 2 * 63 * E * s[0], atol=1e-4 * 2 * 63 * E)


def test_c2_full_batch():
    cfg = CONFIGS[2]
    s = config_waveforms(2)
    check_loss_grad(s, cfg["M"], cfg["loss"])


@pytest.mark.parametrize("normalize", [1, 0])
def test_c3_subset_surface_and_full_plane_isl(normalize):
    cfg = CONFIGS[3]
    s = config_waveforms(3, batch=3, start=3)   # LFM, P4, QPSK
    spec = dict(cfg["loss"], normalize=normalize)
    loss, g, surf = check_loss_grad(s, cfg["M"], spec, out="abs", layout="centered")
    for b in range(3):
        ref = O.surface(s[b], cfg["M"], "abs", "centered")
        assert np.abs(surf.cpu().numpy()[b] - ref).max() <= 1e-5 * O.energy(s[b])


def test_c4_subset():
    cfg = CONFIGS[4]
    s = config_waveforms(4, batch=2)
    check_loss_grad(s, cfg["M"], cfg["loss"])


@pytest.mark.parametrize("N,M", [(512, 512), (1024, 2048)])
def test_c5_shape_full_plane_softpsl_centred(N, M):
    # c5's loss (full-plane ISL + soft-PSL T=0.01, centred fp32 path) at sizes
    # the oracle finishes in seconds.
    s = np.stack([random_phase(SplitMix64(5_000_000 + b), N) for b in range(2)])
    spec = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    check_loss_grad(s, M, spec)


@pytest.mark.parametrize("N,M", [(256, 256), (1024, 1024)])
def test_full_plane_softpsl_single_pass_and_fallback(N, M):
    # the optimistic single pass (reading R13) and its per-waveform fallback: a random
    # code is inside the validity rule, an LFM chirp's ridge (x ~ 1) is outside it; a
    # mixed batch must match the oracle on both
    from graf_inputs import lfm
    s = np.stack([random_phase(SplitMix64(7_000_000), N), lfm(N, 1.0), random_phase(SplitMix64(7_000_001), N)])
    spec = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    check_loss_grad(s.astype(np.complex64), M, spec)


SPECS = [
    dict(k_max=5, d_max=4, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1),
    dict(k_max=7, d_max=16, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1),
    dict(k_max=3, d_max=5, ml_k=1, ml_d=0, lambda_isl=0.5, lambda_psl=0.0, normalize=0),
    # raw-mode soft-PSL: T must sit on the scale of raw chi (~E^2), else the
    # softmax exponent (x - LSE)/T carries fp32 error eps*x/T (R19)
    dict(k_max=60, d_max=60, ml_k=0, ml_d=0, lambda_isl=0.0, lambda_psl=1.0, temperature=2000.0, normalize=0),
    dict(k_max=1000, d_max=1000, ml_k=2, ml_d=3, lambda_isl=0.3, lambda_psl=0.7, temperature=0.01, normalize=1),
]


@pytest.mark.parametrize("si", range(len(SPECS)))
@pytest.mark.parametrize("N,M", [(9, 16), (33, 64), (100, 256), (257, 1024)])
def test_specs_ragged(si, N, M):
    s = cg(3, N, si * 10 + N)
    check_loss_grad(s, M, SPECS[si])


def test_symmetric_weights():
    N, M = 40, 64
    r = SplitMix64(11)
    wk = 0.5 + r.uniform(N)
    wk = np.concatenate([wk[:0:-1], wk]).astype(np.float32)        # symmetric in k
    wd_half = 0.5 + r.uniform(M // 2 + 1)
    d = np.arange(-M // 2, M // 2)
    wd = wd_half[np.abs(d)].astype(np.float32)                      # symmetric in d
    spec = dict(k_max=20, d_max=12, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=0.5, temperature=0.05, normalize=1)
    s = cg(2, N, 3)
    gs = graf.LossSpec.from_dict(spec)
    gs.w_k, gs.w_d = dev(wk), dev(wd)
    loss, g, _ = graf.af_loss_grad(dev(s), M, gs)
    os_ = O.LossSpec.from_dict(spec)
    os_.w_k, os_.w_d = wk.astype(np.float64), wd.astype(np.float64)
    for b in range(2):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, os_)
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= grad_tol(g_ref, t["sigma_g"])


# ------------------------------------------------------------------ forward partials, sharding algebra
@pytest.mark.parametrize("si", [0, 1, 4])
def test_forward_partials_and_delay_sharding_algebra(si):
    N, M = 120, 128
    s = cg(2, N, 77 + si)
    spec = graf.LossSpec.from_dict(SPECS[si])
    ds = dev(s)
    L1, g1, _ = graf.af_loss_grad(ds, M, spec)
    for G in (2, 3, 5):
        parts = torch.stack([graf.af_forward(ds, M, out=None, loss=spec, shard=(r, G))[1] for r in range(G)])
        glob = graf.combine_partials(spec, parts)
        glob_h = graf.combine_partials(spec, parts.cpu())
        assert torch.allclose(glob.cpu(), glob_h, rtol=1e-12, atol=0)
        gsum = torch.zeros_like(g1)
        for r in range(G):
            Lr, gr, _ = graf.af_loss_grad(ds, M, spec, global_partials=glob, shard=(r, G))
            assert torch.allclose(Lr, L1, rtol=1e-6)
            gsum += gr
        tol = 1e-4 * g1.abs().max().item() + 1e-12     # fp32 reassociation across shards
        assert (gsum - g1).abs().max().item() <= tol


# ------------------------------------------------------------------ generic adjoint
@pytest.mark.parametrize("N,M,window", [(16, 16, None), (30, 64, (-7, 12)), (200, 256, None), (100, 1024, (-99, 0)),
                                        (1024, 1024, (500, 1024))])
@pytest.mark.parametrize("layout", ["raw", "centered"])
def test_backward_matches_oracle_adjoint(N, M, window, layout):
    B = 2
    s = cg(B, N, N)
    kb, ke = window if window else (-(N - 1), N)
    rows = np.arange(kb, ke)
    dA = cg(B, len(rows) * M, N + 1).reshape(B, len(rows), M)
    g = graf.af_backward(dev(s), M, dev(dA), k_begin=kb, k_end=ke, layout=layout).cpu().numpy()
    for b in range(B):
        G = dA[b] if layout == "raw" else np.roll(dA[b], -(M // 2), axis=1)   # to raw bins
        ref = O.adjoint(s[b], M, G.astype(np.complex128), rows)
        assert np.abs(g[b] - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
def test_adjoint_inner_product_identity_full_config_size(cfg_id):
    # (A(s+d) - A(s-d))/2 is the exact linearisation of the sesquilinear A:
    # Re<dA, lin> = Re<backward(dA), d>, all through the GPU ABI.
    cfg = CONFIGS[cfg_id]
    N, M = cfg["N"], cfg["M"]
    s = config_waveforms(cfg_id, batch=1)
    dl = cg(1, N, 5)
    kb, ke = -min(N - 1, 300), min(N, 301)
    dA = cg(1, (ke - kb) * M, 6).reshape(1, ke - kb, M)
    ap, _ = graf.af_forward(dev(s + dl), M, out="c64", layout="raw", k_begin=kb, k_end=ke)
    am, _ = graf.af_forward(dev(s - dl), M, out="c64", layout="raw", k_begin=kb, k_end=ke)
    lin = ((ap - am) / 2).cpu().numpy().astype(np.complex128)
    g = graf.af_backward(dev(s), M, dev(dA), k_begin=kb, k_end=ke, layout="raw").cpu().numpy()
    lhs = np.vdot(dA.astype(np.complex128), lin).real
    rhs = np.vdot(g.astype(np.complex128), dl).real
    scale = float(np.sum(np.abs(dA) * np.abs(lin)))
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)


# ------------------------------------------------------------------ properties, determinism, edges
def test_determinism_bitwise():
    cfg = CONFIGS[4]
    s = dev(config_waveforms(4, batch=2))
    spec = graf.LossSpec.from_dict(cfg["loss"])
    a = graf.af_loss_grad(s, cfg["M"], spec)
    b = graf.af_loss_grad(s, cfg["M"], spec)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_c5_full_size_properties():
    # Full N = M = 16384 waveform: gradient invariants that hold at any size
    # (global phase, Doppler modulation, scale invariance of normalised losses).
    cfg = CONFIGS[5]
    s = config_waveforms(5, batch=1)
    spec = graf.LossSpec.from_dict(cfg["loss"])
    loss, g, _ = graf.af_loss_grad(dev(s), cfg["M"], spec)
    g = g.cpu().numpy()[0].astype(np.complex128)
    sd = s[0].astype(np.complex128)
    L = loss.item()
    N = cfg["N"]
    # ISL part is exactly M-1 (volume identity); soft-PSL within its bounds
    assert L > cfg["M"] - 1
    gs = np.abs(g).max() * np.abs(sd).max()
    assert abs(np.vdot(g, sd).imag) <= 1e-3 * gs * N
    assert abs(np.vdot(g, sd).real) <= 1e-3 * gs * N
    assert np.isfinite(g).all()


def test_tiny_and_many_waveforms():
    # N = 1 (single sample), and B > 65535 (grid-chunked launches)
    s = cg(4, 1, 1)
    surf, _ = graf.af_forward(dev(s), 2, out="c64", layout="raw")
    np.testing.assert_allclose(surf.cpu().numpy()[:, 0, :], (np.abs(s) ** 2).repeat(2, 1), rtol=1e-6)
    B = 70000
    s = cg(1, 2 * B, 2).reshape(B, 2)
    surf, _ = graf.af_forward(dev(s), 2, out="c64", layout="raw")
    ref = np.stack([O.surface(s[b], 2, "c64", "raw") for b in (0, 65534, 65535, B - 1)])
    got = surf.cpu().numpy()[[0, 65534, 65535, B - 1]]
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(s).max() ** 2 * 2


def test_autograd_functions():
    N, M = 24, 32
    s_np = cg(2, N, 9)
    spec_d = SPECS[1]
    s = dev(s_np).requires_grad_(True)
    loss = graf.af_loss(s, M, graf.LossSpec.from_dict(spec_d)).sum()
    loss.backward()
    for b in range(2):
        _, g_ref, t = O.loss_and_grad(s_np[b], M, O.LossSpec.from_dict(spec_d))
        assert np.abs(s.grad[b].cpu().numpy() - 2 * g_ref).max() <= 2 * grad_tol(g_ref, t["sigma_g"])
    # AF: arbitrary torch loss on the complex surface, gradient via graf_af_backward
    s2 = dev(s_np).requires_grad_(True)
    A = graf.af(s2, M)
    (A.abs() ** 3).sum().backward()
    st = torch.tensor(s_np.astype(np.complex128), requires_grad=True)
    rows = []
    for k in range(-(N - 1), N):
        lo, hi = max(0, k), min(N, N + k)
        r = torch.zeros(2, M, dtype=torch.complex128)
        r[:, lo:hi] = st[:, lo:hi] * torch.conj(st[:, lo - k:hi - k])
        rows.append(r)
    At = torch.fft.fft(torch.stack(rows, 1), dim=2)
    (At.abs() ** 3).sum().backward()
    ref = st.grad.numpy()
    assert np.abs(s2.grad.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()


# ------------------------------------------------------------------ M = 16384 (split-FFT kernel path)
@pytest.mark.parametrize("N,spec_i", [(300, 1), (1000, 0), (129, 4)])
def test_m16384_loss_grad(N, spec_i):
    M = 16384
    s = cg(2, N, 160 + N)
    spec = dict(SPECS[spec_i], k_max=min(SPECS[spec_i]["k_max"], 40), d_max=min(SPECS[spec_i]["d_max"], 300))
    check_loss_grad(s, M, spec)


def test_m16384_full_plane_small_n():
    # every delay row of a short waveform at M = 16384, soft-PSL + ISL, raw Doppler window
    N, M = 64, 16384
    s = cg(1, N, 77)
    spec = dict(k_max=N - 1, d_max=600, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.01,
                normalize=1)
    check_loss_grad(s, M, spec)


@pytest.mark.parametrize("layout", ["raw", "centered"])
def test_m16384_backward(layout):
    N, M = 64, 16384
    s = cg(1, N, 5)
    kb, ke = -10, 11
    rows = np.arange(kb, ke)
    dA = cg(1, len(rows) * M, 6).reshape(1, len(rows), M)
    g = graf.af_backward(dev(s), M, dev(dA), k_begin=kb, k_end=ke, layout=layout).cpu().numpy()
    G = dA[0] if layout == "raw" else np.roll(dA[0], -(M // 2), axis=1)
    ref = O.adjoint(s[0], M, G.astype(np.complex128), rows)
    assert np.abs(g[0] - ref).max() <= 1e-4 * np.abs(ref).max()


@pytest.mark.parametrize("kb,ke", [(-16383, -16370), (-8193, -8180), (16371, 16384)])
def test_m16384_backward_full_length_edges(kb, ke):
    """graf_af_backward at N = M = 16384 (the split kernel with the global s copies) on
    delay windows at both ends, odd and even rows: the last sample s[N-1] is read from the
    shifted copy for odd negative delays (round-2 fix: rows of NL + M + 2).  dA is nonzero
    on 64 random Doppler bins so the oracle's DFT matrix stays small."""
    N = M = 16384
    s = cg(1, N, 21)
    rows = np.arange(kb, ke)
    rng = np.random.default_rng(3)
    bins = np.sort(rng.choice(M, 64, replace=False))
    G = cg(1, len(rows) * 64, 22).reshape(len(rows), 64)
    dA = np.zeros((1, len(rows), M), np.complex64)
    dA[0][:, bins] = G
    g = graf.af_backward(dev(s), M, dev(dA), k_begin=kb, k_end=ke, layout="raw").cpu().numpy()
    ref = O.adjoint(s[0], M, G.astype(np.complex128), rows, bins)
    assert np.abs(g[0] - ref).max() <= 1e-4 * np.abs(ref).max()
