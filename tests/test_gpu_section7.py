"""GPU parity of the paper's section-7 workload against
the float64 oracle: hard PSL with its argmax subgradient (Eq. 19, PAPER.md
L286-290; reading R23), spectral variance (L417; reading R22), the phase Adam
step (L425) and the batched Eq. 26 optimisation loop (L416).
Tolerances as in test_gpu_parity.py (reading R18)."""
import numpy as np
import pytest
import torch

from graf_inputs import SplitMix64, complex_gaussian, random_phase
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


HSPECS = [
    dict(k_max=5, d_max=4, ml_k=0, ml_d=0, normalize=1),
    dict(k_max=10000, d_max=10000, ml_k=0, ml_d=0, normalize=1),
    dict(k_max=7, d_max=9, ml_k=1, ml_d=1, normalize=0),
]


@pytest.mark.parametrize("si", range(len(HSPECS)))
@pytest.mark.parametrize("N,M,periodic", [(16, 16, False), (33, 64, False), (100, 256, False), (64, 64, True),
                                          (256, 256, True), (512, 1024, False)])
def test_hard_psl_loss_and_subgradient(si, N, M, periodic):
    d = dict(HSPECS[si], lambda_isl=0.0, lambda_psl=0.0)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_hpsl = 1.0
    s = cg(3, N, 7 * si + N)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, periodic=periodic)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(d)
    for b in range(3):
        psl, gref, cell = O.hard_psl_and_grad(s[b], M, ospec, periodic)
        assert abs(loss[b] - psl) <= 1e-4 * abs(psl), (b, loss[b], psl, cell)
        E = O.energy(s[b])
        sig = 2 * psl / E * np.abs(s[b]).max() if ospec.normalize else 0.0   # cancelling normalisation term
        assert np.abs(g[b] - gref).max() <= 1e-4 * max(np.abs(gref).max(), sig), (b, cell)


def test_hard_psl_with_isl_and_softpsl():
    N, M = 120, 128
    d = dict(k_max=30, d_max=20, ml_k=0, ml_d=1, lambda_isl=0.5, lambda_psl=0.7, temperature=0.05, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_hpsl = 2.0
    s = cg(2, N, 5)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec)
    ospec = O.LossSpec.from_dict(d)
    for b in range(2):
        L1, g1, t = O.loss_and_grad(s[b], M, ospec)
        psl, g2, _ = O.hard_psl_and_grad(s[b], M, ospec)
        L_ref, g_ref = L1 + 2.0 * psl, g1 + 2.0 * g2
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= grad_tol(g_ref, t["sigma_g"])


def test_hard_psl_sharding_algebra():
    N, M = 96, 128
    spec = graf.LossSpec(k_max=40, d_max=30, ml_k=0, ml_d=1, lambda_isl=0.0, lambda_psl=0.0, normalize=1)
    spec.lambda_hpsl = 1.0
    s = dev(cg(2, N, 8))
    L1, g1, _ = graf.af_loss_grad(s, M, spec)
    for G in (2, 3):
        parts = torch.stack([graf.af_forward(s, M, out=None, loss=spec, shard=(r, G))[1] for r in range(G)])
        glob = graf.combine_partials(spec, parts)
        assert torch.equal(glob.cpu(), graf.combine_partials(spec, parts.cpu()))
        gsum = torch.zeros_like(g1)
        for r in range(G):
            Lr, gr, _ = graf.af_loss_grad(s, M, spec, global_partials=glob, shard=(r, G))
            assert torch.allclose(Lr, L1, rtol=1e-6)
            gsum += gr
        assert (gsum - g1).abs().max().item() <= 1e-4 * g1.abs().max().item()


@pytest.mark.parametrize("ddof", [0, 1])
@pytest.mark.parametrize("N", [2, 8, 32, 64, 128, 256, 512, 1024, 2048, 4096])
def test_spectral_variance(N, ddof):
    s = cg(3, N, N + 1)
    w = torch.tensor([1.0, 0.5, 3.0], dtype=torch.float32, device="cuda")
    loss, g = graf.spectral_variance(dev(s), weights=w, ddof=ddof)
    for b in range(3):
        sv, gref = O.spectral_variance_and_grad(s[b], ddof=ddof)
        wb = float(w[b])
        assert abs(loss[b].item() - wb * sv) <= 1e-4 * wb * sv + 1e-12
        assert np.abs(g[b].cpu().numpy() - wb * gref).max() <= 1e-4 * wb * np.abs(gref).max() + 1e-12
    # accumulate mode adds onto an existing loss / gradient
    l0 = torch.ones(3, dtype=torch.float64, device="cuda")
    g0 = torch.ones((3, N), dtype=torch.complex64, device="cuda")
    l1, g1 = graf.spectral_variance(dev(s), weights=w, loss=l0.clone(), grad=g0.clone(), accumulate=True,
                                    ddof=ddof)
    assert torch.allclose(l1 - 1.0, loss, rtol=1e-9, atol=1e-15)
    assert (g1 - 1.0 - g).abs().max().item() <= 1e-6 * max(1.0, g.abs().max().item())


def test_spectral_variance_large_invariants():
    N = 16384
    s = dev(cg(2, N, 3))
    loss, g = graf.spectral_variance(s)
    # scale and global-phase invariance of SV: <g, s> = 0; tone -> 1/N
    ip = (torch.conj(g) * s).sum(dim=1)
    assert ip.abs().max().item() <= 1e-4 * (g.abs() * s.abs()).sum(dim=1).max().item()
    tone = torch.exp(2j * np.pi * 7 * torch.arange(N, dtype=torch.float64) / N).to(torch.complex64).cuda()[None]
    lt, _ = graf.spectral_variance(tone)
    assert abs(lt.item() - (N - 1) / N ** 2) <= 1e-3 / N          # population variance
    ones = torch.ones((1, 4), dtype=torch.complex64, device="cuda")
    assert abs(graf.spectral_variance(ones)[0].item() - 0.1875) <= 1e-6   # SPEC.md L331 example


def test_phase_adam_matches_oracle():
    B, N = 3, 40
    r = SplitMix64(5)
    th = (r.uniform(B * N) * 6).reshape(B, N)
    grads = [cg(B, N, 20 + i) for i in range(4)]
    theta = torch.tensor(th, dtype=torch.float32, device="cuda")
    m = torch.zeros_like(theta); v = torch.zeros_like(theta)
    step = torch.zeros(B, dtype=torch.int32, device="cuda")
    s_out = torch.empty((B, N), dtype=torch.complex64, device="cuda")
    x = th.copy(); mo = np.zeros_like(th); vo = np.zeros_like(th)
    for t, gr in enumerate(grads, start=1):
        s_cur = np.exp(1j * x)
        graf.phase_adam_step(theta, m, v, step, dev(gr.astype(np.complex64)), s_out)
        x, mo, vo = O.adam_step(x, mo, vo, O.phase_grad(s_cur, gr.astype(np.complex64).astype(complex)), t)
        assert np.abs(theta.cpu().numpy() - x).max() < 1e-4
    assert step.cpu().tolist() == [4, 4, 4]
    np.testing.assert_allclose(s_out.cpu().numpy(), np.exp(1j * theta.cpu().numpy().astype(np.float64)), atol=1e-6)


def test_lpi_optimizer_follows_the_oracle_loop():
    # Eq. 26 with the paper's settings (periodic surface, PSL over the plane minus the
    # origin, alpha = 2000, Adam lr 0.01) on a small batch: lambda sweep in one batch
    B, N, iters = 3, 32, 6
    lam = np.array([0.1, 0.5, 1.0])
    th0 = np.stack([np.angle(random_phase(SplitMix64(b), N)) for b in range(B)])
    opt = graf.LpiOptimizer(torch.tensor(th0, dtype=torch.float32, device="cuda"), torch.tensor(lam),
                            per_graph=2)
    loss = opt.run(iters).cpu().numpy()
    spec = O.LossSpec(k_max=N, d_max=N, normalize=1)
    for b in range(B):
        x = th0[b].astype(np.float32).astype(np.float64)
        mo = np.zeros(N); vo = np.zeros(N)
        for t in range(1, iters + 1):
            L, gth, _ = O.lpi_loss_and_grad(x, spec, lam[b])
            x, mo, vo = O.adam_step(x, mo, vo, gth, t)
        assert abs(loss[b] - L) <= 1e-3 * abs(L)
        assert np.abs(opt.theta[b].cpu().numpy() - x).max() < 1e-3
