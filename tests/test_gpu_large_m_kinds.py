"""GPU parity of the remaining loss kinds on the tensor-memory row kernels (M = 8192, 16384),
which loss-only calls run as their own instantiation without the surface epilogue
(graf_launch.cuh, flavour 1): the hard PSL of the paper's section 7 (Eq. 19 with its
argmax subgradient, pass 1 K_FWDA + psl_grad_kernel) and the
match loss ||x - x_target||^2 (K_MATCH, reading R24), against the float64 oracle."""
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


@pytest.mark.parametrize("N,M", [(300, 8192), (700, 16384), (16384, 16384)])
def test_hard_psl_large_m(N, M):
    d = dict(k_max=min(N - 1, 60), d_max=200, ml_k=0, ml_d=1, lambda_isl=0.5, lambda_psl=0.0, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_hpsl = 1.5
    s = cg(2, N, N % 97 + 3)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec)
    loss, g = loss.cpu().numpy(), g.cpu().numpy()
    ospec = O.LossSpec.from_dict(d)
    for b in range(2):
        L1, g1, t = O.loss_and_grad(s[b], M, ospec)
        psl, g2, cell = O.hard_psl_and_grad(s[b], M, ospec)
        L_ref, g_ref = L1 + 1.5 * psl, g1 + 1.5 * g2
        assert abs(loss[b] - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b], L_ref, cell)
        assert np.abs(g[b] - g_ref).max() <= grad_tol(g_ref, t["sigma_g"]), (b, cell)


@pytest.mark.parametrize("N,M", [(200, 8192), (150, 16384)])
@pytest.mark.parametrize("layout", ["centered", "raw"])
def test_match_loss_large_m(N, M, layout):
    B = 2
    s = cg(B, N, N + 11)
    k_max, d_max = 12, 40
    kb, ke = -k_max, k_max + 1                  # the window holds every delay of the region
    r = SplitMix64(N + M)
    tgt = (r.uniform(B * (ke - kb) * M) * 1e-3).reshape(B, ke - kb, M).astype(np.float32)
    d = dict(k_max=k_max, d_max=d_max, ml_k=0, ml_d=1, lambda_isl=0.3, lambda_psl=0.0, normalize=1)
    spec = graf.LossSpec.from_dict(d)
    spec.lambda_match = 2.0
    spec.target = dev(tgt)
    loss, g, _ = graf.af_loss_grad(dev(s), M, spec, layout=layout, k_begin=kb, k_end=ke)
    ospec = O.LossSpec.from_dict(d)
    for b in range(B):
        Lm, gm = O.match_loss_and_grad(s[b], M, ospec, tgt[b].astype(np.float64), kb, layout, False)
        Li, gi, t = O.loss_and_grad(s[b], M, ospec)
        L_ref, g_ref = Li + 2.0 * Lm, gi + 2.0 * gm
        assert abs(loss[b].item() - L_ref) <= 1e-4 * abs(L_ref), (b, loss[b].item(), L_ref)
        assert np.abs(g[b].cpu().numpy() - g_ref).max() <= grad_tol(g_ref, t["sigma_g"]), b
