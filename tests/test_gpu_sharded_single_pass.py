"""GPU parity of the delay-sharded single pass (graf_af_loss_grad_sp_begin / _end;
DESIGN.md readings R13, R27) against the float64 oracle.
G shards run on one GPU in one process (the exchange is the rank-order
graf_combine_partials the sharding layer performs after its all_gather); the sum
of the shard gradients must be dL/ds* and every shard must report the same loss.
Tolerances as in test_gpu_parity.py (reading R18).
"""
import numpy as np
import pytest
import torch

from graf_inputs import CONFIGS, SplitMix64, lfm, random_phase
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


def sharded(ds, M, spec, G):
    ws = [graf.graf.Workspace() for _ in range(G)]
    parts = torch.stack([graf.af_loss_grad_sp_begin(ds, M, spec, (r, G), ws=ws[r]) for r in range(G)])
    glob = graf.combine_partials(spec, parts)
    outs = [graf.af_loss_grad_sp_end(ds, M, spec, (r, G), glob, ws=ws[r]) for r in range(G)]
    g = sum(o[1] for o in outs)
    return [o[0] for o in outs], g, outs[0][2]


# (zero-padded M >= 2N puts the mainlobe's neighbours at x ~ 0.4: outside the R13 rule at T = 0.01)
@pytest.mark.parametrize("N,M,G", [(64, 64, 2), (256, 256, 3), (300, 512, 4), (1024, 1024, 2), (1000, 1024, 5)])
def test_sharded_single_pass_matches_oracle(N, M, G):
    s = np.stack([random_phase(SplitMix64(8_000_000 + b), N) for b in range(3)])
    spec_d = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    spec = graf.LossSpec.from_dict(spec_d)
    ds = dev(s)
    assert graf.single_pass_eligible(ds, M, spec, (0, G))
    losses, g, valid = sharded(ds, M, spec, G)
    assert valid.cpu().numpy().tolist() == [1, 1, 1]
    ospec = O.LossSpec.from_dict(spec_d)
    g = g.cpu().numpy()
    for b in range(3):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        for lo in losses:
            assert abs(lo[b].item() - L_ref) <= 1e-4 * abs(L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol, (b, np.abs(g[b] - g_ref).max(), tol)


def test_sharded_single_pass_validity_flags_and_fallback():
    # an LFM ridge (x ~ 1 next to the mainlobe) is outside the R13 rule at T = 0.01:
    # its flag is 0, loss NaN and gradient 0; the random codes beside it are valid.
    # The sharding layer then reruns the batch with two passes; here the two-pass ABI
    # calls over the same shards must reproduce the oracle.
    N = M = 256
    s = np.stack([random_phase(SplitMix64(8_100_000), N), lfm(N, 1.0).astype(np.complex64),
                  random_phase(SplitMix64(8_100_001), N)])
    spec_d = dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2)
    spec = graf.LossSpec.from_dict(spec_d)
    ds = dev(s)
    losses, g, valid = sharded(ds, M, spec, 2)
    assert valid.cpu().numpy().tolist() == [1, 0, 1]
    assert np.isnan(losses[0][1].item()) and np.abs(g[1].cpu().numpy()).max() == 0.0
    G = 2
    parts = torch.stack([graf.af_forward(ds, M, out=None, loss=spec, shard=(r, G))[1] for r in range(G)])
    glob = graf.combine_partials(spec, parts)
    g2 = sum(graf.af_loss_grad(ds, M, spec, global_partials=glob, shard=(r, G))[1] for r in range(G)).cpu().numpy()
    ospec = O.LossSpec.from_dict(spec_d)
    for b in range(3):
        L_ref, g_ref, t = O.loss_and_grad(s[b], M, ospec)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g2[b] - g_ref).max() <= tol
        if b != 1:
            assert np.abs(g[b].cpu().numpy() - g_ref).max() <= tol


def test_sharded_single_pass_c5_size_against_unsharded():
    # c5's shape (N = M = 16384, full-plane ISL + soft-PSL) over 4 delay shards against
    # the unsharded single pass of the same waveform (both on the GPU; the oracle pins
    # the unsharded path at this size in test_gpu_parity.py::test_c5_full_size_properties)
    N = M = 16384
    s = random_phase(SplitMix64(8_200_000), N)[None]
    spec = graf.LossSpec.from_dict(dict(CONFIGS[5]["loss"], k_max=N - 1, d_max=M // 2))
    ds = dev(s)
    L1, g1, _ = graf.af_loss_grad(ds, M, spec)
    losses, g, valid = sharded(ds, M, spec, 4)
    assert valid.item() == 1
    for lo in losses:
        assert abs(lo.item() - L1.item()) <= 1e-5 * abs(L1.item())
    assert (g - g1).abs().max().item() <= 1e-4 * g1.abs().max().item()


def test_sharded_single_pass_argument_errors():
    N = M = 64
    ds = dev(random_phase(SplitMix64(1), N)[None])
    full = graf.LossSpec(k_max=N - 1, d_max=M // 2, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05)
    with pytest.raises(graf.GrafError):          # shard_count < 2: the unsharded call does this
        graf.af_loss_grad_sp_begin(ds, M, full, (0, 1))
    masked = graf.LossSpec(k_max=10, d_max=8, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05)
    assert not graf.single_pass_eligible(ds, M, masked, (0, 2))
    with pytest.raises(graf.GrafError):          # not the full plane: EUNSUPPORTED
        graf.af_loss_grad_sp_begin(ds, M, masked, (0, 2))
    isl_only = graf.LossSpec(k_max=N - 1, d_max=M // 2, lambda_isl=1.0)
    assert not graf.single_pass_eligible(ds, M, isl_only, (0, 2))


@pytest.mark.parametrize("N,G", [(64, 2), (256, 3)])
def test_sharded_single_pass_periodic(N, G):
    # the paper's circular surface (periodic = 1, M = N): the folded residues k % G == r
    s = np.stack([random_phase(SplitMix64(8_300_000 + b), N) for b in range(2)])
    spec_d = dict(CONFIGS[5]["loss"], k_max=N, d_max=N)
    spec = graf.LossSpec.from_dict(spec_d)
    ds = dev(s)
    assert graf.single_pass_eligible(ds, N, spec, (0, G), periodic=True)
    ws = [graf.graf.Workspace() for _ in range(G)]
    parts = torch.stack([graf.af_loss_grad_sp_begin(ds, N, spec, (r, G), ws=ws[r], periodic=True) for r in range(G)])
    glob = graf.combine_partials(spec, parts)
    outs = [graf.af_loss_grad_sp_end(ds, N, spec, (r, G), glob, ws=ws[r], periodic=True) for r in range(G)]
    assert outs[0][2].cpu().numpy().tolist() == [1, 1]
    g = sum(o[1] for o in outs).cpu().numpy()
    ospec = O.LossSpec.from_dict(spec_d)
    for b in range(2):
        L_ref, g_ref, t = O.loss_and_grad(s[b], N, ospec, periodic=True)
        assert abs(outs[G - 1][0][b].item() - L_ref) <= 1e-4 * abs(L_ref)
        tol = grad_tol(g_ref, t["sigma_g"])
        assert np.abs(g[b] - g_ref).max() <= tol
