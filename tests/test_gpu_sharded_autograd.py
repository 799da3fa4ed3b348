"""graf.af_loss(..., shard="delay" | "batch") (sharding.ShardedAFLoss) on one GPU with no
process group (world size 1): it must reproduce the unsharded autograd loss and torch's
.grad = 2 dL/ds* through the C ABI.  The multi-rank exchange itself is covered by
tests/test_sharding_gloo.py::test_sharded_af_loss_autograd_gloo_world2 (gloo, oracle backend)."""
import numpy as np
import pytest
import torch

from graf_inputs import SplitMix64, complex_gaussian

pytestmark = pytest.mark.gpu

graf = pytest.importorskip("paper_2506_22935_b200")


@pytest.mark.parametrize("shard", ["delay", "batch"])
def test_sharded_af_loss_world1_matches_unsharded(shard):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    N, M = 200, 256
    spec = graf.LossSpec.from_dict(dict(k_max=40, d_max=30, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0,
                                        temperature=0.05, normalize=1))
    s0 = torch.from_numpy(np.stack([complex_gaussian(SplitMix64(31 + b), N) for b in range(3)])).cuda()
    w = torch.tensor([1.0, -2.0, 0.5], dtype=torch.float64, device="cuda")
    a = s0.clone().requires_grad_(True)
    la = graf.af_loss(a, M, spec)
    (la * w).sum().backward()
    b = s0.clone().requires_grad_(True)
    lb = graf.af_loss(b, M, spec, shard=shard)
    (lb * w).sum().backward()
    torch.testing.assert_close(lb, la, rtol=1e-6, atol=0.0)
    torch.testing.assert_close(b.grad, a.grad, rtol=1e-5, atol=1e-5 * a.grad.abs().max().item())
