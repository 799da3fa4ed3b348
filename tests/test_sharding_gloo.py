"""Multi-process (gloo, world_size 2, CPU) tests of the sharding layer
(paper_2506_22935_b200/sharding.py): the exchange steps (all_gather of LSE
partials, rank-order combine, all_reduce of the gradient) must reproduce the
unsharded result.  The per-shard compute is a float64 oracle-backed stand-in for
the C ABI (no GPU here); on the GPU the same algebra is checked through the ABI
in test_gpu_parity.py::test_forward_partials_and_delay_sharding_algebra.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from graf_inputs import SplitMix64, complex_gaussian
from oracle import graf_oracle as O


class OracleShardBackend:
    """Per-shard quantities from the oracle: folded delay rows k >= 0 with
    k % G == r stand for the rows +-k of the full region."""

    def __init__(self, N, M):
        self.N, self.M = N, M

    def _rows(self, spec, shard):
        r, G = shard
        K = min(spec.k_max, self.N - 1)
        return np.array([k for k in range(-K, K + 1) if abs(k) % G == r])

    def _cells(self, s, spec, shard):
        rows_all, bins, mask, w = O.region(self.N, self.M, spec)
        keep = np.isin(rows_all, self._rows(spec, shard))
        A = O.ambiguity(s, self.M, rows_all[keep], bins)
        return rows_all[keep], bins, mask[keep], w[keep], A

    def _key_lo(self, spec):
        return -min(spec.k_max, self.N - 1)

    def forward_partials(self, s_b, M, spec, shard, skip=None):
        out = []
        for b, s in enumerate(s_b.numpy()):
            if skip is not None and int(skip[b]):
                out.append([0.0, -np.inf, 0.0, 0.0, float(0x7fffffff), 0.0])   # identity partials
                continue
            rows, bins, mask, w, A = self._cells(s, spec, shard)
            E = O.energy(s)
            chi = np.abs(A) ** 2
            x = chi / E ** 2 if spec.normalize else chi
            S = float(np.sum(w[mask] * chi[mask]))
            key = float(0x7fffffff)
            if mask.any():
                c = float(np.max(x[mask]))
                Z = float(np.sum(np.exp((x[mask] - c) / spec.temperature)))
                # hard PSL: row-major key (delay index from key_lo) * M + raw bin of the
                # lowest-keyed maximal cell (include/graf.h graf_partials.psl_key)
                ii, jj = np.nonzero(mask & (x == c))
                key = float(min((int(rows[i]) - self._key_lo(spec)) * M + int(bins[j]) for i, j in zip(ii, jj)))
            else:
                c, Z = -np.inf, 0.0
            out.append([S, c, Z, 0.0, key, 0.0])
        return torch.tensor(out, dtype=torch.float64)

    def combine(self, spec, parts):
        from paper_2506_22935_b200 import graf
        return graf.combine_partials(spec, parts)

    def loss_grad(self, s_b, M, spec, glob, shard, skip=None, loss_out=None, grad=None):
        hpsl = getattr(spec, "lambda_hpsl", 0.0)
        if glob is None and (spec.lambda_psl != 0 or hpsl != 0):
            # like graf_af_loss_grad with global = NULL: this call's own partials
            glob = self.forward_partials(s_b, M, spec, shard)
        losses, grads = [], []
        T = spec.temperature
        for b, s in enumerate(s_b.numpy()):
            if skip is not None and int(skip[b]):
                losses.append(loss_out[b].item())
                grads.append(grad[b].numpy())
                continue
            rows, bins, mask, w, A = self._cells(s, spec, shard)
            E = O.energy(s)
            chi = np.abs(A) ** 2
            x = chi / E ** 2 if spec.normalize else chi
            if glob is not None:
                S, c, Z = glob[b, 0].item(), glob[b, 1].item(), glob[b, 2].item()
            else:
                S, c, Z = float(np.sum(w[mask] * chi[mask])), 0.0, 1.0
            lse = c + T * np.log(Z)
            isl = S / E ** 2 if spec.normalize else S
            L = spec.lambda_isl * isl + (spec.lambda_psl * lse if spec.lambda_psl else 0.0)
            fp = np.where(mask, spec.lambda_isl * w + spec.lambda_psl * np.exp((x - lse) / T), 0.0)
            G = fp * A / E ** 2 if spec.normalize else fp * A
            g = O.adjoint(s, self.M, G, rows, bins)
            if spec.normalize:
                g = g - (2.0 / E ** 3) * float(np.sum(fp * chi)) * s
            if hpsl:
                # hard PSL from the GLOBAL max and argmax key; the subgradient term is held by
                # shard 0 only (the sum over shards is the full gradient)
                L += hpsl * glob[b, 1].item()
                if shard[0] == 0:
                    key = int(glob[b, 4].item())
                    k, m = key // M + self._key_lo(spec), key % M
                    Ak = O.ambiguity(s, M, rows=np.array([k]), bins=np.array([m]))
                    Gk = hpsl * (Ak / E ** 2 if spec.normalize else Ak)
                    g = g + O.adjoint(s, M, Gk, np.array([k]), np.array([m]))
                    if spec.normalize:
                        g = g - (2.0 / E ** 3) * hpsl * float(np.abs(Ak[0, 0]) ** 2) * s
            losses.append(L)
            grads.append(g)
        lo, go = torch.tensor(losses, dtype=torch.float64), torch.tensor(np.stack(grads))
        if loss_out is not None:        # in place, like the ABI's caller-owned outputs
            loss_out.copy_(lo)
            grad.copy_(go)
            return loss_out, grad
        return lo, go


class OracleSinglePassBackend(OracleShardBackend):
    """Adds the delay-sharded single pass (graf_af_loss_grad_sp_begin / _end, reading
    R27) in float64: phase 1 returns (S, max x, 0, sum expm1((x - xbar)/T)) over the
    shard's cells; phase 2 uses the global sums, f' = lambda_psl e / Z_c (ISL and
    constant terms dropped, as on the GPU: their sum over all shards vanishes on the
    full plane) and the R13 rule on the global max."""

    def _full(self, spec):
        return (spec.k_max >= self.N - 1 and spec.d_max >= self.M // 2 and spec.ml_k == 0 and spec.ml_d == 0
                and spec.normalize == 1 and spec.lambda_psl != 0 and spec.w_k is None and spec.w_d is None)

    def single_pass_eligible(self, s, M, spec, shard):
        return self._full(spec)

    def _xbar(self):
        omega = (2 * self.N - 1) * self.M - 1
        return omega, (self.M - 1) / omega

    def sp_begin(self, s_b, M, spec, shard):
        _, xbar = self._xbar()
        out = []
        for s in s_b.numpy():
            rows, bins, mask, w, A = self._cells(s, spec, shard)
            E = O.energy(s)
            chi = np.abs(A) ** 2
            x = chi / E ** 2
            e = np.expm1((x[mask] - xbar) / spec.temperature)
            c = float(np.max(x[mask])) if mask.any() else -np.inf
            out.append([float(np.sum(w[mask] * chi[mask])), c, 0.0, float(np.sum(e)), 0.0, 0.0])
        return torch.tensor(out, dtype=torch.float64)

    def sp_end(self, s_b, M, spec, glob, shard):
        # (returns NaN loss / zero grad where the rule fails, like the ABI)
        omega, xbar = self._xbar()
        T = spec.temperature
        losses, grads, valid = [], [], []
        for b, s in enumerate(s_b.numpy()):
            rows, bins, mask, w, A = self._cells(s, spec, shard)
            E = O.energy(s)
            chi = np.abs(A) ** 2
            x = chi / E ** 2
            S, m, C = glob[b, 0].item(), glob[b, 1].item(), glob[b, 3].item()
            ok = np.isfinite(C) and (m - xbar) / T <= 40.0
            zc = omega + C
            losses.append(spec.lambda_isl * S / E ** 2 + spec.lambda_psl * (xbar + T * np.log(zc)) if ok else np.nan)
            fp = np.where(mask, spec.lambda_psl * np.expm1((x - xbar) / T) / zc, 0.0) if ok else np.zeros_like(x)
            g = O.adjoint(s, self.M, fp * A / E ** 2, rows, bins) - (2.0 / E ** 3) * float(np.sum(fp * chi)) * s
            grads.append(g)
            valid.append(1 if ok else 0)
        return (torch.tensor(losses, dtype=torch.float64), torch.tensor(np.stack(grads)),
                torch.tensor(valid, dtype=torch.int32))


def _sp_worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_22935_b200 import sharding, LossSpec
        N, M, spec_d = case
        s = np.stack([complex_gaussian(SplitMix64(700 + b), N) for b in range(3)]).astype(np.complex128)
        be = OracleSinglePassBackend(N, M)
        calls = []
        fwd = be.forward_partials

        def spy(*a, skip=None):
            # the device-side fallback always runs; it does work only for unskipped waveforms
            if skip is None or not bool(skip.all()):
                calls.append("two-pass")
            return fwd(*a, skip=skip)
        be.forward_partials = spy
        loss, g = sharding.delay_sharded_loss_grad(torch.tensor(s), M, LossSpec.from_dict(spec_d), backend=be)
        q.put((rank, loss.numpy(), g.numpy(), calls))
    finally:
        dist.destroy_process_group()


SP_CASES = [
    # full plane, T = 0.05: the single pass is valid for every waveform
    ((12, 16, dict(k_max=11, d_max=8, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1)), False),
    # T = 0.004: max x - xbar > 40 T, every rank falls back to the two-pass protocol
    ((12, 16, dict(k_max=11, d_max=8, lambda_isl=0.5, lambda_psl=1.0, temperature=0.004, normalize=1)), True),
]


@pytest.mark.parametrize("case,fallback", SP_CASES)
def test_delay_sharded_single_pass_gloo_world2(case, fallback):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sp_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, M, spec_d = case
    s = np.stack([complex_gaussian(SplitMix64(700 + b), N) for b in range(3)]).astype(np.complex128)
    ospec = O.LossSpec.from_dict(spec_d)
    refs = [O.loss_and_grad(s[b], M, ospec) for b in range(3)]
    L_ref = np.array([r[0] for r in refs])
    g_ref = np.stack([r[1] for r in refs])
    for rank, loss, g, calls in res:
        assert (len(calls) > 0) == fallback, calls
        np.testing.assert_allclose(loss, L_ref, rtol=1e-10)
        np.testing.assert_allclose(g, g_ref, atol=1e-9 * np.abs(g_ref).max())


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_22935_b200 import sharding, LossSpec
        N, M, spec_d = case
        s = np.stack([complex_gaussian(SplitMix64(900 + b), N) for b in range(3)]).astype(np.complex128)
        spec = LossSpec.from_dict(spec_d)
        be = OracleShardBackend(N, M)
        loss, g = sharding.delay_sharded_loss_grad(torch.tensor(s), M, spec, backend=be)
        sl, lb, gb = sharding.batch_sharded_loss_grad(torch.tensor(s), M, spec, backend=be)
        q.put((rank, loss.numpy(), g.numpy(), (sl.start, sl.stop), lb.numpy(), gb.numpy()))
    finally:
        dist.destroy_process_group()


CASES = [
    (12, 16, dict(k_max=6, d_max=5, ml_k=0, ml_d=0, lambda_isl=1.0, lambda_psl=0.0, normalize=1)),
    # hard PSL (section-7 loss) needs the global argmax: the two-pass protocol, not the
    # ISL-only shortcut
    (12, 16, dict(k_max=6, d_max=5, ml_k=0, ml_d=0, lambda_isl=0.5, lambda_psl=0.0, lambda_hpsl=1.0,
                  normalize=1)),
    (12, 16, dict(k_max=11, d_max=8, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1)),
    (9, 16, dict(k_max=4, d_max=6, ml_k=1, ml_d=0, lambda_isl=0.0, lambda_psl=1.0, temperature=50.0, normalize=0)),
]


@pytest.mark.parametrize("case", CASES)
def test_delay_and_batch_sharding_gloo_world2(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, M, spec_d = case
    s = np.stack([complex_gaussian(SplitMix64(900 + b), N) for b in range(3)]).astype(np.complex128)
    ospec = O.LossSpec.from_dict(spec_d)
    refs = [O.loss_and_grad(s[b], M, ospec) for b in range(3)]
    L_ref = np.array([r[0] for r in refs])
    g_ref = np.stack([r[1] for r in refs])
    if spec_d.get("lambda_hpsl"):
        hp = [O.hard_psl_and_grad(s[b], M, ospec) for b in range(3)]
        L_ref = L_ref + spec_d["lambda_hpsl"] * np.array([h[0] for h in hp])
        g_ref = g_ref + spec_d["lambda_hpsl"] * np.stack([h[1] for h in hp])
    for rank, loss, g, (a, z), lb, gb in res:
        np.testing.assert_allclose(loss, L_ref, rtol=1e-10)
        np.testing.assert_allclose(g, g_ref, atol=1e-10 * np.abs(g_ref).max())
        np.testing.assert_allclose(lb, L_ref[a:z], rtol=1e-10)
        np.testing.assert_allclose(gb, g_ref[a:z], atol=1e-10 * np.abs(g_ref).max())
    blocks = sorted((a, z) for _, _, _, (a, z), _, _ in res)
    assert blocks == [(0, 2), (2, 3)]


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_22935_b200 import sharding

        class Fake:
            def loss_grad(self, s, M, spec, glob, shard):
                return s.real.sum(1).double(), s
        s = torch.arange(7, dtype=torch.float64).to(torch.complex128)[:, None].repeat(1, 3)
        sl, loss, g = sharding.batch_sharded_loss_grad(s, 4, None, backend=Fake(), gather_loss=True)
        q.put((rank, loss.numpy()))
    finally:
        dist.destroy_process_group()


def test_batch_sharded_gather_loss_unequal_blocks():
    """B = 7 over 2 ranks (blocks of 4 and 3): the padded all_gather returns the full,
    correctly ordered loss vector (equal-size collective buffers)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, loss in res:
        np.testing.assert_array_equal(loss, 3.0 * np.arange(7))


def test_batch_slice_partition():
    from paper_2506_22935_b200.sharding import batch_slice
    for B in (1, 7, 256):
        for G in (1, 2, 3, 8):
            sl = [batch_slice(B, r, G) for r in range(G)]
            assert sl[0].start == 0 and sl[-1].stop == B
            assert all(sl[i].stop == sl[i + 1].start for i in range(G - 1))
            assert max(x.stop - x.start for x in sl) - min(x.stop - x.start for x in sl) <= 1


def _autograd_worker(rank, world, port, shard, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2506_22935_b200 import LossSpec, graf
        N, M = 12, 16
        spec_d = dict(k_max=11, d_max=8, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05,
                      normalize=1)
        s = torch.tensor(np.stack([complex_gaussian(SplitMix64(950 + b), N) for b in range(3)]).astype(np.complex128),
                         requires_grad=True)
        loss = graf.af_loss(s, M, LossSpec.from_dict(spec_d), shard=shard, backend=OracleShardBackend(N, M))
        (loss * torch.arange(1, loss.shape[0] + 1, dtype=loss.dtype)).sum().backward()
        q.put((rank, loss.detach().numpy(), s.grad.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shard", ["delay", "batch"])
def test_sharded_af_loss_autograd_gloo_world2(shard):
    """graf.af_loss(..., shard=) (sharding.ShardedAFLoss) on world_size 2 with the oracle
    backend: the loss and torch's .grad = 2 dL/ds* against the unsharded float64 oracle,
    with a non-uniform upstream gradient (weights 1, 2, ... per waveform)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_autograd_worker, args=(r, 2, port, shard, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    N, M = 12, 16
    spec_d = dict(k_max=11, d_max=8, ml_k=0, ml_d=1, lambda_isl=1.0, lambda_psl=1.0, temperature=0.05, normalize=1)
    s = np.stack([complex_gaussian(SplitMix64(950 + b), N) for b in range(3)]).astype(np.complex128)
    refs = [O.loss_and_grad(s[b], M, O.LossSpec.from_dict(spec_d)) for b in range(3)]
    L_ref = np.array([r[0] for r in refs])
    g_ref = np.stack([r[1] for r in refs])
    from paper_2506_22935_b200.sharding import batch_slice
    total = np.zeros_like(g_ref)
    for rank, loss, grad in res:
        sl = slice(None) if shard == "delay" else batch_slice(3, rank, 2)
        np.testing.assert_allclose(loss, L_ref[sl], rtol=1e-10)
        w = np.arange(1, len(loss) + 1)          # the worker's upstream weights on ITS loss vector
        want = np.zeros_like(g_ref)
        want[sl] = 2.0 * w[:, None] * g_ref[sl]
        np.testing.assert_allclose(grad, want, atol=1e-10 * np.abs(want).max())
        total += grad
    if shard == "batch":   # the ranks' gradients are disjoint blocks that tile the batch
        assert np.all(total != 0)
