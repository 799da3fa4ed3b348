"""Multi-GPU layers over torch.distributed.

One process per GPU.  Two partitionings of the same hot path:

* Batch sharding (configs c2-c4): rank r owns a contiguous block of waveforms;
  waveforms are independent, so there is NO collective on the data path.

* Delay sharding (config c5, one waveform larger than a single GPU's share):
  rank r owns the folded delay rows k >= 0 with k % G == r (interleaved, which
  balances the (N-k)-long lag/correlation work).  The exchange steps are
    1. soft-PSL only: all_gather of the per-shard partials (isl_sum, lse_max,
       lse_sum, cen_sum) [B x 32 B], combined in rank order (graf_combine_partials,
       deterministic) -> every rank holds the global log-sum-exp;
    2. all_reduce(SUM) of the per-shard gradient g_r [B, N] (complex64), which
       already includes the shard's share of the normalisation term (linear in
       its own partial sums), so the sum is the full dL/ds*.
  ISL-only losses are linear in the per-row sums, so step 1 is skipped and the
  per-shard losses are summed with the gradient.  Hard PSL (lambda_hpsl) needs the
  global max, so it runs step 1 like soft-PSL.
  The full-plane normalised soft-PSL (c5) runs ONE pass per shard instead of two
  (reading R13 across shards, R27).  Phase 1 computes each shard's partials, including
  the centred sum sum expm1((x - xbar)/T); those are all-gathered and combined.  Phase 2
  scales each shard's gradient by the global 1/Z_c, and then comes the gradient
  all_reduce.  Waveforms outside the global validity rule are recomputed by the two-pass
  protocol with the others masked out (graf_af_desc.skip): the decision stays on the
  device, so there is no host synchronisation and the step is graph-capturable.

`backend` is the object that runs the per-shard compute; the default calls the
C ABI (graf_af_forward / graf_af_loss_grad / graf_combine_partials).  Tests on CPU
(gloo, world_size 2) substitute a float64 oracle-backed backend to check the
exchange logic without a GPU.
"""
from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist

from . import graf as _graf

__all__ = ["GrafBackend", "batch_slice", "batch_sharded_loss_grad", "delay_sharded_loss_grad", "ShardedAFLoss",
           "sharded_af_loss"]


class GrafBackend:
    """Per-shard compute through the C ABI (device tensors).  Each instance owns its
    workspaces (the single pass keeps its unscaled gradient in `ws_sp` between phases)."""

    def __init__(self):
        self.ws = _graf.Workspace()
        self.ws_sp = _graf.Workspace()

    def forward_partials(self, s, M, spec, shard, skip=None):
        return _graf.af_forward(s, M, out=None, loss=spec, shard=shard, ws=self.ws, skip=skip)[1]

    def loss_grad(self, s, M, spec, global_partials, shard, skip=None, loss_out=None, grad=None):
        loss, g, _ = _graf.af_loss_grad(s, M, spec, global_partials=global_partials, shard=shard, ws=self.ws,
                                        skip=skip, loss_out=loss_out, grad=grad)
        return loss, g

    def combine(self, spec, parts):
        return _graf.combine_partials(spec, parts)

    def single_pass_eligible(self, s, M, spec, shard):
        return _graf.single_pass_eligible(s, M, spec, shard)

    def sp_begin(self, s, M, spec, shard):
        return _graf.af_loss_grad_sp_begin(s, M, spec, shard, ws=self.ws_sp)

    def sp_end(self, s, M, spec, glob, shard):
        return _graf.af_loss_grad_sp_end(s, M, spec, shard, glob, ws=self.ws_sp)


def _world(group) -> Tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def batch_slice(B: int, rank: int, world: int) -> slice:
    """Contiguous block of waveforms owned by `rank` (sizes differ by at most 1)."""
    base, rem = divmod(B, world)
    start = rank * base + min(rank, rem)
    return slice(start, start + base + (1 if rank < rem else 0))


def batch_sharded_loss_grad(s_all: torch.Tensor, M: int, spec, group=None, backend=None,
                            gather_loss: bool = False):
    """Batch sharding: this rank's waveforms only; no data-path collective.
    Returns (slice, loss[b], grad[b]) for the local block; with gather_loss the
    full loss vector [B] is all-gathered for reporting (off the hot path)."""
    backend = backend or GrafBackend()
    r, G = _world(group)
    B = s_all.shape[0]
    sl = batch_slice(B, r, G)
    loss, g = backend.loss_grad(s_all[sl], M, spec, None, (0, 1))
    if gather_loss and G > 1:
        # blocks differ in size by at most one: pad every block to ceil(B/G) so the
        # collective moves equal-size buffers, then trim by the known slices
        bmax = -(-B // G)
        pad = torch.zeros((bmax,), dtype=loss.dtype, device=loss.device)
        pad[:loss.shape[0]] = loss
        parts = [torch.empty_like(pad) for _ in range(G)]
        dist.all_gather(parts, pad, group=group)
        loss = torch.cat([parts[q][:batch_slice(B, q, G).stop - batch_slice(B, q, G).start] for q in range(G)])
    return sl, loss, g


def _gather_combine(backend, spec, part, G, group):
    gathered = [torch.empty_like(part) for _ in range(G)]
    dist.all_gather(gathered, part.contiguous(), group=group)
    return backend.combine(spec, torch.stack(gathered))


def delay_sharded_loss_grad(s: torch.Tensor, M: int, spec, group=None, backend=None):
    """Delay sharding of every waveform in `s` across the ranks of `group`.
    Returns (loss[B] float64, grad[B, N] complex64 = dL/ds*), identical on all ranks.
    No host synchronisation on any branch (the single pass's fallback decision stays on
    the device), so a step can be captured in a CUDA graph with its NCCL collectives."""
    backend = backend or GrafBackend()
    r, G = _world(group)
    shard = (r, G)
    if G == 1:
        return backend.loss_grad(s, M, spec, None, (0, 1))
    hpsl = getattr(spec, "lambda_hpsl", 0.0) != 0
    match = getattr(spec, "lambda_match", 0.0) != 0
    if spec.lambda_psl == 0 and not hpsl:
        # ISL / match only: linear in the rows, one fused pass per shard; loss and gradient
        # are sums over shards
        loss, g = backend.loss_grad(s, M, spec, None, shard)
        dist.all_reduce(loss, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(torch.view_as_real(g), op=dist.ReduceOp.SUM, group=group)
        return loss, g
    if match:
        raise NotImplementedError("delay sharding of a match loss with soft/hard PSL: the match term "
                                  "needs unsharded calls in v1 (graf_af_loss_grad rejects it with `global`)")
    if hasattr(backend, "sp_begin") and backend.single_pass_eligible(s, M, spec, shard):
        # full-plane soft-PSL: one pass per shard, the global 1/Z_c applied in phase 2
        glob = _gather_combine(backend, spec, backend.sp_begin(s, M, spec, shard), G, group)
        loss, g, valid = backend.sp_end(s, M, spec, glob, shard)
        # device-side fallback: the two-pass protocol over the waveforms whose single pass
        # broke the R13 rule (valid == 0); valid waveforms are skipped (their CTAs exit at
        # once, their loss / grad are left as phase 2 wrote them).  Every rank holds the
        # same `valid`, so the collectives below match.
        skip = valid.to(torch.int32).contiguous()
        glob2 = _gather_combine(backend, spec, backend.forward_partials(s, M, spec, shard, skip=skip), G, group)
        loss, g = backend.loss_grad(s, M, spec, glob2, shard, skip=skip, loss_out=loss, grad=g)
        dist.all_reduce(torch.view_as_real(g), op=dist.ReduceOp.SUM, group=group)
        return loss, g
    # soft-PSL / hard PSL: pass 1 partials -> all_gather -> combine (rank order) -> pass 2
    # (hard PSL: the global argmax key travels in the partials) -> all_reduce of g
    glob = _gather_combine(backend, spec, backend.forward_partials(s, M, spec, shard), G, group)
    loss, g = backend.loss_grad(s, M, spec, glob, shard)
    dist.all_reduce(torch.view_as_real(g), op=dist.ReduceOp.SUM, group=group)
    return loss, g


class ShardedAFLoss(torch.autograd.Function):
    """Differentiable sharded loss (SURVEY.md §8(b) "Python (L3)": af_loss(s, M, spec, group,
    shard)).  Every rank passes the whole batch s [B, N].
      shard="delay": the loss of every waveform, identical on all ranks, and in backward the
        full gradient (the forward's all_reduce already summed the shards) on every rank.
      shard="batch": this rank's block of waveforms only (no collective); the
        loss of that block, and in backward a gradient that is zero outside the block (sum
        s.grad over the ranks, as data-parallel training does, for the whole batch's).
    torch's convention: .grad = 2 dL/ds* (the ABI returns dL/ds*)."""

    @staticmethod
    def forward(ctx, s, M, spec, shard, group, backend):
        if shard == "delay":
            loss, g = delay_sharded_loss_grad(s.detach(), M, spec, group=group, backend=backend)
            ctx.block = None
        elif shard == "batch":
            sl, loss, g = batch_sharded_loss_grad(s.detach(), M, spec, group=group, backend=backend)
            ctx.block = (sl.start, sl.stop)
        else:
            raise ValueError(f"shard must be 'delay' or 'batch', not {shard!r}")
        ctx.save_for_backward(g)
        ctx.s_meta = (s.shape, s.dtype)
        return loss

    @staticmethod
    def backward(ctx, grad_out):
        (g,) = ctx.saved_tensors
        shape, dtype = ctx.s_meta
        gl = (2.0 * grad_out.to(g.real.dtype)[:, None] * g).to(dtype)
        if ctx.block is None:
            return gl, None, None, None, None, None
        gs = torch.zeros(shape, dtype=dtype, device=g.device)
        gs[ctx.block[0]:ctx.block[1]] = gl
        return gs, None, None, None, None, None


def sharded_af_loss(s, M, spec, shard="delay", group=None, backend=None):
    """ShardedAFLoss.apply with keyword defaults (see the class)."""
    return ShardedAFLoss.apply(s, M, spec, shard, group, backend)
