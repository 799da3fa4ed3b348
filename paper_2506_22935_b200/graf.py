"""Python binding of the GRAF C ABI (include/graf.h): argument marshalling only.

Every step of the path runs in libgraf.so's CUDA kernels; torch supplies device
memory, the current stream and (in `sharding.py`) process groups.  Function
names follow the ABI: af_forward, af_loss_grad, af_backward, combine_partials.

Gradient convention: the ABI returns g = dL/ds* (Wirtinger; SPEC.md L113-118,
PAPER.md L219).  torch's complex autograd carries 2*dL/ds*, so the autograd
Functions below multiply by 2 (SURVEY.md finding 7).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Tuple

import torch

from . import _lib as L

__all__ = ["LossSpec", "af_forward", "af_loss_grad", "af_backward", "combine_partials",
           "workspace_bytes", "AF", "AFLoss", "af", "af_loss"]

_OUT = {None: L.OUT_NONE, "none": L.OUT_NONE, "c64": L.OUT_C64, "abs": L.OUT_ABS_F32, "pow": L.OUT_POW_F32}
_LAYOUT = {"raw": L.DOPPLER_RAW, "centered": L.DOPPLER_CENTERED, "centred": L.DOPPLER_CENTERED}


@dataclass
class LossSpec:
    """graf_loss_desc (include/graf.h): region |k|<=k_max, |d|<=d_max minus the
    mainlobe |k|<=ml_k && |d|<=ml_d; L = lambda_isl*ISL + lambda_psl*softPSL + lambda_hpsl*PSL
    (hard PSL with its argmax subgradient, the paper's section-7 loss)."""
    k_max: int
    d_max: int
    ml_k: int = 0
    ml_d: int = 0
    lambda_isl: float = 1.0
    lambda_psl: float = 0.0
    temperature: float = 0.01
    normalize: int = 1
    lambda_hpsl: float = 0.0
    lambda_match: float = 0.0
    target: Optional[torch.Tensor] = None      # fp32 [rows, M] or [B, rows, M], surface-window layout
    w_k: Optional[torch.Tensor] = None   # device float32 [2N-1], symmetric
    w_d: Optional[torch.Tensor] = None   # device float32 [M], symmetric

    @classmethod
    def from_dict(cls, d: dict) -> "LossSpec":
        return cls(**{k: v for k, v in d.items() if k in cls.__dataclass_fields__})

    def desc(self) -> L.LossDesc:
        return L.LossDesc(int(self.k_max), int(self.d_max), int(self.ml_k), int(self.ml_d),
                          _ptr(self.w_k), _ptr(self.w_d), float(self.lambda_isl),
                          float(self.lambda_psl), float(self.temperature), int(self.normalize),
                          float(self.lambda_hpsl), float(self.lambda_match), _ptr(self.target),
                          int(self.target.shape[-1] * self.target.shape[-2]) if (self.target is not None and
                                                                                self.target.dim() == 3) else 0)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("graf: tensors must live on a CUDA device")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _check_s(s: torch.Tensor) -> torch.Tensor:
    if s.dtype != torch.complex64:
        raise TypeError("graf: s must be complex64")
    if not s.is_cuda:
        raise ValueError("graf: s must be a CUDA tensor (no CPU fallback)")
    if s.dim() == 1:
        s = s[None]
    return s.contiguous()


def _skip_ptr(skip: Optional[torch.Tensor], B: int):
    if skip is None:
        return None
    if skip.dtype != torch.int32 or not skip.is_cuda or skip.shape != (B,) or not skip.is_contiguous():
        raise ValueError("graf: skip must be a contiguous int32 CUDA tensor of shape [B]")
    return ctypes.c_void_p(skip.data_ptr())


def _desc(s: torch.Tensor, M: int, out=None, layout="centered", k_begin=None, k_end=None,
          normalize_output=False, shard=(0, 1), periodic=False, skip=None) -> L.AfDesc:
    B, N = s.shape
    if periodic:   # Alg. 1: delays 0..N-1 (mod N)
        kb = 0 if k_begin is None else int(k_begin)
    else:
        kb = -(N - 1) if k_begin is None else int(k_begin)
    ke = N if k_end is None else int(k_end)
    return L.AfDesc(L.ABI_VERSION, int(N), int(M), _OUT[out], int(B), kb, ke, _LAYOUT[layout],
                    int(bool(normalize_output)), int(shard[0]), int(shard[1]), int(bool(periodic)),
                    _skip_ptr(skip, B))


def workspace_bytes(desc: L.AfDesc, loss: Optional[L.LossDesc]) -> int:
    return int(L.lib().graf_workspace_bytes(ctypes.byref(desc), ctypes.byref(loss) if loss else None))


class Workspace:
    """Grow-only device workspace (the library never allocates)."""

    def __init__(self):
        self.buf: Optional[torch.Tensor] = None

    def get(self, nbytes: int, device) -> Tuple[int, int]:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf.data_ptr(), self.buf.numel()


_ws = Workspace()
NPART = 6   # doubles per graf_partials record


def _surface_alloc(desc: L.AfDesc, device) -> Optional[torch.Tensor]:
    if desc.out_kind == L.OUT_NONE:
        return None
    rows = desc.k_end - desc.k_begin
    dt = torch.complex64 if desc.out_kind == L.OUT_C64 else torch.float32
    return torch.empty((desc.batch, rows, desc.m), dtype=dt, device=device)


def af_forward(s: torch.Tensor, M: int, *, out: Optional[str] = "c64", layout: str = "centered",
               k_begin: Optional[int] = None, k_end: Optional[int] = None, normalize_output: bool = False,
               loss: Optional[LossSpec] = None, shard=(0, 1), ws: Optional[Workspace] = None,
               surface: Optional[torch.Tensor] = None, stream=None, periodic: bool = False,
               skip: Optional[torch.Tensor] = None, partials: Optional[torch.Tensor] = None):
    """graf_af_forward: surface window and/or this shard's loss partials [B,6] (float64).
    periodic=True: the paper's circular surface (Eq. 2 / Alg. 1), M == N.
    skip: int32 [B] device mask, waveforms with skip[b] != 0 are left untouched (ABI v6)."""
    s = _check_s(s)
    d = _desc(s, M, out, layout, k_begin, k_end, normalize_output, shard, periodic, skip)
    ld = loss.desc() if loss is not None else None
    if surface is None:
        surface = _surface_alloc(d, s.device)
    if partials is None and loss is not None:
        partials = torch.empty((s.shape[0], NPART), dtype=torch.float64, device=s.device)
    nbytes = workspace_bytes(d, ld)
    wp, wn = (ws or _ws).get(nbytes, s.device)
    L.check(L.lib().graf_af_forward(ctypes.byref(d), ctypes.byref(ld) if ld else None,
                                    ctypes.c_void_p(s.data_ptr()), _ptr(surface), _ptr(partials),
                                    ctypes.c_void_p(wp), wn, _stream(stream)))
    return surface, partials


def af_loss_grad(s: torch.Tensor, M: int, loss: LossSpec, *, global_partials: Optional[torch.Tensor] = None,
                 out: Optional[str] = None, layout: str = "centered", k_begin=None, k_end=None,
                 normalize_output: bool = False, shard=(0, 1), ws: Optional[Workspace] = None,
                 grad: Optional[torch.Tensor] = None, loss_out: Optional[torch.Tensor] = None,
                 surface: Optional[torch.Tensor] = None, want_loss: bool = True, stream=None,
                 periodic: bool = False, skip: Optional[torch.Tensor] = None):
    """graf_af_loss_grad -> (loss[B] float64, grad[B,N] complex64 = dL/ds*, surface or None).
    skip: int32 [B] device mask; the outputs of waveforms with skip[b] != 0 (in the given
    loss_out / grad buffers) are left untouched (ABI v6)."""
    s = _check_s(s)
    d = _desc(s, M, out, layout, k_begin, k_end, normalize_output, shard, periodic, skip)
    ld = loss.desc()
    B, N = s.shape
    if grad is None:
        grad = torch.empty((B, N), dtype=torch.complex64, device=s.device)
    if loss_out is None and want_loss:
        loss_out = torch.empty((B,), dtype=torch.float64, device=s.device)
    if surface is None:
        surface = _surface_alloc(d, s.device)
    if global_partials is not None:
        assert global_partials.dtype == torch.float64 and global_partials.shape == (B, NPART)
    nbytes = workspace_bytes(d, ld)
    wp, wn = (ws or _ws).get(nbytes, s.device)
    L.check(L.lib().graf_af_loss_grad(ctypes.byref(d), ctypes.byref(ld), ctypes.c_void_p(s.data_ptr()),
                                      _ptr(global_partials), _ptr(loss_out), ctypes.c_void_p(grad.data_ptr()),
                                      _ptr(surface), ctypes.c_void_p(wp), wn, _stream(stream)))
    return loss_out, grad, surface


def af_backward(s: torch.Tensor, M: int, dA: torch.Tensor, *, k_begin=None, k_end=None,
                layout: str = "centered", ws: Optional[Workspace] = None, stream=None,
                periodic: bool = False) -> torch.Tensor:
    """graf_af_backward: dL/ds* from dA = dL/dA* over rows [k_begin, k_end)."""
    s = _check_s(s)
    if dA.dtype != torch.complex64 or not dA.is_cuda:
        raise TypeError("graf: dA must be a complex64 CUDA tensor")
    dA = dA.contiguous()
    d = _desc(s, M, None, layout, k_begin, k_end, periodic=periodic)
    B, N = s.shape
    if dA.shape != (B, d.k_end - d.k_begin, M):
        raise ValueError(f"dA shape {tuple(dA.shape)} != {(B, d.k_end - d.k_begin, M)}")
    grad = torch.empty((B, N), dtype=torch.complex64, device=s.device)
    nbytes = workspace_bytes(d, None)
    wp, wn = (ws or _ws).get(nbytes, s.device)
    L.check(L.lib().graf_af_backward(ctypes.byref(d), ctypes.c_void_p(s.data_ptr()),
                                     ctypes.c_void_p(dA.data_ptr()), ctypes.c_void_p(grad.data_ptr()),
                                     ctypes.c_void_p(wp), wn, _stream(stream)))
    return grad


def single_pass_eligible(s: torch.Tensor, M: int, loss: LossSpec, shard=(0, 1), periodic: bool = False) -> bool:
    """graf_af_single_pass_eligible: the full-plane centred soft-PSL that runs as one pass."""
    d = _desc(s, M, None, "centered", None, None, False, shard, periodic)
    return bool(L.lib().graf_af_single_pass_eligible(ctypes.byref(d), ctypes.byref(loss.desc())))


def af_loss_grad_sp_begin(s: torch.Tensor, M: int, loss: LossSpec, shard, *, ws: Optional[Workspace] = None,
                          stream=None, periodic: bool = False) -> torch.Tensor:
    """graf_af_loss_grad_sp_begin: phase 1 of the delay-sharded single pass -> this
    shard's partials [B, 6] (float64).  `ws` must be passed unchanged to phase 2."""
    s = _check_s(s)
    d = _desc(s, M, None, "centered", None, None, False, shard, periodic)
    ld = loss.desc()
    partials = torch.empty((s.shape[0], NPART), dtype=torch.float64, device=s.device)
    wp, wn = (ws or _ws).get(workspace_bytes(d, ld), s.device)
    L.check(L.lib().graf_af_loss_grad_sp_begin(ctypes.byref(d), ctypes.byref(ld), ctypes.c_void_p(s.data_ptr()),
                                               ctypes.c_void_p(partials.data_ptr()), ctypes.c_void_p(wp), wn,
                                               _stream(stream)))
    return partials


def af_loss_grad_sp_end(s: torch.Tensor, M: int, loss: LossSpec, shard, global_partials: torch.Tensor, *,
                        ws: Optional[Workspace] = None, stream=None, periodic: bool = False):
    """graf_af_loss_grad_sp_end: phase 2 -> (loss [B] float64, this shard's grad [B,N]
    complex64, valid [B] int32).  Where valid is 0 the caller recomputes with two passes."""
    s = _check_s(s)
    d = _desc(s, M, None, "centered", None, None, False, shard, periodic)
    ld = loss.desc()
    B, N = s.shape
    assert global_partials.dtype == torch.float64 and global_partials.shape == (B, NPART)
    global_partials = global_partials.contiguous()
    lo = torch.empty((B,), dtype=torch.float64, device=s.device)
    g = torch.empty((B, N), dtype=torch.complex64, device=s.device)
    valid = torch.empty((B,), dtype=torch.int32, device=s.device)
    wp, wn = (ws or _ws).get(workspace_bytes(d, ld), s.device)
    L.check(L.lib().graf_af_loss_grad_sp_end(ctypes.byref(d), ctypes.byref(ld), ctypes.c_void_p(s.data_ptr()),
                                             ctypes.c_void_p(global_partials.data_ptr()),
                                             ctypes.c_void_p(lo.data_ptr()), ctypes.c_void_p(g.data_ptr()),
                                             ctypes.c_void_p(valid.data_ptr()), ctypes.c_void_p(wp), wn,
                                             _stream(stream)))
    return lo, g, valid


def combine_partials(loss: LossSpec, shards: torch.Tensor, stream=None) -> torch.Tensor:
    """graf_combine_partials: shards [G,B,6] float64 -> [B,6], in shard order."""
    G, B, npart = shards.shape
    assert npart == NPART and shards.dtype == torch.float64
    shards = shards.contiguous()
    out = torch.empty((B, NPART), dtype=torch.float64, device=shards.device)
    ld = loss.desc()
    if shards.is_cuda:
        L.check(L.lib().graf_combine_partials(ctypes.byref(ld), ctypes.c_void_p(shards.data_ptr()), G, B,
                                              ctypes.c_void_p(out.data_ptr()), 1, _stream(stream)))
    else:
        L.check(L.lib().graf_combine_partials(ctypes.byref(ld), ctypes.c_void_p(shards.data_ptr()), G, B,
                                              ctypes.c_void_p(out.data_ptr()), 0, None))
    return out


# ---------------------------------------------------------------------------
# torch autograd integration (§4.3 "Complex gradient handling", L274)
# ---------------------------------------------------------------------------
class AF(torch.autograd.Function):
    """Differentiable complex surface A (rows [k_begin,k_end), layout)."""

    @staticmethod
    def forward(ctx, s, M, layout="centered", k_begin=None, k_end=None, periodic=False):
        surf, _ = af_forward(s.detach(), M, out="c64", layout=layout, k_begin=k_begin, k_end=k_end,
                             periodic=periodic)
        ctx.save_for_backward(s)
        ctx.cfg = (M, layout, k_begin, k_end, s.dim(), periodic)
        return surf if s.dim() == 2 else surf[0]

    @staticmethod
    def backward(ctx, grad_out):
        (s,) = ctx.saved_tensors
        M, layout, kb, ke, dim, periodic = ctx.cfg
        g = grad_out if dim == 2 else grad_out[None]
        # torch hands 2*dL/dA*; the adjoint is linear, so the result is torch's 2*dL/ds*.
        gs = af_backward(s.detach(), M, g.to(torch.complex64), k_begin=kb, k_end=ke, layout=layout,
                         periodic=periodic)
        return (gs if dim == 2 else gs[0]), None, None, None, None, None


class AFLoss(torch.autograd.Function):
    """Per-waveform loss L_b (float64 [B]) with the fused kernels' gradient."""

    @staticmethod
    def forward(ctx, s, M, spec, periodic=False):
        lo, g, _ = af_loss_grad(s.detach(), M, spec, periodic=periodic)
        ctx.save_for_backward(g)
        ctx.dim = s.dim()
        return lo if s.dim() == 2 else lo[0]

    @staticmethod
    def backward(ctx, grad_out):
        (g,) = ctx.saved_tensors
        go = grad_out if ctx.dim == 2 else grad_out[None]
        gs = 2.0 * go.to(torch.float32)[:, None] * g          # torch .grad = 2 dL/ds*
        return (gs if ctx.dim == 2 else gs[0]), None, None, None


def af(s, M, layout="centered", k_begin=None, k_end=None, periodic=False):
    return AF.apply(s, M, layout, k_begin, k_end, periodic)


def af_loss(s, M, spec: LossSpec, periodic=False, *, shard=None, group=None, backend=None):
    """Differentiable per-waveform loss.  shard = None: one device; "delay" / "batch": the
    torch.distributed layers of sharding.py (ShardedAFLoss), aperiodic."""
    if shard is None:
        return AFLoss.apply(s, M, spec, periodic)
    if periodic:
        raise ValueError("the sharded losses run the aperiodic surface")
    from .sharding import sharded_af_loss
    return sharded_af_loss(s, M, spec, shard=shard, group=group, backend=backend)


# ---------------------------------------------------------------------------
# The paper's section-7 workload:
# L_b = PSL_b + lambda_b * alpha * SV_b on s = exp(j theta), Adam on theta.
# Every step is one of the library's kernels (hard-PSL pass, psl_grad, spectral
# variance, Adam); Python only marshals pointers and replays CUDA graphs.
# ---------------------------------------------------------------------------
def spectral_variance(s: torch.Tensor, weight: float = 1.0, weights: Optional[torch.Tensor] = None,
                      loss: Optional[torch.Tensor] = None, grad: Optional[torch.Tensor] = None,
                      accumulate: bool = False, ddof: int = 0, stream=None):
    """graf_spectral_variance -> (weight*SV [B] float64, weight*dSV/ds* [B,N] complex64);
    ddof = 0 population variance, 1 unbiased."""
    s = _check_s(s)
    B, N = s.shape
    if loss is None:
        loss = torch.zeros((B,), dtype=torch.float64, device=s.device)
    if grad is None:
        grad = torch.zeros((B, N), dtype=torch.complex64, device=s.device)
    if weights is not None:
        assert weights.dtype == torch.float32 and weights.is_cuda and weights.shape == (B,)
    L.check(L.lib().graf_spectral_variance(B, N, ctypes.c_void_p(s.data_ptr()), float(weight), _ptr(weights),
                                           _ptr(loss), ctypes.c_void_p(grad.data_ptr()), int(bool(accumulate)),
                                           int(ddof), _stream(stream)))
    return loss, grad


def phase_adam_step(theta, m, v, step, grad, s_out, lr=0.01, betas=(0.9, 0.999), eps=1e-8, stream=None):
    """graf_phase_adam_step: in place on theta/m/v/step [B,N] float32 / [B] int32; s_out = exp(j theta)."""
    B, N = theta.shape
    L.check(L.lib().graf_phase_adam_step(B, N, _ptr(theta), _ptr(m), _ptr(v), _ptr(step), _ptr(grad), _ptr(s_out),
                                         float(lr), float(betas[0]), float(betas[1]), float(eps), _stream(stream)))


class LpiOptimizer:
    """Batched section-7 optimisation: each waveform b has its own trade-off lambda_b
    (a lambda sweep x seeds is one batch).  One iteration = hard-PSL pass 1 +
    argmax subgradient + spectral variance (accumulated) + Adam, captured once as
    a CUDA graph of `per_graph` iterations and replayed."""

    def __init__(self, theta0: torch.Tensor, lam, spec: Optional[LossSpec] = None, alpha: float = 2000.0,
                 lr: float = 0.01, periodic: bool = True, per_graph: int = 50):
        self.theta = theta0.detach().to(torch.float32).contiguous().clone()
        B, N = self.theta.shape
        dev = self.theta.device
        self.spec = spec or LossSpec(k_max=N, d_max=N, lambda_isl=0.0, lambda_psl=0.0, normalize=1)
        self.spec.lambda_hpsl = 1.0
        self.spec.lambda_isl = 0.0
        self.spec.lambda_psl = 0.0
        lam = torch.as_tensor(lam, dtype=torch.float32, device=dev).expand(B).contiguous()
        self.weights = (lam * float(alpha)).contiguous()
        self.lr, self.periodic = lr, periodic
        self.m = torch.zeros_like(self.theta)
        self.v = torch.zeros_like(self.theta)
        self.step = torch.zeros((B,), dtype=torch.int32, device=dev)
        self.s = torch.polar(torch.ones_like(self.theta), self.theta).to(torch.complex64).contiguous()
        self.grad = torch.empty((B, N), dtype=torch.complex64, device=dev)
        self.loss = torch.empty((B,), dtype=torch.float64, device=dev)
        self.ws = Workspace()
        self.stream = torch.cuda.Stream(dev)
        self.per_graph = per_graph
        self.graph = None

    def _iteration(self):
        B, N = self.theta.shape
        af_loss_grad(self.s, N, self.spec, ws=self.ws, grad=self.grad, loss_out=self.loss, stream=self.stream,
                     periodic=self.periodic)
        spectral_variance(self.s, weights=self.weights, loss=self.loss, grad=self.grad, accumulate=True,
                          stream=self.stream)
        phase_adam_step(self.theta, self.m, self.v, self.step, self.grad, self.s, lr=self.lr, stream=self.stream)

    def run(self, iters: int) -> torch.Tensor:
        """Advance `iters` iterations; returns the loss [B] of the last one (float64)."""
        with torch.cuda.stream(self.stream):
            if self.graph is None:
                self._iteration()                              # workspace + twiddles, outside capture
                iters -= 1
                self.graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(self.graph, stream=self.stream):
                    for _ in range(self.per_graph):
                        self._iteration()
            while iters >= self.per_graph:
                self.graph.replay()
                iters -= self.per_graph
            for _ in range(iters):
                self._iteration()
        self.stream.synchronize()
        return self.loss


# ---------------------------------------------------------------------------
# Cross-ambiguity X[k,m] = sum_n s1[n] conj(s2[n-k]) W^{mn}
# ---------------------------------------------------------------------------
def xaf_forward(s1: torch.Tensor, s2: torch.Tensor, M: int, *, out: Optional[str] = "c64",
                layout: str = "centered", k_begin=None, k_end=None, normalize_output: bool = False,
                loss: Optional[LossSpec] = None, ws: Optional[Workspace] = None, surface=None, stream=None):
    """graf_xaf_forward: cross surface window and/or loss partials."""
    s1, s2 = _check_s(s1), _check_s(s2)
    assert s1.shape == s2.shape
    d = _desc(s1, M, out, layout, k_begin, k_end, normalize_output)
    ld = loss.desc() if loss is not None else None
    if surface is None:
        surface = _surface_alloc(d, s1.device)
    partials = torch.empty((s1.shape[0], NPART), dtype=torch.float64, device=s1.device) if loss is not None else None
    nbytes = int(L.lib().graf_xaf_workspace_bytes(ctypes.byref(d), ctypes.byref(ld) if ld else None))
    wp, wn = (ws or _ws).get(nbytes, s1.device)
    L.check(L.lib().graf_xaf_forward(ctypes.byref(d), ctypes.byref(ld) if ld else None,
                                     ctypes.c_void_p(s1.data_ptr()), ctypes.c_void_p(s2.data_ptr()), _ptr(surface),
                                     _ptr(partials), ctypes.c_void_p(wp), wn, _stream(stream)))
    return surface, partials


def xaf_loss_grad(s1: torch.Tensor, s2: torch.Tensor, M: int, loss: LossSpec, *, out: Optional[str] = None,
                  layout: str = "centered", k_begin=None, k_end=None, ws: Optional[Workspace] = None,
                  surface=None, stream=None):
    """graf_xaf_loss_grad -> (loss[B] float64, dL/ds1* [B,N], dL/ds2* [B,N], surface or None)."""
    s1, s2 = _check_s(s1), _check_s(s2)
    assert s1.shape == s2.shape
    d = _desc(s1, M, out, layout, k_begin, k_end)
    ld = loss.desc()
    B, N = s1.shape
    g1 = torch.empty((B, N), dtype=torch.complex64, device=s1.device)
    g2 = torch.empty_like(g1)
    lo = torch.empty((B,), dtype=torch.float64, device=s1.device)
    if surface is None:
        surface = _surface_alloc(d, s1.device)
    nbytes = int(L.lib().graf_xaf_workspace_bytes(ctypes.byref(d), ctypes.byref(ld)))
    wp, wn = (ws or _ws).get(nbytes, s1.device)
    L.check(L.lib().graf_xaf_loss_grad(ctypes.byref(d), ctypes.byref(ld), ctypes.c_void_p(s1.data_ptr()),
                                       ctypes.c_void_p(s2.data_ptr()), None, _ptr(lo), _ptr(g1), _ptr(g2),
                                       _ptr(surface), ctypes.c_void_p(wp), wn, _stream(stream)))
    return lo, g1, g2, surface


def xaf_backward(s1: torch.Tensor, s2: torch.Tensor, M: int, dA: torch.Tensor, *, k_begin=None, k_end=None,
                 layout: str = "centered", ws: Optional[Workspace] = None, stream=None):
    """graf_xaf_backward: (dL/ds1*, dL/ds2*) from dA = dL/dX* over rows [k_begin, k_end)."""
    s1, s2 = _check_s(s1), _check_s(s2)
    dA = dA.contiguous()
    d = _desc(s1, M, None, layout, k_begin, k_end)
    B, N = s1.shape
    g1 = torch.empty((B, N), dtype=torch.complex64, device=s1.device)
    g2 = torch.empty_like(g1)
    nbytes = int(L.lib().graf_xaf_workspace_bytes(ctypes.byref(d), None))
    wp, wn = (ws or _ws).get(nbytes, s1.device)
    L.check(L.lib().graf_xaf_backward(ctypes.byref(d), ctypes.c_void_p(s1.data_ptr()),
                                      ctypes.c_void_p(s2.data_ptr()), ctypes.c_void_p(dA.data_ptr()), _ptr(g1),
                                      _ptr(g2), ctypes.c_void_p(wp), wn, _stream(stream)))
    return g1, g2


def mainlobe_width(s: torch.Tensor, gamma: float, weight: float = 1.0, periodic: bool = False,
                   loss: Optional[torch.Tensor] = None, grad: Optional[torch.Tensor] = None,
                   accumulate: bool = False, stream=None):
    """graf_mainlobe_width -> (weight*W [B] float64, weight*dW/ds* [B,N] complex64)."""
    s = _check_s(s)
    B, N = s.shape
    if loss is None:
        loss = torch.zeros((B,), dtype=torch.float64, device=s.device)
    if grad is None:
        grad = torch.zeros((B, N), dtype=torch.complex64, device=s.device)
    L.check(L.lib().graf_mainlobe_width(B, N, ctypes.c_void_p(s.data_ptr()), float(gamma), float(weight),
                                        int(bool(periodic)), _ptr(loss), ctypes.c_void_p(grad.data_ptr()),
                                        int(bool(accumulate)), _stream(stream)))
    return loss, grad
