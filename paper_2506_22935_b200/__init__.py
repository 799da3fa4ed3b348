"""B200-native (sm_100a) GRAF ambiguity-function hot path (arXiv 2506.22935).

Public API (thin binding of include/graf.h; all compute in libgraf.so):
    af_forward, af_loss_grad, af_backward, combine_partials, LossSpec,
    af / af_loss (torch autograd), sharding.* (torch.distributed layers),
    spectral_variance, phase_adam_step, LpiOptimizer (the paper's section-7 workload).
"""
from ._lib import GrafError, lib  # noqa: F401
from .graf import (AF, AFLoss, LossSpec, LpiOptimizer, af, af_backward, af_forward, af_loss,  # noqa: F401
                   af_loss_grad, combine_partials, phase_adam_step, spectral_variance, workspace_bytes,
                   mainlobe_width, xaf_backward, xaf_forward, xaf_loss_grad, single_pass_eligible,
                   af_loss_grad_sp_begin, af_loss_grad_sp_end)

__all__ = ["AF", "AFLoss", "LossSpec", "af", "af_backward", "af_forward", "af_loss", "af_loss_grad",
           "combine_partials", "workspace_bytes", "GrafError", "lib", "spectral_variance", "phase_adam_step",
           "LpiOptimizer", "xaf_forward", "xaf_loss_grad", "xaf_backward", "mainlobe_width",
           "single_pass_eligible", "af_loss_grad_sp_begin", "af_loss_grad_sp_end"]
