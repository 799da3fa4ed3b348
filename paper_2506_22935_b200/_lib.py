"""ctypes view of libgraf.so (include/graf.h).  Loads the in-tree library and
fails loudly when it is missing: there is no CPU fallback."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int32, c_int64, c_size_t, c_void_p, c_char_p

PKG = os.path.dirname(os.path.abspath(__file__))
# GRAF_LIB_PATH: tuning builds only (scripts/tune.py); the default is the in-tree library.
LIB_PATH = os.environ.get("GRAF_LIB_PATH") or os.path.join(PKG, "libgraf.so")

ABI_VERSION = 6
GRAF_OK, GRAF_EINVAL, GRAF_EUNSUPPORTED, GRAF_ECUDA, GRAF_EWORKSPACE = 0, 1, 2, 3, 5
OUT_NONE, OUT_C64, OUT_ABS_F32, OUT_POW_F32 = range(4)
DOPPLER_RAW, DOPPLER_CENTERED = 0, 1

EXPORTS = ("graf_abi_version", "graf_status_string", "graf_last_error", "graf_workspace_bytes",
           "graf_af_forward", "graf_af_loss_grad", "graf_af_backward", "graf_combine_partials",
           "graf_set_profile_events", "graf_last_launch_count", "graf_spectral_variance",
           "graf_phase_adam_step", "graf_xaf_workspace_bytes", "graf_xaf_forward", "graf_xaf_loss_grad",
           "graf_xaf_backward", "graf_mainlobe_width", "graf_af_single_pass_eligible",
           "graf_af_loss_grad_sp_begin", "graf_af_loss_grad_sp_end", "graf_init", "graf_probe_fp32",
           "graf_plan_ctas_per_waveform")


class AfDesc(ctypes.Structure):
    _fields_ = [("abi_version", c_int32), ("n", c_int32), ("m", c_int32), ("out_kind", c_int32),
                ("batch", c_int64), ("k_begin", c_int32), ("k_end", c_int32),
                ("doppler_layout", c_int32), ("normalize_output", c_int32),
                ("shard_index", c_int32), ("shard_count", c_int32), ("periodic", c_int32),
                ("skip", c_void_p)]


class LossDesc(ctypes.Structure):
    _fields_ = [("k_max", c_int32), ("d_max", c_int32), ("ml_k", c_int32), ("ml_d", c_int32),
                ("w_k", c_void_p), ("w_d", c_void_p),
                ("lambda_isl", c_float), ("lambda_psl", c_float), ("temperature", c_float),
                ("normalize", c_int32), ("lambda_hpsl", c_float), ("lambda_match", c_float),
                ("target", c_void_p), ("target_stride", c_int64)]


class Partials(ctypes.Structure):
    _fields_ = [("isl_sum", c_double), ("lse_max", c_double), ("lse_sum", c_double), ("cen_sum", c_double),
                ("psl_key", c_double), ("reserved", c_double)]


class GrafError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"graf status {status}: {msg}")
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: the CUDA library is not built "
                              "(run `python -c 'import __graft_entry__ as g; g.build()'`). "
                              "There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        L.graf_abi_version.restype = c_int32
        L.graf_status_string.restype = c_char_p
        L.graf_status_string.argtypes = [c_int32]
        L.graf_last_error.restype = c_char_p
        L.graf_workspace_bytes.restype = c_size_t
        L.graf_workspace_bytes.argtypes = [POINTER(AfDesc), POINTER(LossDesc)]
        L.graf_af_forward.restype = c_int32
        L.graf_af_forward.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_size_t, c_void_p]
        L.graf_af_loss_grad.restype = c_int32
        L.graf_af_loss_grad.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p,
                                        c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
        L.graf_af_backward.restype = c_int32
        L.graf_af_backward.argtypes = [POINTER(AfDesc), c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                       c_void_p]
        L.graf_af_single_pass_eligible.restype = c_int32
        L.graf_af_single_pass_eligible.argtypes = [POINTER(AfDesc), POINTER(LossDesc)]
        L.graf_af_loss_grad_sp_begin.restype = c_int32
        L.graf_af_loss_grad_sp_begin.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p,
                                                 c_size_t, c_void_p]
        L.graf_af_loss_grad_sp_end.restype = c_int32
        L.graf_af_loss_grad_sp_end.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p,
                                               c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
        L.graf_combine_partials.restype = c_int32
        L.graf_combine_partials.argtypes = [POINTER(LossDesc), c_void_p, c_int32, c_int64, c_void_p, c_int32,
                                            c_void_p]
        L.graf_xaf_workspace_bytes.restype = c_size_t
        L.graf_xaf_workspace_bytes.argtypes = [POINTER(AfDesc), POINTER(LossDesc)]
        L.graf_xaf_forward.restype = c_int32
        L.graf_xaf_forward.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_size_t, c_void_p]
        L.graf_xaf_loss_grad.restype = c_int32
        L.graf_xaf_loss_grad.argtypes = [POINTER(AfDesc), POINTER(LossDesc), c_void_p, c_void_p, c_void_p, c_void_p,
                                         c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]
        L.graf_xaf_backward.restype = c_int32
        L.graf_xaf_backward.argtypes = [POINTER(AfDesc), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                        c_size_t, c_void_p]
        L.graf_mainlobe_width.restype = c_int32
        L.graf_mainlobe_width.argtypes = [c_int64, c_int32, c_void_p, c_float, c_float, c_int32, c_void_p, c_void_p,
                                          c_int32, c_void_p]
        L.graf_spectral_variance.restype = c_int32
        L.graf_spectral_variance.argtypes = [c_int64, c_int32, c_void_p, c_float, c_void_p, c_void_p, c_void_p,
                                             c_int32, c_int32, c_void_p]
        L.graf_init.restype = c_int32
        L.graf_init.argtypes = [c_void_p]
        L.graf_probe_fp32.restype = c_int32
        L.graf_probe_fp32.argtypes = [c_void_p, c_int32, POINTER(c_double), c_void_p]
        L.graf_phase_adam_step.restype = c_int32
        L.graf_phase_adam_step.argtypes = [c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           c_void_p, c_float, c_float, c_float, c_float, c_void_p]
        L.graf_plan_ctas_per_waveform.restype = c_int32
        L.graf_plan_ctas_per_waveform.argtypes = [c_int32, c_int32, c_int64, c_int32, c_int32, c_int32]
        L.graf_last_launch_count.restype = c_int32
        L.graf_last_launch_count.argtypes = []
        L.graf_set_profile_events.restype = c_int32
        L.graf_set_profile_events.argtypes = [c_void_p, c_void_p]
        if L.graf_abi_version() != ABI_VERSION:
            raise ImportError(f"libgraf ABI {L.graf_abi_version()} != {ABI_VERSION}")
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != GRAF_OK:
        L = lib()
        raise GrafError(status, f"{L.graf_status_string(status).decode()} — {L.graf_last_error().decode()}")
