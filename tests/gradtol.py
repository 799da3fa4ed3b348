"""The gradient gate of the GPU parity tests (north star: "loss and gradient within 1e-4
relative"; VERDICT r1 "what's weak" 1 and 9).

Plain relative: max|g_gpu - g_ref| <= 1e-4 max|g_ref|.  The one exception is a gradient
that is identically zero in exact arithmetic -- the normalised full-plane ISL, constant
M - 1 by the volume identity (reading R12) -- where the float64 oracle's
g_ref is itself rounding noise of the cancelling terms; it is recognised by
max|g_ref| <= 1e-6 sigma_g (sigma_g = (2/E^3)|sum f' chi| max|s|, the size of those terms)
and gated at 1e-4 sigma_g, i.e. "zero to within the terms' fp32 rounding".
"""
import numpy as np


def grad_tol(g_ref, sigma_g, rel=1e-4):
    gmax = float(np.abs(g_ref).max()) if np.size(g_ref) else 0.0
    if gmax <= 1e-6 * sigma_g:
        return rel * sigma_g
    return rel * gmax
