"""Factor-2 spatial grid transfers on Dirichlet grids (transfers.py).

Interior-only arrays: fine index i = 1..nf-1 at array position i-1, coarse j
at fine index 2j.  All four run as sm_100a kernels (csrc/transfer.cu).
"""
from __future__ import annotations

from . import _capi as capi
from ._device import like_input, new_field, ptr, require_field, scratch, stream_ptr, to_device


def _fine_n(shape):
    dims = set(shape)
    if len(dims) != 1:
        raise ValueError("grid arrays must be cubic")
    return shape[0] + 1


def _restrict(u, fn):
    t, host = to_device(u)
    nf = _fine_n(tuple(t.shape))
    if nf < 4:
        raise ValueError("grid too small to coarsen")
    out = new_field((nf // 2 - 1,) * t.dim())
    capi.check(fn(ptr(t), ptr(out), t.dim(), nf, stream_ptr()))
    return like_input(out, host)


def full_weighting(u):
    """(1, 2, 1)/4 per dimension, axis 0 first (transfers.py:27-34)."""
    return _restrict(u, capi.lib().pl_full_weighting)


def inject(u):
    """Coarse point takes the coincident fine value (transfers.py:19-24)."""
    return _restrict(u, capi.lib().pl_inject)


def interp_linear_into(coarse, fine, accumulate):
    require_field(coarse, coarse.dim(), "interp_linear_into(coarse)")
    require_field(fine, coarse.dim(), "interp_linear_into(fine)")
    nf = 2 * (coarse.shape[0] + 1)
    capi.check(capi.lib().pl_interp_linear(ptr(coarse), ptr(fine), coarse.dim(), nf,
                                           int(accumulate), stream_ptr()), "interp_linear")
    return fine


def interp_cubic_into(coarse, fine, accumulate):
    require_field(coarse, coarse.dim(), "interp_cubic_into(coarse)")
    require_field(fine, coarse.dim(), "interp_cubic_into(fine)")
    nf = 2 * (coarse.shape[0] + 1)
    nb = capi.lib().pl_interp_cubic_scratch_bytes(coarse.dim(), nf)
    s = scratch("cubic", nb)
    capi.check(capi.lib().pl_interp_cubic(ptr(coarse), ptr(fine), coarse.dim(), nf,
                                          int(accumulate), s.data_ptr(), stream_ptr()),
               "interp_cubic")
    return fine


def _interp(u, fn):
    t, host = to_device(u)
    nf = 2 * (t.shape[0] + 1)
    out = new_field((nf - 1,) * t.dim())
    fn(t, out, False)
    return like_input(out, host)


def interp_linear(u):
    """Linear interpolation to the factor-2 finer grid (transfers.py:37-50)."""
    return _interp(u, interp_linear_into)


def interp_cubic(u):
    """Cubic interpolation with zero boundary samples (transfers.py:53-89)."""
    return _interp(u, interp_cubic_into)


def interp_space(u, order: int):
    """transfers.py:92-97."""
    if order == 2:
        return interp_linear(u)
    if order == 4:
        return interp_cubic(u)
    raise ValueError(f"spatial interpolation order must be 2 or 4, got {order}")
