"""ctypes binding of include/pintlab_b200.h (lib/libpintlab_b200.so).

The product path has no fallback: if the library is missing this module
raises on first use, and every CUDA failure surfaces as an exception.
Status codes map to the reference's exception types (multigrid.py:77-83,
sdc.py:75-81): PL_ERR_MGCAP -> MultigridError, negative -> ValueError /
NotImplementedError, PL_ERR_CUDA -> RuntimeError.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from ._build import LIB

PL_OK, PL_ERR_MGCAP, PL_ERR_CUDA = 0, 1, 2
PL_ERR_ARG, PL_ERR_UNSUPPORTED, PL_ERR_STATE = -1, -2, -3
PL_MAX_NODES = 17
SMOOTHERS = {"jacobi": 0, "gauss-seidel": 1, "jor-rb": 2}
RESTRICT = {"full-weighting": 0, "inject": 1, "copy": 2}
STATUS = {0: "fixed", 1: "converged", 2: "stalled", 3: "direct"}
NUM_KINDS = 17          # refreshed from the library by num_kinds()

_lib = None
_lock = threading.Lock()

dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)
vp = C.c_void_p
i32, i64, f64, sz = C.c_int, C.c_longlong, C.c_double, C.c_size_t


class SweepDesc(C.Structure):
    _fields_ = [("m", C.c_int),
                ("qdelta", C.c_double * (PL_MAX_NODES * PL_MAX_NODES)),
                ("gammas", C.c_double * PL_MAX_NODES),
                ("policy", C.c_int),
                ("fixed_cycles", C.c_int),
                ("tol", C.c_double),
                ("stall", C.c_double),
                ("max_cycles", C.c_int)]


_SIGS = {
    "pl_abi_version": (i32, []),
    "pl_last_error": (C.c_char_p, []),
    "pl_set_option": (i32, [i32, i32]),
    "pl_field_elems": (i64, [i32, i32]),
    "pl_heat_apply": (i32, [vp, vp, i32, i32, f64, f64, i32, vp]),
    "pl_heat_diagonal": (i32, [vp, i32, i32, f64, f64, i32, f64, i32, vp]),
    "pl_shifted_apply": (i32, [vp, vp, i32, i32, f64, f64, i32, f64, vp]),
    "pl_full_weighting": (i32, [vp, vp, i32, i32, vp]),
    "pl_inject": (i32, [vp, vp, i32, i32, vp]),
    "pl_interp_linear": (i32, [vp, vp, i32, i32, i32, vp]),
    "pl_interp_cubic_scratch_bytes": (sz, [i32, i32]),
    "pl_interp_cubic": (i32, [vp, vp, i32, i32, i32, vp, vp]),
    "pl_mg_workspace_bytes": (sz, [i32, i32, i32]),
    "pl_mg_plan_create": (i32, [C.POINTER(vp), i32, i32, f64, f64, i32, i32, f64, i32, i32,
                                i32, vp, sz]),
    "pl_mg_plan_destroy": (i32, [vp]),
    "pl_mg_prepare": (i32, [vp, f64, vp]),
    "pl_mg_set_coarsest_lu": (i32, [vp, f64, dp, ip, vp]),
    "pl_mg_coarsest_size": (i32, [vp]),
    "pl_mg_smooth": (i32, [vp, vp, vp, f64, i32, vp]),
    "pl_mg_vcycles": (i32, [vp, vp, vp, f64, i32, i32, vp]),
    "pl_mg_solve_tol": (i32, [vp, vp, vp, f64, f64, f64, i32, ip, ip, dp, vp]),
    "pl_sweep_workspace_bytes": (sz, [i32, i32, i32]),
    "pl_mg_set_direct": (i32, [vp, dp, dp, dp, dp, dp, vp]),
    "pl_mg_direct": (i32, [vp, vp, vp, f64, vp]),
    "pl_sdc_sweep": (i32, [vp, C.POINTER(SweepDesc), vp, vp, vp, vp, f64, vp, sz, ip, ip, ip,
                           ip, dp, ip, vp]),
    "pl_sdc_residual": (i32, [vp, vp, vp, vp, dp, i32, f64, i32, i32, vp, vp]),
    "pl_restrict_state": (i32, [vp, ip, i32, vp, vp, i32, i32, i32, i32, f64, f64, i32, vp]),
    "pl_compute_fas": (i32, [vp, vp, i32, dp, ip, i32, vp, dp, i32, f64, vp, vp, i32, i32, i32,
                             i32, vp]),
    "pl_compute_fas_scratch_bytes": (sz, [i32, i32, i32]),
    "pl_coarse_correction": (i32, [vp, vp, i32, vp, vp, i32, dp, i32, i32, i32, i32, f64, f64,
                                   i32, vp, vp]),
    "pl_coarse_correction_scratch_bytes": (sz, [i32, i32, i32, i32, i32]),
    "pl_stats_reset": (i32, []),
    "pl_stats_get": (i32, [C.POINTER(i64), dp, i32]),
    "pl_timing_enable": (i32, [C.c_uint]),
    "pl_timing_collect": (i32, [i32, C.POINTER(i64), dp, dp]),
    "pl_timing_dump": (i32, [i32, i64, dp, C.POINTER(C.c_float), C.POINTER(i64)]),
    "pl_kind_name": (C.c_char_p, [i32]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load the shared library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB):
                raise RuntimeError(
                    f"CUDA library {LIB} is missing: run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            h = C.CDLL(LIB)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            if h.pl_abi_version() != 2:
                raise RuntimeError("ABI version mismatch")
            _lib = h
    return _lib


def num_kinds():
    """Number of kernel kinds the loaded library reports (pl_kind_name)."""
    global NUM_KINDS
    h = lib()
    k = 0
    while k < 64 and h.pl_kind_name(k).decode() != "?":
        k += 1
    NUM_KINDS = k
    return k


class MultigridErrorBase(RuntimeError):
    pass


OPT_ZMARCH = 0
OPT_ZMARCH_MIN_N = 1
OPT_GRAPHS = 2
OPT_FUSE_PROLONG = 4
OPT_MID = 6
OPT_MID_TAIL_N = 7
OPT_RFW = 8
OPT_ZC_FLOOR = 9
OPT_FAST_TAIL = 10
OPT_ZC_CTAS = 11
OPT_MID_CTAS = 13
OPT_ZRB_RING = 14
OPT_FUSE_APPLY_RHS = 17
OPT_ZREV = 19
OPT_FUSE_FAS_FW = 20
OPT_ZC_FIT = 22
OPT_TOL_DEVICE = 24


_OPTION_VALUES = {}      # options set through this module (the library defaults otherwise)


def set_option(key, value):
    check(lib().pl_set_option(key, int(value)), "set_option")
    _OPTION_VALUES[key] = int(value)


class option:
    """Scoped pl_set_option: ``with option(OPT_MID_CTAS, 32): ...`` restores the
    previous value (or ``default``) on exit."""

    def __init__(self, key, value, default):
        self.key, self.value, self.default = key, int(value), default

    def __enter__(self):
        self.prev = _OPTION_VALUES.get(self.key, self.default)
        set_option(self.key, self.value)
        return self

    def __exit__(self, *exc):
        set_option(self.key, self.prev)
        return False


def last_error():
    return lib().pl_last_error().decode(errors="replace")


def check(rc, what=""):
    if rc == PL_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == PL_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc < 0:
        raise ValueError(msg)
    raise RuntimeError(msg)


def stats():
    """(launches, alg_bytes) per kernel kind since the last reset."""
    nk = num_kinds()
    n = (i64 * nk)()
    b = (f64 * nk)()
    lib().pl_stats_get(n, b, nk)
    names = [lib().pl_kind_name(k).decode() for k in range(nk)]
    return {names[k]: (int(n[k]), float(b[k])) for k in range(nk)}


def stats_reset():
    lib().pl_stats_reset()


def kind_index(name):
    for k in range(num_kinds()):
        if lib().pl_kind_name(k).decode() == name:
            return k
    raise KeyError(name)


def kind_names():
    return [lib().pl_kind_name(k).decode() for k in range(num_kinds())]


def timing_enable(names):
    """Record CUDA events around every launch of the given kernel kinds
    (None / empty: off)."""
    mask = 0
    for n in names or ():
        mask |= 1 << kind_index(n)
    lib().pl_timing_enable(mask)


def timing_by_size(name, nmax=1 << 20):
    """{alg_bytes_per_launch: (launches, total_ms)} for one kind: separates
    the multigrid levels (each level has its own byte count)."""
    b = (f64 * nmax)()
    t = (C.c_float * nmax)()
    n = i64(0)
    check(lib().pl_timing_dump(kind_index(name), nmax, b, t, C.byref(n)))
    out = {}
    for i in range(n.value):
        k = b[i]
        c, s = out.get(k, (0, 0.0))
        out[k] = (c + 1, s + t[i])
    return out


def timing_collect(name):
    """(launches, total_ms, alg_bytes) for one kind since timing_enable."""
    n, t, b = i64(0), f64(0), f64(0)
    check(lib().pl_timing_collect(kind_index(name), C.byref(n), C.byref(t), C.byref(b)))
    return int(n.value), float(t.value), float(b.value)
