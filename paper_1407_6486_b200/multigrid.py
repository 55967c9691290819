"""Geometric multigrid for (I - sigma nu Lap_h) u = b  (multigrid.py).

Same configuration objects, policies and results as the reference; the
V-cycle itself runs inside lib/libpintlab_b200.so (csrc/mg.cu): grid-wide
HBM-streaming kernels on the fine levels and one single-CTA shared-memory
kernel for the latency-bound tail (coarse levels + dense LU on n <= 4).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Union

import numpy as np
import scipy.linalg
import torch

from . import _capi as capi
from ._device import (clone_field, device, like_input, new_field, ptr, require_field,
                      stream_ptr, to_device)
from .heat import Grid, HeatOperator


@dataclass(frozen=True)
class MgConfig:
    """multigrid.py:24-38."""

    smoother: str = "jacobi"   # jacobi | gauss-seidel | jor-rb
    omega: float = 2.0 / 3.0
    pre_sweeps: int = 2
    post_sweeps: int = 2
    coarsest_n: int = 4

    def __post_init__(self):
        if self.smoother not in ("jacobi", "gauss-seidel", "jor-rb"):
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.pre_sweeps < 0 or self.post_sweeps < 0:
            raise ValueError("sweep counts must be non-negative")
        if self.coarsest_n < 2:
            raise ValueError("coarsest grid needs at least one interior point")


@dataclass(frozen=True)
class FixedCycles:
    """multigrid.py:41-47."""

    cycles: int

    def __post_init__(self):
        if self.cycles < 1:
            raise ValueError("need at least one V-cycle")


@dataclass(frozen=True)
class ToTolerance:
    """multigrid.py:50-60."""

    tol: float = 1e-12
    stall: float = 0.75
    max_cycles: int = 100

    def __post_init__(self):
        if self.tol <= 0:
            raise ValueError("tolerance must be positive")
        if not 0.0 < self.stall < 1.0:
            raise ValueError("stall factor must be in (0, 1)")


@dataclass(frozen=True)
class Direct:
    """Exact solve (multigrid.py:63-65).  The reference factors the sparse
    shifted matrix with SuperLU; the GPU path diagonalises the Kronecker sum
    (pl_mg_direct: dense cuBLAS GEMMs along each axis and a point-wise scale),
    equal to rounding."""


SolvePolicy = Union[FixedCycles, ToTolerance, Direct]


class MultigridError(RuntimeError):
    """Tolerance solve hit the cycle cap (multigrid.py:77-83)."""

    def __init__(self, message, residual, cycles):
        super().__init__(message)
        self.residual = residual
        self.cycles = cycles


class _Plan:
    """Device workspace + C plan for one (operator, MgConfig, stream)."""

    def __init__(self, op: HeatOperator, cfg: MgConfig):
        g = op.grid
        lib = capi.lib()
        nbytes = lib.pl_mg_workspace_bytes(g.dim, g.n, cfg.coarsest_n)
        self.ws = torch.zeros(max(nbytes, 8), dtype=torch.uint8, device=device())
        h = C.c_void_p()
        capi.check(lib.pl_mg_plan_create(C.byref(h), g.dim, g.n, float(g.length), float(op.nu),
                                         op.order, capi.SMOOTHERS[cfg.smoother],
                                         float(cfg.omega), cfg.pre_sweeps, cfg.post_sweeps,
                                         cfg.coarsest_n, self.ws.data_ptr(), nbytes),
                   "MG plan")
        self.handle = h
        self.op, self.cfg = op, cfg
        self._factored = set()
        n = g.n
        while n > cfg.coarsest_n and n >= 4:
            n //= 2
        self.coarsest = HeatOperator(Grid(g.dim, n, g.length), op.nu, op.order)

    def ensure(self, sigma: float):
        """Factor the coarsest-grid system I - sigma A once per sigma with the
        reference's own LAPACK call (scipy.linalg.lu_factor, multigrid.py:
        161-164) and install the factors; the solve itself runs on the GPU."""
        sigma = float(sigma)
        if sigma in self._factored:
            return
        lu, piv = scipy.linalg.lu_factor(_dense_shifted(self.coarsest, sigma))
        lu = np.ascontiguousarray(lu)
        piv = np.ascontiguousarray(piv, dtype=np.int32)
        capi.check(capi.lib().pl_mg_set_coarsest_lu(
            self.handle.value, sigma, lu.ctypes.data_as(C.POINTER(C.c_double)),
            piv.ctypes.data_as(C.POINTER(C.c_int)), stream_ptr()), "coarsest LU")
        self._factored.add(sigma)

    def ensure_direct(self):
        """Install the eigen-decomposition T = V diag(lam) V^-1 of the 1-D
        stencil matrix (the reference's entries, multigrid.py:86-107) for the
        Direct policy: numpy eigh for the symmetric order-2 matrix, eig + inv
        for order 4 (boundary rows make it non-symmetric).  Host setup, like
        the coarsest LU; the solves run on the GPU."""
        if getattr(self, "_direct", False):
            return
        g = self.op.grid
        t = _laplacian_1d(g.n, g.length, self.op.order)
        if self.op.order == 2:
            lam, v = np.linalg.eigh(t)
            w = v.T.copy()
        else:
            lam, v = np.linalg.eig(t)
            if np.max(np.abs(lam.imag)) > 1e-9 * np.max(np.abs(lam.real)):
                raise RuntimeError("order-4 stencil matrix has complex eigenvalues")
            lam, v = lam.real.copy(), v.real.copy()
            w = np.linalg.inv(v)
        arrs = [np.ascontiguousarray(a, dtype=np.float64)
                for a in (w, w.T, v, v.T, lam)]
        dp = C.POINTER(C.c_double)
        capi.check(capi.lib().pl_mg_set_direct(self.handle.value,
                                               *[a.ctypes.data_as(dp) for a in arrs],
                                               stream_ptr()), "direct factors")
        self._direct = True

    def __del__(self):
        try:
            if self.handle:
                capi.lib().pl_mg_plan_destroy(self.handle)
        except Exception:
            pass


_plans: dict = {}


def _laplacian_1d(n, length, order):
    """Dense 1-D nu-free stencil matrix with the reference's entry values
    (multigrid.py:86-107)."""
    dx2 = (length / n) ** 2
    npts = n - 1
    a = np.zeros((npts, npts))
    for i in range(npts):
        if order == 2 or i in (0, npts - 1):
            a[i, i] = -2.0 / dx2
            if i > 0:
                a[i, i - 1] = 1.0 / dx2
            if i < npts - 1:
                a[i, i + 1] = 1.0 / dx2
        else:
            for off, w in ((-2, -1.0), (-1, 16.0), (0, -30.0), (1, 16.0), (2, -1.0)):
                if 0 <= i + off < npts:
                    a[i, i + off] = w / (12.0 * dx2)
    return a


def _dense_shifted(op: HeatOperator, sigma: float):
    """I - sigma * nu * (Kronecker sum of the 1-D stencils, axis order)
    (multigrid.py:110-135); dense, only for the <= 3^d coarsest grid."""
    g = op.grid
    d1 = _laplacian_1d(g.n, g.length, op.order)
    eye = np.eye(g.n - 1)
    total = None
    for axis in range(g.dim):
        term = None
        for k in range(g.dim):
            f = d1 if k == axis else eye
            term = f if term is None else np.kron(term, f)
        total = term if total is None else total + term
    return np.eye(total.shape[0]) - sigma * (op.nu * total)


def plan_for(op: HeatOperator, cfg: MgConfig) -> _Plan:
    key = (op.grid, float(op.nu), op.order, cfg, stream_ptr(), torch.cuda.current_device())
    p = _plans.get(key)
    if p is None:
        p = _Plan(op, cfg)
        _plans[key] = p
    return p


class ShiftedOperator:
    """I - sigma * A for the heat operator (multigrid.py:178-208)."""

    def __init__(self, base: HeatOperator, sigma: float):
        if sigma < 0:
            raise ValueError("shift must be non-negative")
        self.base = base
        self.sigma = sigma

    @property
    def grid(self) -> Grid:
        return self.base.grid

    def apply(self, u):
        g = self.base.grid
        t, host = to_device(u, g.dim)
        out = new_field(g.shape)
        capi.check(capi.lib().pl_shifted_apply(ptr(t), ptr(out), g.dim, g.n, float(g.length),
                                               float(self.base.nu), self.base.order,
                                               float(self.sigma), stream_ptr()),
                   "ShiftedOperator.apply")
        return like_input(out, host)

    def diagonal(self, as_numpy: bool = True):
        g = self.base.grid
        out = new_field(g.shape)
        capi.check(capi.lib().pl_heat_diagonal(ptr(out), g.dim, g.n, float(g.length),
                                               float(self.base.nu), self.base.order,
                                               float(self.sigma), 1, stream_ptr()),
                   "ShiftedOperator.diagonal")
        return like_input(out, as_numpy)

    def solve_direct(self, b):
        """multigrid.py:203-208: (I - sigma A)^-1 b."""
        g = self.base.grid
        tb, host = to_device(b, g.dim)
        out = new_field(g.shape)
        direct_into(self, out, tb, MgConfig())
        return like_input(out, host)


def direct_into(op: "ShiftedOperator", u, b, cfg: MgConfig):
    """u = (I - sigma A)^-1 b on the device (Direct policy)."""
    require_field(u, op.grid.dim, "direct(u)")
    require_field(b, op.grid.dim, "direct(b)")
    p = plan_for(op.base, cfg)
    p.ensure_direct()
    capi.check(capi.lib().pl_mg_direct(p.handle.value, ptr(u), ptr(b), float(op.sigma),
                                       stream_ptr()), "direct solve")
    return u


def _check_policy(policy):
    if not isinstance(policy, (FixedCycles, ToTolerance, Direct)):
        raise ValueError(f"unknown solve policy {policy!r}")


def smooth(op: ShiftedOperator, u, b, cfg: MgConfig, count: int):
    """multigrid.py:211-234 (returns a new array, like the reference)."""
    if tuple(np.shape(u)) != tuple(np.shape(b)):
        raise ValueError("shape mismatch between iterate and right-hand side")
    d = op.grid.dim
    tu, host = to_device(u, d)
    tb, _ = to_device(b, d)
    out = clone_field(tu)
    if count:
        p = plan_for(op.base, cfg)
        capi.check(capi.lib().pl_mg_smooth(p.handle.value, ptr(out), ptr(tb), float(op.sigma),
                                           count, stream_ptr()), "smooth")
    return like_input(out, host)


def vcycles_into(op: ShiftedOperator, u, b, cfg: MgConfig, ncycles: int, zero_guess=False):
    """ncycles V-cycles in place on the device tensor u."""
    require_field(u, op.grid.dim, "vcycles_into(u)")
    require_field(b, op.grid.dim, "vcycles_into(b)")
    p = plan_for(op.base, cfg)
    p.ensure(op.sigma)
    capi.check(capi.lib().pl_mg_vcycles(p.handle.value, ptr(u), ptr(b), float(op.sigma),
                                        ncycles, int(zero_guess), stream_ptr()), "v_cycle")
    return u


def v_cycle(op: ShiftedOperator, u, b, cfg: MgConfig):
    """multigrid.py:237-251 (returns a new array)."""
    d = op.grid.dim
    tu, host = to_device(u, d)
    tb, _ = to_device(b, d)
    out = clone_field(tu)
    vcycles_into(op, out, tb, cfg, 1)
    return like_input(out, host)


@dataclass
class SolveResult:
    """multigrid.py:254-258."""

    u: object
    cycles: int
    status: str  # fixed | converged | stalled


def solve_into(op: ShiftedOperator, u, b, cfg: MgConfig, policy) -> tuple:
    """In-place device solve; returns (cycles, status).  Raises MultigridError."""
    _check_policy(policy)
    require_field(u, op.grid.dim, "solve_into(u)")
    require_field(b, op.grid.dim, "solve_into(b)")
    if isinstance(policy, Direct):            # multigrid.py:263-264
        direct_into(op, u, b, cfg)
        return 0, "direct"
    if isinstance(policy, FixedCycles):
        vcycles_into(op, u, b, cfg, policy.cycles)
        return policy.cycles, "fixed"
    p = plan_for(op.base, cfg)
    p.ensure(op.sigma)
    cyc, st, res = C.c_int(0), C.c_int(0), C.c_double(0)
    rc = capi.lib().pl_mg_solve_tol(p.handle.value, ptr(u), ptr(b), float(op.sigma),
                                    float(policy.tol), float(policy.stall), policy.max_cycles,
                                    C.byref(cyc), C.byref(st), C.byref(res), stream_ptr())
    if rc == capi.PL_ERR_MGCAP:
        raise MultigridError(capi.last_error(), res.value, cyc.value)
    capi.check(rc, "solve")
    return cyc.value, capi.STATUS[st.value]


def solve(op: ShiftedOperator, u0, b, cfg: MgConfig, policy: SolvePolicy) -> SolveResult:
    """multigrid.py:261-288."""
    d = op.grid.dim
    tu, host = to_device(u0, d)
    tb, _ = to_device(b, d)
    out = clone_field(tu)
    cycles, status = solve_into(op, out, tb, cfg, policy)
    return SolveResult(like_input(out, host), cycles, status)
