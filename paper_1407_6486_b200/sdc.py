"""Single-level SDC sweeps with multigrid sub-step solves (sdc.py).

``sdc_sweep`` is ONE native call (pl_sdc_sweep): the node-to-node quadrature
as a single streaming pass over the M+1 nodal fields, then per sub-step the
right-hand side, the V-cycles and the f refresh -- all on the caller's CUDA
stream, no host round trip for FixedCycles.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _capi as capi
from ._device import clone_field, new_field, ptr, scratch, stream_ptr, to_device, zeros
from .heat import HeatOperator
from .multigrid import (Direct, FixedCycles, MgConfig, MultigridError, SolvePolicy,
                        ToTolerance, _check_policy, plan_for)
from .quadrature import QuadratureTable


class NodeStates:
    """Values y and cached f = A y at all M+1 nodes (sdc.py:24-47), stored as
    fp64 CUDA tensors of shape (M+1, *grid.shape)."""

    __slots__ = ("table", "y", "f")

    def __init__(self, table: QuadratureTable, y, f):
        self.table = table
        self.y = to_device(y, np.ndim(y) - 1)[0]
        self.f = to_device(f, np.ndim(f) - 1)[0]

    @classmethod
    def spread(cls, op: HeatOperator, table: QuadratureTable, y0) -> "NodeStates":
        t, _ = to_device(y0, op.grid.dim)
        shape = tuple(t.shape)
        y = new_field(shape, (table.m + 1,))
        y.copy_(t.unsqueeze(0).expand_as(y))
        f0 = new_field(shape)
        op.apply_into(t, f0)
        f = new_field(shape, (table.m + 1,))
        f.copy_(f0.unsqueeze(0).expand_as(f))
        return cls(table, y, f)

    @classmethod
    def empty(cls, op: HeatOperator, table: QuadratureTable) -> "NodeStates":
        lead = (table.m + 1,)
        return cls(table, new_field(op.grid.shape, lead), new_field(op.grid.shape, lead))

    def copy(self) -> "NodeStates":
        d = self.y.dim() - 1
        return NodeStates(self.table, clone_field(self.y, d), clone_field(self.f, d))

    def refresh(self, op: HeatOperator) -> None:
        for m in range(self.table.m + 1):
            op.apply_into(self.y[m], self.f[m])


class SubStepError(RuntimeError):
    """Multigrid failure inside a sweep (sdc.py:75-81)."""

    def __init__(self, substep: int, cause: MultigridError):
        super().__init__(f"sub-step {substep}: {cause}")
        self.substep = substep
        self.cause = cause


_descs: dict = {}


def sweep_desc(table: QuadratureTable, policy) -> capi.SweepDesc:
    key = (id(table), table.m, policy)
    d = _descs.get(key)
    if d is not None and d[0] is table:
        return d[1]
    m = table.m
    if m + 1 > capi.PL_MAX_NODES:
        raise ValueError(f"at most {capi.PL_MAX_NODES - 1} sub-steps on the GPU path")
    desc = capi.SweepDesc()
    desc.m = m
    q = table.q
    qd = q[1:] - q[:-1]                     # sdc.py:95, rounded like numpy
    for r in range(m):
        for c in range(m + 1):
            desc.qdelta[r * (m + 1) + c] = float(qd[r, c])
    for i, g in enumerate(table.nodes.gammas):
        desc.gammas[i] = float(g)
    if isinstance(policy, FixedCycles):
        desc.policy, desc.fixed_cycles = 0, policy.cycles
    elif isinstance(policy, Direct):
        desc.policy = 2
    else:
        desc.policy = 1
        desc.tol, desc.stall, desc.max_cycles = policy.tol, policy.stall, policy.max_cycles
    _descs[key] = (table, desc)
    return desc


# Receiver of per-solve records while a PFASST run logs them (pfasst_run's
# ``solve_log``): called with the list of records of one sweep.
_solve_sink = None


def sdc_sweep(states: NodeStates, y0, dt: float, op: HeatOperator, mg_cfg: MgConfig,
              policy: SolvePolicy, tau=None, solve_log: list | None = None) -> int:
    """One sweep through the sub-steps, in place; returns V-cycles used
    (sdc.py:84-114).

    ``solve_log`` (optional list) receives one ``[n, sigma, cycles, status]``
    record per sub-step solve -- the grid size, sigma = float(gamma_m) * dt and
    the ``SolveResult.cycles`` / ``.status`` the reference's ``multigrid.solve``
    returns for it (multigrid.py:261-288, called at sdc.py:105-113)."""
    _check_policy(policy)
    d = op.grid.dim
    ty0, _ = to_device(y0, d)
    ttau = to_device(tau, d)[0] if tau is not None else None
    desc = sweep_desc(states.table, policy)
    plan = plan_for(op, mg_cfg)
    if isinstance(policy, Direct):
        plan.ensure_direct()
    for gam in states.table.nodes.gammas:
        plan.ensure(float(gam) * dt)            # sdc.py:101 sigma of each sub-step
    g = op.grid
    nb = capi.lib().pl_sweep_workspace_bytes(g.dim, g.n, states.table.m)
    ws = scratch("sweep", nb)
    cyc, fsub, fres, fcyc = C.c_int(0), C.c_int(0), C.c_double(0), C.c_int(0)
    m = states.table.m
    sub_c, sub_s = (C.c_int * m)(), (C.c_int * m)()
    rc = capi.lib().pl_sdc_sweep(plan.handle.value, C.byref(desc), ptr(states.y),
                                 ptr(states.f), ptr(ty0), ptr(ttau), float(dt), ws.data_ptr(),
                                 ws.numel(), C.byref(cyc), sub_c, sub_s, C.byref(fsub),
                                 C.byref(fres), C.byref(fcyc), stream_ptr())
    if rc == capi.PL_ERR_MGCAP:
        cause = MultigridError(capi.last_error(), fres.value, fcyc.value)
        raise SubStepError(fsub.value, cause) from cause
    capi.check(rc, "sdc_sweep")
    if solve_log is not None or _solve_sink is not None:
        gam = states.table.nodes.gammas
        recs = [[g.n, float(gam[i]) * dt, int(sub_c[i]), capi.STATUS[sub_s[i]]]
                for i in range(m)]
        if solve_log is not None:
            solve_log.extend(recs)
        if _solve_sink is not None:
            _solve_sink(recs)
    return cyc.value


def residual_into(states: NodeStates, y0, dt: float, out, tau=None):
    """Device-side residual (asynchronous) into the 0-d/1-element tensor out."""
    m = states.table.m
    q = (C.c_double * ((m + 1) * (m + 1)))(*[float(v) for v in states.table.q.ravel()])
    d = states.y.dim() - 1
    n = states.y.shape[-1] + 1
    capi.check(capi.lib().pl_sdc_residual(ptr(states.y), ptr(states.f), ptr(y0), ptr(tau), q,
                                          m, float(dt), d, n, ptr(out), stream_ptr()),
               "residual")
    return out


def residual(states: NodeStates, y0, dt: float, tau=None) -> float:
    """Max over nodes of the max-norm of the collocation residual (sdc.py:117-124)."""
    d = states.y.dim() - 1
    ty0, _ = to_device(y0, d)
    ttau = to_device(tau, d)[0] if tau is not None else None
    out = zeros((1,))
    residual_into(states, ty0, dt, out, ttau)
    return float(out.item())


@dataclass
class RunResult:
    """sdc.py:127-133."""

    u: object
    iterations: list = field(default_factory=list)
    residuals: list = field(default_factory=list)
    vcycles: int = 0
    exhausted_steps: list = field(default_factory=list)


def run_sdc(op: HeatOperator, table: QuadratureTable, u0, t_end: float, n_steps: int,
            tol: float, max_iter: int, mg_cfg: MgConfig, policy: SolvePolicy,
            solve_log: list | None = None) -> RunResult:
    """Serial SDC / ISDC over n_steps steps (sdc.py:136-166); ``solve_log``
    as in sdc_sweep."""
    if n_steps < 1:
        raise ValueError("need at least one time step")
    dt = t_end / n_steps
    u, host = to_device(u0, op.grid.dim)
    result = RunResult(u=u0)
    for step in range(n_steps):
        states = NodeStates.spread(op, table, u)
        history = []
        sweeps = 0
        for _ in range(max_iter):
            result.vcycles += sdc_sweep(states, u, dt, op, mg_cfg, policy, solve_log=solve_log)
            sweeps += 1
            res = residual(states, u, dt)
            history.append(res)
            if res <= tol:
                break
        else:
            result.exhausted_steps.append(step)
        result.iterations.append(sweeps)
        result.residuals.append(history)
        u = clone_field(states.y[-1])
    result.u = u.contiguous().cpu().numpy() if host else u
    return result
