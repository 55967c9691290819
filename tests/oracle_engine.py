"""A CPU engine for the PFASST schedule built on the oracle (TEST ONLY).

``paper_1407_6486_b200.pfasst.pfasst_run`` drives time ranks through an
engine interface (DeviceEngine on the GPU).  This engine implements the same
interface with the numpy oracle so the multi-process exchange logic of the
"nccl" executor can be exercised with gloo on CPU, and its results compared
bit for bit with the oracle's serial schedule.
"""
import numpy as np
import torch

from oracle import pintlab_oracle as O


def oracle_levels(levels):
    """Product Level objects -> oracle levels (same parameters)."""
    out = []
    for lv in levels:
        g = lv.operator.grid
        pol = lv.policy
        opol = O.Fixed(pol.cycles) if hasattr(pol, "cycles") else O.ToTol(pol.tol, pol.stall,
                                                                         pol.max_cycles)
        cfg = lv.mg_cfg
        out.append(O.Lvl(O.Op(g.dim, g.n, lv.operator.nu, lv.operator.order, g.length),
                         O.make_table(tuple(lv.table.nodes.nodes)),
                         O.Mg(cfg.smoother, cfg.omega, cfg.pre_sweeps, cfg.post_sweeps,
                              cfg.coarsest_n),
                         opol, lv.space_interp_order, lv.space_restrict))
    return out


class OracleEngine:
    def __init__(self, levels, dt, ranks):
        self.levels = oracle_levels(levels)
        self.dt = dt
        self.L = len(levels)
        self.ranks = list(ranks)
        self.ts = {}
        self.copies = {}

    def spread(self, n, u):
        u = u.numpy() if isinstance(u, torch.Tensor) else np.asarray(u)
        ts = O.Step.spread(self.levels, u)
        self.ts[n] = ts
        self.copies[n] = [s.copy() for s in ts.states]

    def coarse_payload(self, n):
        return torch.from_numpy(self.ts[n].states[self.L - 1].y[-1])

    def fine_payload(self, n):
        return torch.from_numpy(self.ts[n].states[0].y[-1])

    def set_coarse_y0(self, n, t):
        self.ts[n].y0[self.L - 1] = t.numpy().copy()

    def set_fine_y0(self, n, t):
        ts = self.ts[n]
        v = t.numpy().copy()
        ts.y0[0] = v
        ts.states[0].y[0] = v
        ts.states[0].f[0] = O.heat_apply(self.levels[0].op, v)

    def burn_in(self, n):
        return O.burn_in(self.ts[n], self.dt, 1)

    def interpolate_up(self, n, exact):
        ts = self.ts[n]
        O.interpolate_up(ts, self.copies[n], exact_y0=ts.y0[0] if exact else None)

    def iteration(self, n, pre_coarse):
        return O.mlsdc_iteration(self.ts[n], self.dt, pre_coarse=pre_coarse)

    def residual(self, n):
        ts = self.ts[n]
        return O.residual(ts.states[0], ts.y0[0], self.dt)

    def read(self, n, handle):
        return handle

    def snapshot(self, t):
        return t.clone()

    def to_wire(self, t):
        return t.contiguous().clone()

    def wire_buffer(self, like):
        return torch.empty_like(like.contiguous())

    def from_wire(self, buf, like):
        return buf.reshape(like.shape)
