"""Full-size BASELINE config 4 kernel pins from the REAL reference (build
container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_cfg4_kernels.py

A whole config-4 PFASST run at 511^3 is infeasible on the CPU (SURVEY.md 8(c):
~40 s per V-cycle, ~200 GB of state).  Its hot kernels are pinned at full size
instead, on the reference's own code: one Jacobi V(2,2) cycle of
(I - sigma A) u = b at 511^3 (sigma = dt / 4 = 1/256, the sub-step shift of
5 uniform nodes at dt = 1/64) from seeded normal u, b; and one SDC sweep
(4 sub-steps, FixedCycles(1)) of the seeded u0 of SURVEY.md 8(d) at 511^3 with
dt = 1/64.  Writes ``tests/golden/cfg4_kernels.npz`` (32-strided samples) and
``tests/golden/manifest_cfg4_kernels.json`` (exact sums and maxima, cycles).
"""

from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def summary(x):
    return {"sum": math.fsum(x.ravel().tolist()), "absmax": float(np.max(np.abs(x)))}


def main():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import pintlab.multigrid as mg
    from pintlab import quadrature, sdc
    from pintlab.heat import Grid, HeatOperator

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.pintlab_oracle import seeded_field

    op = HeatOperator(Grid(3, 512), 1.0, 2)
    cfg = mg.MgConfig(smoother="jacobi", omega=2.0 / 3.0, pre_sweeps=2, post_sweeps=2)
    rng = np.random.default_rng(511)
    u = rng.standard_normal(op.grid.shape)
    b = rng.standard_normal(op.grid.shape)
    t0 = time.time()
    v = mg.v_cycle(mg.ShiftedOperator(op, 1.0 / 256), u, b, cfg)
    t_v = time.time() - t0
    del u, b
    meta = {"vcycle": {**summary(v), "sigma": 1.0 / 256, "seed": 511, "wall_s": t_v}}
    arrays = {"vcycle_sample": np.ascontiguousarray(v[::32, ::32, ::32])}
    del v
    u0 = seeded_field(3, 512)
    table = quadrature.uniform_table(4)
    states = sdc.NodeStates.spread(op, table, u0)
    t0 = time.time()
    cycles = sdc.sdc_sweep(states, u0, 1 / 64, op, cfg, mg.FixedCycles(1))
    t_s = time.time() - t0
    meta["sweep"] = {"cycles": cycles, "dt": 1 / 64, "wall_s": t_s,
                     "y_last": summary(states.y[-1]), "f_last": summary(states.f[-1]),
                     "res": float(sdc.residual(states, u0, 1 / 64))}
    arrays["sweep_y_last_sample"] = np.ascontiguousarray(states.y[-1][::32, ::32, ::32])
    arrays["sweep_y_mid_sample"] = np.ascontiguousarray(states.y[2][::32, ::32, ::32])
    np.savez_compressed(OUT / "cfg4_kernels.npz", **arrays)
    (OUT / "manifest_cfg4_kernels.json").write_text(
        json.dumps({"cases": {"cfg4_kernels": meta}}, indent=1))
    print("v-cycle", round(t_v), "s; sweep", round(t_s), "s", flush=True)


if __name__ == "__main__":
    main()
