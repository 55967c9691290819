"""Full-size BASELINE config 2 pins from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_cfg2_full.py

BASELINE config 2 at full size: 2-D heat nu = 1 on the unit square,
1023^2 / 511^2 interior points, 5 / 3 uniform nodes, Jacobi omega = 2/3
V(2,2), 8 time ranks, dt = 1/64, seeded u0 of SURVEY.md 8(d), full
``max_iter = 20`` PFASST runs with FixedCycles(1) and FixedCycles(2) per
sub-step at tol 1e-10 (95-332 s each on the CPU).  Writes
``tests/golden/cfg2_full.npz`` (8-strided samples of the final fields) and
``tests/golden/manifest_cfg2_full.json`` (counts, flags, residual traces,
exact sums and maxima).
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


def main():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import pintlab.multigrid as mg
    from pintlab import hierarchy, pfasst, quadrature
    from pintlab.heat import Grid, HeatOperator

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.pintlab_oracle import seeded_field

    cfg = mg.MgConfig(smoother="jacobi", omega=2.0 / 3.0, pre_sweeps=2, post_sweeps=2)
    u0 = seeded_field(2, 1024)
    meta, arrays = {"cases": {}}, {}
    for cycles in (1, 2):
        levels = [hierarchy.Level(HeatOperator(Grid(2, n), 1.0, 2),
                                  quadrature.uniform_table(m - 1), cfg,
                                  mg.FixedCycles(cycles), space_interp_order=4,
                                  space_restrict="full-weighting")
                  for n, m in ((1024, 5), (512, 3))]
        t0 = time.time()
        res = pfasst.pfasst_run(levels, u0, 8 / 64, 8, tol=1e-10, max_iter=20,
                                executor="threaded")
        wall = time.time() - t0
        u = res.u
        name = f"cfg2_full_fc{cycles}"
        arrays[f"{name}_sample"] = np.ascontiguousarray(u[::8, ::8])
        meta["cases"][name] = {
            "grids": [1023, 511], "nodes": [5, 3], "p": 8, "dt": 1 / 64, "tol": 1e-10,
            "max_iter": 20, "cycles": cycles, "rank_iterations": res.rank_iterations,
            "rank_vcycles": res.rank_vcycles, "converged": res.converged,
            "trace": [[t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles]
                      for t in res.trace],
            "u_sum": math.fsum(u.ravel().tolist()), "u_absmax": float(np.max(np.abs(u))),
            "sample_stride": 8, "reference_wall_s": wall}
        print(name, res.rank_iterations, round(wall), "s", flush=True)
    np.savez_compressed(OUT / "cfg2_full.npz", **arrays)
    (OUT / "manifest_cfg2_full.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
