"""Full-size BASELINE config 3 pins from the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_cfg3_full.py

Runs ``pintlab.pfasst.pfasst_run`` on BASELINE config 3 at full size (3-D heat,
255^3 / 127^3 / 63^3, 9 / 5 / 3 uniform nodes, jor-rb omega = 1 V(1,1),
FixedCycles(1), 8 time ranks, dt = 1/64, tol 1e-10, seeded u0 of SURVEY.md
8(d)) with ``max_iter = 2`` (the full 20 iterations take hours on the CPU;
SURVEY.md 8(c) measured ~85 s per rank-iteration and 47 GB peak RSS).  Writes
``tests/golden/cfg3_full_it2.npz`` (a 16-strided sample of the final field and
its exact sum / max) and ``tests/golden/manifest_cfg3_full.json`` (counts, the
residual trace).  The GPU test ``test_cfg3_full_size_two_iterations`` runs the
same configuration on the B200 and compares.
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

    cfg = mg.MgConfig(smoother="jor-rb", omega=1.0, pre_sweeps=1, post_sweeps=1)
    levels = [hierarchy.Level(HeatOperator(Grid(3, n), 1.0, 2), quadrature.uniform_table(m - 1),
                              cfg, mg.FixedCycles(1), space_interp_order=4,
                              space_restrict="full-weighting")
              for n, m in ((256, 9), (128, 5), (64, 3))]
    u0 = seeded_field(3, 256)
    t0 = time.time()
    res = pfasst.pfasst_run(levels, u0, 8 / 64, 8, tol=1e-10, max_iter=2, executor="serial")
    wall = time.time() - t0
    u = res.u
    sample = np.ascontiguousarray(u[::16, ::16, ::16])
    meta = {"cases": {"cfg3_full_it2": {
        "grids": [255, 127, 63], "nodes": [9, 5, 3], "p": 8, "dt": 1 / 64, "tol": 1e-10,
        "max_iter": 2, "rank_iterations": res.rank_iterations,
        "rank_vcycles": res.rank_vcycles, "converged": res.converged,
        "trace": [[t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles]
                  for t in res.trace],
        "u_sum": math.fsum(u.ravel().tolist()), "u_absmax": float(np.max(np.abs(u))),
        "sample_stride": 16, "reference_wall_s": wall}}}
    np.savez_compressed(OUT / "cfg3_full_it2.npz", sample=sample)
    (OUT / "manifest_cfg3_full.json").write_text(json.dumps(meta, indent=1))
    print("wrote cfg3_full_it2 in", round(wall), "s")


if __name__ == "__main__":
    main()
