"""Golden vectors for the lexicographic Gauss-Seidel smoother and the Direct
policy, produced by the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden_gs_direct.py

Imports ``pintlab`` read-only from ``/root/reference/pkg/src`` and writes
``tests/golden/gsd_*.npz`` plus ``tests/golden/manifest_gsd.json``.  Kept apart
from make_golden.py so the earlier fixtures are not regenerated.
"""

from __future__ import annotations

import json
import platform
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def main():
    sys.path.insert(0, REF)
    sys.dont_write_bytecode = True
    import pintlab.multigrid as mg
    from pintlab import heat, hierarchy, pfasst, quadrature, sdc
    from pintlab.heat import Grid, HeatOperator

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.pintlab_oracle import seeded_field

    manifest = {"env": {"numpy": np.__version__, "python": platform.python_version(),
                        "reference": REF}, "cases": {}}
    # per-solve log: multigrid.solve is looked up as a module attribute at
    # sdc.py:107, so wrapping it records every sub-step solve in call order
    log = []
    real_solve = mg.solve

    def logged_solve(op, u0, b, cfg, policy):
        res = real_solve(op, u0, b, cfg, policy)
        log.append([op.grid.n, op.sigma, res.cycles, res.status])
        return res
    rng = np.random.default_rng(1407_0001)

    # ---- kernels: GS sweeps, GS V-cycles, Direct solves (multigrid.py:211-288)
    sizes = {(1, 2): 64, (1, 4): 64, (2, 2): 64, (2, 4): 32, (3, 2): 32, (3, 4): 16}
    for (d, o), n in sizes.items():
        for L, nu in ((1.0, 1.0), (1.5, 0.7)):
            op = HeatOperator(Grid(d, n, L), nu, o)
            u = rng.standard_normal(op.grid.shape)
            b = rng.standard_normal(op.grid.shape)
            sigma = 0.0131 if d < 3 else 0.0021
            sop = mg.ShiftedOperator(op, sigma)
            cfg = mg.MgConfig(smoother="gauss-seidel")
            cfg11 = mg.MgConfig(smoother="gauss-seidel", pre_sweeps=1, post_sweeps=1)
            arr = {"u": u, "b": b,
                   "gs1": mg.smooth(sop, u, b, cfg, 1), "gs2": mg.smooth(sop, u, b, cfg, 2),
                   "vc22": mg.v_cycle(sop, u, b, cfg),
                   "vc11z": mg.v_cycle(sop, np.zeros_like(b), b, cfg11),
                   "direct": mg.solve(sop, u, b, cfg, mg.Direct()).u}
            tol = mg.solve(sop, u, b, cfg, mg.ToTolerance(1e-10))
            arr["tol_u"] = tol.u
            name = f"gsd_k_d{d}_o{o}_L{L:g}"
            manifest["cases"][name] = {"dim": d, "n": n, "order": o, "length": L, "nu": nu,
                                       "sigma": sigma, "tol_cycles": tol.cycles,
                                       "tol_status": tol.status}
            np.savez_compressed(OUT / f"{name}.npz", **arr)

    # ---- serial ISDC with GS + ToTolerance and with Direct (sdc.py:136-166)
    op = HeatOperator(Grid(1, 64), 1.0, 2)
    u0 = heat.initial_condition(op.grid, 1)
    sdc.multigrid.solve = logged_solve
    log.clear()
    r1 = sdc.run_sdc(op, quadrature.uniform_table(4), u0, 0.25, 4, 1e-10, 20,
                     mg.MgConfig(smoother="gauss-seidel"), mg.ToTolerance(1e-12))
    solves_gs = [list(x) for x in log]
    op2 = HeatOperator(Grid(2, 16), 1.0, 4)
    u02 = seeded_field(2, 16)
    log.clear()
    r2 = sdc.run_sdc(op2, quadrature.uniform_table(4), u02, 0.125, 2, 1e-11, 30,
                     mg.MgConfig(smoother="gauss-seidel"), mg.Direct())
    solves_direct = [list(x) for x in log]
    manifest["cases"]["gsd_sdc"] = {
        "gs": {"iterations": r1.iterations, "residuals": r1.residuals, "vcycles": r1.vcycles,
               "solves": solves_gs},
        "direct": {"iterations": r2.iterations, "residuals": r2.residuals,
                   "vcycles": r2.vcycles, "solves": solves_direct}}
    np.savez_compressed(OUT / "gsd_sdc.npz", u0=u0, gs_u=r1.u, u02=u02, direct_u=r2.u)

    # ---- PFASST with the GS smoother (the reference's config default) and
    # with Direct solves on every level (pfasst.py:256-287)
    runs = {
        "gs2d": dict(d=2, ns=(32, 16), nodes=(5, 3), pol=mg.FixedCycles(1), p=3, dt=1 / 64,
                     tol=1e-10),
        "direct1d": dict(d=1, ns=(64, 32), nodes=(5, 3), pol=mg.Direct(), p=4, dt=1 / 32,
                         tol=1e-11),
    }
    for name, r in runs.items():
        levels = [hierarchy.Level(HeatOperator(Grid(r["d"], n), 1.0, 2),
                                  quadrature.uniform_table(m - 1),
                                  mg.MgConfig(smoother="gauss-seidel"), r["pol"],
                                  space_interp_order=4)
                  for n, m in zip(r["ns"], r["nodes"])]
        u0 = seeded_field(r["d"], r["ns"][0])
        log.clear()
        res = pfasst.pfasst_run(levels, u0, r["dt"] * r["p"], r["p"], tol=r["tol"],
                                max_iter=20, executor="serial")
        meta = {k: (list(v) if isinstance(v, tuple) else v) for k, v in r.items()
                if k != "pol"}
        meta["policy"] = "direct" if isinstance(r["pol"], mg.Direct) else ["fixed", 1]
        meta.update(rank_iterations=res.rank_iterations, rank_vcycles=res.rank_vcycles,
                    converged=res.converged,
                    trace=[[t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles]
                           for t in res.trace],
                    solves=[list(x) for x in log])
        manifest["cases"][f"gsd_run_{name}"] = meta
        np.savez_compressed(OUT / f"gsd_run_{name}.npz", u0=u0, u=res.u)

    sdc.multigrid.solve = real_solve
    (OUT / "manifest_gsd.json").write_text(json.dumps(manifest, indent=1))
    print("wrote", len(manifest["cases"]), "cases")


if __name__ == "__main__":
    main()
