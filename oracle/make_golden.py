"""Generate golden vectors by running the REAL reference (build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

Imports ``pintlab`` read-only from ``/root/reference/pkg/src`` (never copied),
runs it on seeded inputs and writes ``tests/golden/<case>.npz`` plus
``tests/golden/manifest.json`` (scalars, counts, traces, environment).  The
fixtures pin both the oracle (``oracle/pintlab_oracle.py``, bit-for-bit, CPU
tests) and the CUDA path (tolerance + identical counts, ``-m gpu`` tests).
``/root/reference`` does not exist on the GPU box; only the committed fixtures
travel.
"""

from __future__ import annotations

import json
import os
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
    from pintlab import heat, hierarchy, pfasst, quadrature, sdc, transfers
    from pintlab.heat import Grid, HeatOperator

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from oracle.pintlab_oracle import seeded_field

    OUT.mkdir(parents=True, exist_ok=True)
    manifest = {"env": {"numpy": np.__version__,
                        "python": platform.python_version(),
                        "machine": platform.processor() or platform.machine(),
                        "reference": REF}, "cases": {}}
    arrays = {}

    def put(case, meta=None, **arr):
        arrays[case] = arr
        manifest["cases"][case] = meta or {}

    # solve log: multigrid.solve is looked up as a module attribute (sdc.py:107)
    log = []
    real_solve = mg.solve

    def logged_solve(op, u0, b, cfg, policy):
        res = real_solve(op, u0, b, cfg, policy)
        log.append([op.grid.n, op.sigma, res.cycles, res.status])
        return res

    sdc.multigrid.solve = logged_solve

    rng = np.random.default_rng(20140724)
    sizes = {1: 64, 2: 32, 3: 16}

    # ---- L1: stencil, diagonal, shifted operator (heat.py:111-158)
    for d, n in sizes.items():
        for order in (2, 4):
            for nu in (1.0, 0.7):
                op = HeatOperator(Grid(d, n), nu, order)
                u = rng.standard_normal(op.grid.shape)
                sig = 0.013
                sop = mg.ShiftedOperator(op, sig)
                put(f"apply_d{d}_o{order}_nu{nu}", {"dim": d, "n": n, "order": order,
                                                   "nu": nu, "sigma": sig},
                    u=u, f=op.apply(u), diag=op.diagonal(), au=sop.apply(u),
                    sdiag=sop.diagonal())
    # non-unit domain length (dx2 not a power of two)
    op = HeatOperator(Grid(2, 16, 3.0), 1.0, 2)
    u = rng.standard_normal(op.grid.shape)
    put("apply_d2_o2_L3", {"dim": 2, "n": 16, "order": 2, "nu": 1.0, "length": 3.0},
        u=u, f=op.apply(u), diag=op.diagonal())

    # ---- transfers (transfers.py)
    for d, n in sizes.items():
        u = rng.standard_normal((n - 1,) * d)
        c = rng.standard_normal((n // 2 - 1,) * d)
        put(f"transfer_d{d}", {"dim": d, "n": n}, u=u, fw=transfers.full_weighting(u),
            inj=transfers.inject(u), c=c, lin=transfers.interp_linear(c),
            cub=transfers.interp_cubic(c))
    for nf in (4, 8, 16):   # cubic windows with nc < 3 and boundary rows
        c = rng.standard_normal((nf // 2 - 1,))
        put(f"cubic_1d_nf{nf}", {"nf": nf}, c=c, cub=transfers.interp_cubic(c),
            mat=transfers._cubic_matrix(nf))

    # ---- smoothers and V-cycles (multigrid.py:211-251)
    for d, n in sizes.items():
        for order in (2, 4):
            for sm, om in (("jacobi", 2.0 / 3.0), ("jor-rb", 1.0), ("jor-rb", 0.8)):
                cfg = mg.MgConfig(smoother=sm, omega=om, pre_sweeps=2, post_sweeps=1)
                op = mg.ShiftedOperator(HeatOperator(Grid(d, n), 1.0, order), 0.02)
                u = rng.standard_normal(op.grid.shape)
                b = rng.standard_normal(op.grid.shape)
                put(f"mg_d{d}_o{order}_{sm}_{om:.3f}",
                    {"dim": d, "n": n, "order": order, "smoother": sm, "omega": om,
                     "pre": 2, "post": 1, "sigma": 0.02},
                    u=u, b=b, sm2=mg.smooth(op, u, b, cfg, 2),
                    vc=mg.v_cycle(op, u, b, cfg),
                    vc0=mg.v_cycle(op, np.zeros_like(b), b, cfg))
    # coarsest grid alone (n <= coarsest_n)
    for d in (1, 2, 3):
        op = mg.ShiftedOperator(HeatOperator(Grid(d, 4), 1.0, 2), 0.3)
        b = rng.standard_normal(op.grid.shape)
        put(f"coarsest_d{d}", {"dim": d, "n": 4, "sigma": 0.3}, b=b,
            u=mg.v_cycle(op, np.zeros_like(b), b, mg.MgConfig()))

    # ---- solve policies (multigrid.py:261-288)
    for d, n in sizes.items():
        op = mg.ShiftedOperator(HeatOperator(Grid(d, n), 1.0, 2), 0.05)
        b = rng.standard_normal(op.grid.shape)
        u0 = rng.standard_normal(op.grid.shape)
        r2 = mg.solve(op, u0, b, mg.MgConfig(), mg.FixedCycles(2))
        rt = mg.solve(op, u0, b, mg.MgConfig(), mg.ToTolerance(1e-12))
        rs = mg.solve(op, np.zeros_like(b), b, mg.MgConfig(pre_sweeps=0, post_sweeps=0),
                      mg.ToTolerance(1e-14))
        try:
            mg.solve(op, np.zeros_like(b), b, mg.MgConfig(),
                     mg.ToTolerance(1e-14, stall=1.0 - 1e-12, max_cycles=3))
            cap = None
        except mg.MultigridError as exc:
            cap = {"cycles": exc.cycles, "residual": exc.residual}
        put(f"solve_d{d}", {"dim": d, "n": n, "sigma": 0.05,
                            "tol_cycles": rt.cycles, "tol_status": rt.status,
                            "stall_cycles": rs.cycles, "stall_status": rs.status,
                            "cap": cap},
            b=b, u0=u0, fixed2=r2.u, tol=rt.u, stall=rs.u)

    # ---- SDC sweep + residual (sdc.py:84-124)
    for d, n in sizes.items():
        for M in (2, 4, 8):
            for with_tau in (False, True):
                op = HeatOperator(Grid(d, n), 1.0, 2)
                table = quadrature.uniform_table(M)
                y = rng.standard_normal((M + 1,) + op.grid.shape)
                st = sdc.NodeStates(table, y.copy(), np.stack([op.apply(v) for v in y]))
                y0 = rng.standard_normal(op.grid.shape)
                tau = 1e-3 * rng.standard_normal(y.shape) if with_tau else None
                dt = 0.05
                pol = mg.FixedCycles(1) if d > 1 else mg.ToTolerance(1e-12)
                cfg = mg.MgConfig()
                log.clear()
                cyc = sdc.sdc_sweep(st, y0, dt, op, cfg, pol, tau=tau)
                res = sdc.residual(st, y0, dt, tau=tau)
                extra = {"tau": tau} if with_tau else {}
                put(f"sweep_d{d}_M{M}_tau{int(with_tau)}",
                    {"dim": d, "n": n, "M": M, "dt": dt, "cycles": cyc, "residual": res,
                     "policy": "fixed1" if d > 1 else "tol1e-12",
                     "solves": [list(x) for x in log]},
                    y=y, y0=y0, y_out=st.y, f_out=st.f, **extra)

    # ---- FAS machinery (hierarchy.py:85-122), 3 levels incl. a same-n level
    for d, ns in ((1, (64, 32, 32)), (2, (32, 16, 8)), (3, (16, 8, 4))):
        for interp in (2, 4):
            levels = []
            for n, M in zip(ns, (4, 2, 1)):
                levels.append(hierarchy.Level(HeatOperator(Grid(d, n), 1.0, 2),
                                              quadrature.uniform_table(M),
                                              mg.MgConfig(), mg.FixedCycles(1),
                                              space_interp_order=interp))
            f, c = levels[0], levels[1]
            y = rng.standard_normal((5,) + f.grid.shape)
            fst = sdc.NodeStates(f.table, y.copy(), np.stack([f.operator.apply(v) for v in y]))
            ftau = 1e-3 * rng.standard_normal(y.shape)
            rs = hierarchy.restrict_state(fst, f, c)
            tau = hierarchy.compute_fas(fst, rs, f, c, 0.05, fine_tau=ftau)
            tau0 = hierarchy.compute_fas(fst, rs, f, c, 0.05)
            newc = rs.copy()
            newc.y = newc.y + 1e-2 * rng.standard_normal(newc.y.shape)
            cc = fst.copy()
            hierarchy.coarse_correction(cc, rs, newc, f, c)
            # full 3-level MLSDC iteration
            u0 = rng.standard_normal(f.grid.shape)
            log.clear()
            ts, cyc0 = hierarchy.initialize_step(levels, u0, 0.05)
            cyc = hierarchy.mlsdc_iteration(ts, 0.05)
            res = ts.fine_residual(0.05)
            put(f"fas_d{d}_i{interp}",
                {"dim": d, "ns": list(ns), "interp": interp, "dt": 0.05,
                 "init_cycles": cyc0, "it_cycles": cyc, "residual": res},
                y=y, ftau=ftau, ry=rs.y, rf=rs.f, tau=tau, tau0=tau0, newc=newc.y,
                cc_y=cc.y, cc_f=cc.f, u0=u0, ml_y0=ts.states[0].y, ml_y1=ts.states[1].y,
                ml_y2=ts.states[2].y, ml_tau1=ts.tau[1], ml_tau2=ts.tau[2])

    # ---- end-to-end PFASST runs (pfasst.py:256-287)
    def levels_for(d, ns, nodes, sm, om, pre, post, pol, interp=4, orders=None):
        orders = orders or [2] * len(ns)
        return [hierarchy.Level(HeatOperator(Grid(d, n), 1.0, o),
                                quadrature.uniform_table(m - 1),
                                mg.MgConfig(smoother=sm, omega=om, pre_sweeps=pre,
                                            post_sweeps=post),
                                pol, space_interp_order=interp)
                for n, m, o in zip(ns, nodes, orders)]

    runs = {
        # BASELINE configs 0 and 1 at full size (1-D, 255 points)
        "cfg0": dict(d=1, ns=(256, 128), nodes=(5, 3), sm="jacobi", om=2 / 3, pre=2,
                     post=2, pol=mg.ToTolerance(1e-12), p=4, blocks=1, dt=1 / 32,
                     tol=1e-10, u0="sine"),
        "cfg0_interp2": dict(d=1, ns=(256, 128), nodes=(5, 3), sm="jacobi", om=2 / 3,
                             pre=2, post=2, pol=mg.ToTolerance(1e-12), p=4, blocks=1,
                             dt=1 / 32, tol=1e-10, u0="sine", interp=2),
        "cfg1": dict(d=1, ns=(256, 128), nodes=(5, 3), sm="jacobi", om=2 / 3, pre=2,
                     post=2, pol=mg.FixedCycles(1), p=4, blocks=1, dt=1 / 32,
                     tol=1e-10, u0="sine"),
        "cfg1_fc2": dict(d=1, ns=(256, 128), nodes=(5, 3), sm="jacobi", om=2 / 3, pre=2,
                         post=2, pol=mg.FixedCycles(2), p=4, blocks=1, dt=1 / 32,
                         tol=1e-10, u0="sine"),
        # reduced stand-ins with the structure of configs 2-4
        "cfg2_small": dict(d=2, ns=(64, 32), nodes=(5, 3), sm="jacobi", om=2 / 3, pre=2,
                           post=2, pol=mg.FixedCycles(1), p=8, blocks=1, dt=1 / 64,
                           tol=1e-10, u0="seeded"),
        "cfg2_small_fc2": dict(d=2, ns=(64, 32), nodes=(5, 3), sm="jacobi", om=2 / 3,
                               pre=2, post=2, pol=mg.FixedCycles(2), p=8, blocks=1,
                               dt=1 / 64, tol=1e-10, u0="seeded"),
        "cfg3_small": dict(d=3, ns=(32, 16, 8), nodes=(9, 5, 3), sm="jor-rb", om=1.0,
                           pre=1, post=1, pol=mg.FixedCycles(1), p=8, blocks=1,
                           dt=1 / 64, tol=1e-10, u0="seeded"),
        "cfg4_small": dict(d=3, ns=(32, 16), nodes=(5, 3), sm="jacobi", om=2 / 3, pre=2,
                           post=2, pol=mg.FixedCycles(1), p=4, blocks=2, dt=1 / 64,
                           tol=1e-9, u0="seeded"),
        "cfg4_small_tol": dict(d=3, ns=(16, 8), nodes=(5, 3), sm="jacobi", om=2 / 3,
                               pre=2, post=2, pol=mg.ToTolerance(1e-12), p=4, blocks=2,
                               dt=1 / 64, tol=1e-9, u0="seeded"),
        "order4_small": dict(d=2, ns=(32, 16), nodes=(5, 3), sm="jor-rb", om=1.0, pre=1,
                             post=1, pol=mg.FixedCycles(2), p=3, blocks=1, dt=1 / 64,
                             tol=1e-10, u0="seeded", orders=[4, 2]),
        "same_n_3lvl": dict(d=1, ns=(64, 64, 32), nodes=(5, 3, 2), sm="jacobi",
                            om=2 / 3, pre=2, post=2, pol=mg.FixedCycles(1), p=3,
                            blocks=2, dt=1 / 64, tol=1e-10, u0="sine", interp=2),
    }
    for name, r in runs.items():
        levels = levels_for(r["d"], r["ns"], r["nodes"], r["sm"], r["om"], r["pre"],
                            r["post"], r["pol"], r.get("interp", 4), r.get("orders"))
        n0 = r["ns"][0]
        if r["u0"] == "sine":
            u0 = heat.initial_condition(Grid(r["d"], n0), 1)
        else:
            u0 = seeded_field(r["d"], n0)
        t_end = r["dt"] * r["p"] * r["blocks"]
        log.clear()
        res = pfasst.pfasst_run(levels, u0, t_end, r["p"], blocks=r["blocks"],
                                tol=r["tol"], max_iter=20, executor="serial",
                                record_final_values=True)
        pol = r["pol"]
        meta = {k: (v if not isinstance(v, tuple) else list(v)) for k, v in r.items()
                if k != "pol"}
        meta["policy"] = (["fixed", pol.cycles] if isinstance(pol, mg.FixedCycles)
                          else ["tol", pol.tol, pol.stall, pol.max_cycles])
        meta.update(rank_iterations=res.rank_iterations, rank_vcycles=res.rank_vcycles,
                    converged=res.converged,
                    trace=[[t.block, t.rank, t.iteration, t.level, t.residual, t.vcycles]
                           for t in res.trace],
                    solves=[list(x) for x in log],
                    err_pde=float(np.max(np.abs(res.u - heat.exact_pde(
                        Grid(r["d"], n0), 1, 1.0, t_end)))))
        finals = res.final_values[-1]
        keep = finals if r["d"] == 1 else finals[-2:]      # bound fixture size
        meta["finals_kept_from"] = len(finals) - len(keep)
        put(f"run_{name}", meta, u0=u0, u=res.u,
            finals=np.stack(keep) if keep else np.zeros((0,) + u0.shape))

    # serial MLSDC / ISDC drivers and P=1 equivalence (hierarchy.py:262, sdc.py:136)
    levels = levels_for(1, (64, 32), (3, 2), "jacobi", 2 / 3, 2, 2, mg.FixedCycles(1))
    u0 = heat.initial_condition(Grid(1, 64), 1)
    ml = hierarchy.run_mlsdc(levels, u0, 0.25, 4, 1e-10, 20)
    p1 = pfasst.pfasst_run(levels, u0, 0.25 / 4, 1, tol=1e-10, max_iter=20)
    isdc = sdc.run_sdc(levels[0].operator, levels[0].table, u0, 0.25, 4, 1e-10, 20,
                       levels[0].mg_cfg, levels[0].policy)
    put("serial_drivers", {"ml_iterations": ml.iterations, "ml_residuals": ml.residuals,
                           "ml_vcycles": ml.vcycles, "sdc_iterations": isdc.iterations,
                           "sdc_residuals": isdc.residuals, "sdc_vcycles": isdc.vcycles,
                           "p1_iterations": p1.rank_iterations},
        u0=u0, ml_u=ml.u, sdc_u=isdc.u, p1_u=p1.u)

    # ---- 3-D n = 32 cases (exercise the z-marching / fused-sweep kernels,
    # which engage from 31^3 up); appended last so earlier draws are unchanged
    rng2 = np.random.default_rng(4242)
    op32 = HeatOperator(Grid(3, 32), 1.0, 2)
    u = rng2.standard_normal(op32.grid.shape)
    b = rng2.standard_normal(op32.grid.shape)
    sop = mg.ShiftedOperator(op32, 1.0 / 256)
    meta = {"dim": 3, "n": 32, "sigma": 1.0 / 256}
    arr = {"u": u, "b": b, "f": op32.apply(u), "r": b - sop.apply(u)}
    for sm, om in (("jacobi", 2.0 / 3.0), ("jor-rb", 1.0), ("jor-rb", 0.8)):
        cfg = mg.MgConfig(smoother=sm, omega=om, pre_sweeps=2, post_sweeps=2)
        tag = f"{sm}_{om:.3f}"
        for cnt in (1, 2, 3):
            arr[f"sm{cnt}_{tag}"] = mg.smooth(sop, u, b, cfg, cnt)
        arr[f"vc22_{tag}"] = mg.v_cycle(sop, u, b, cfg)
        arr[f"vc22z_{tag}"] = mg.v_cycle(sop, np.zeros_like(b), b, cfg)
        cfg11 = mg.MgConfig(smoother=sm, omega=om, pre_sweeps=1, post_sweeps=1)
        arr[f"vc11_{tag}"] = mg.v_cycle(sop, u, b, cfg11)
    put("mg32_d3", meta, **arr)

    for case, arr in arrays.items():
        np.savez_compressed(OUT / f"{case}.npz", **arr)
    with open(OUT / "manifest.json", "w") as fh:
        json.dump(manifest, fh, indent=1, default=float)
    total = sum(os.path.getsize(OUT / f"{c}.npz") for c in arrays)
    print(f"wrote {len(arrays)} cases, {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
