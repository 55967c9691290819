"""Per-kernel micro-benchmark on one grid (CUDA events, warm, median of reps).

    python tools/kernel_bench.py [--dim 3] [--n 256] [--reps 20] [--only jacobi,...]

Prints one JSON object: per kernel the median ms, the algorithmic bytes of
SURVEY.md 8(d) and the implied GB/s.  Used for the ncu captures under
profiles/ (run it under `ncu -k regex:...`)."""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_6486_b200 import _capi, transfers  # noqa: E402
from paper_1407_6486_b200._device import new_field, to_device  # noqa: E402
from paper_1407_6486_b200.heat import Grid, HeatOperator  # noqa: E402
from paper_1407_6486_b200.multigrid import MgConfig, ShiftedOperator, plan_for, vcycles_into  # noqa: E402
from paper_1407_6486_b200.quadrature import uniform_table  # noqa: E402
from paper_1407_6486_b200.sdc import NodeStates, residual_into, sdc_sweep  # noqa: E402
from paper_1407_6486_b200.multigrid import FixedCycles  # noqa: E402


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--opts", default="", help="pl_set_option pairs KEY=VAL,...")
    args = ap.parse_args()
    for kv in filter(None, args.opts.split(",")):
        k, v = kv.split("=")
        _capi.set_option(int(k), int(v))
    g = Grid(args.dim, args.n)
    N = g.dof
    rng = np.random.default_rng(0)
    u = to_device(rng.standard_normal(g.shape))[0]
    b = to_device(rng.standard_normal(g.shape))[0]
    out = new_field(g.shape)
    op = HeatOperator(g)
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    sig = 1.0 / 512
    res = {}
    only = set(args.only.split(",")) if args.only else None

    def run(name, fn, alg):
        if only and name not in only:
            return
        ms = timeit(fn, args.reps)
        res[name] = {"ms": ms, "alg_bytes": alg, "alg_gbs": alg / (ms / 1e3) / 1e9}

    run("apply", lambda: op.apply_into(u, out), 16.0 * N)
    for sm, om in (("jacobi", 2 / 3), ("jor-rb", 1.0)):
        cfg = MgConfig(sm, om, 1, 1)
        p = plan_for(op, cfg)
        p.ensure(sig)
        run(f"smooth1_{sm}", lambda p=p: lib.pl_mg_smooth(p.handle.value, u.data_ptr(),
                                                          b.data_ptr(), sig, 1, s), 24.0 * N)
        sop = ShiftedOperator(op, sig)
        run(f"vcycle_{sm}_V11", lambda sop=sop, cfg=cfg: vcycles_into(sop, u, b, cfg, 1),
            (24.0 * 2 + 32 + 16 / 2 ** args.dim) / (1 - 2.0 ** -args.dim) * N)
    cfg = MgConfig("jacobi", 2 / 3, 2, 2)
    sop = ShiftedOperator(op, sig)
    run("vcycle_jacobi_V22", lambda: vcycles_into(sop, u, b, cfg, 1),
        (24.0 * 4 + 32 + 16 / 2 ** args.dim) / (1 - 2.0 ** -args.dim) * N)
    run("residual", lambda: lib.pl_shifted_apply(u.data_ptr(), out.data_ptr(), g.dim, g.n,
                                                 1.0, 1.0, 2, sig, s), 16.0 * N)
    c = new_field((g.n // 2 - 1,) * g.dim)
    run("full_weighting", lambda: lib.pl_full_weighting(u.data_ptr(), c.data_ptr(), g.dim,
                                                        g.n, s), 8.0 * N * (1 + 2.0 ** -g.dim))
    run("prolong_add", lambda: lib.pl_interp_linear(c.data_ptr(), u.data_ptr(), g.dim, g.n, 1,
                                                    s), 8.0 * N * (2 + 2.0 ** -g.dim))
    run("interp_cubic_add", lambda: transfers.interp_cubic_into(c, u, True),
        8.0 * N * (2 + 2.0 ** -g.dim))
    if args.dim == 3:   # FAS machinery of a 9/5-node, n/n/2 level pair (BASELINE config 3)
        from paper_1407_6486_b200 import hierarchy
        from paper_1407_6486_b200.hierarchy import Level
        cfgm = MgConfig("jor-rb", 1.0, 1, 1)
        fl = Level(op, uniform_table(8), cfgm, FixedCycles(1), space_interp_order=4)
        cl = Level(HeatOperator(Grid(3, g.n // 2)), uniform_table(4), cfgm, FixedCycles(1),
                   space_interp_order=4)
        fst = NodeStates.spread(op, fl.table, u)
        rs = hierarchy.restrict_state(fst, fl, cl)
        nc = (g.n // 2 - 1) ** 3
        run("restrict_state", lambda: hierarchy.restrict_state(fst, fl, cl, out=rs),
            8.0 * N * 5 + 24.0 * 5 * nc)
        tau = hierarchy.compute_fas(fst, rs, fl, cl, 1 / 64)
        run("compute_fas", lambda: hierarchy.compute_fas(fst, rs, fl, cl, 1 / 64, out=tau),
            8.0 * N * 9 + 8.0 * 9 * nc)
        old = rs.copy()
        run("coarse_correction", lambda: hierarchy.coarse_correction(fst, old, rs, fl, cl),
            (8.0 * 2 + 16.0) * 9 * N)
    for M in (4, 8):
        table = uniform_table(M)
        st = NodeStates.spread(op, table, u)
        y0 = to_device(u.cpu().numpy())[0]
        r = torch.zeros(1, dtype=torch.float64, device="cuda")
        run(f"residual_max_M{M}", lambda st=st, y0=y0, r=r: residual_into(st, y0, 0.01, r),
            8.0 * N * (2 * M + 2))
        run(f"sweep_M{M}_jorrb_V11",
            lambda st=st, y0=y0: sdc_sweep(st, y0, 1 / 64, op, MgConfig("jor-rb", 1.0, 1, 1),
                                           FixedCycles(1)), None or 0.0)
    print(json.dumps({"dim": g.dim, "n": g.n, "dof": N, "opts": args.opts, "kernels": res}))


if __name__ == "__main__":
    main()
