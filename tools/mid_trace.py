"""Per-phase timeline of the cooperative small-level V-cycle kernel (k_mid).

    PL_MID_TRACE=1 python tools/mid_trace.py [--n 256] [--opts K=V,...]

Runs a few jor-rb V(1,1) cycles at n and prints, from the library's stderr
trace, the %globaltimer deltas between grid-wide phases; then the median
V-cycle time with tracing off (run without PL_MID_TRACE for that)."""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_6486_b200 import _capi  # noqa: E402
from paper_1407_6486_b200._device import to_device  # noqa: E402
from paper_1407_6486_b200.heat import Grid, HeatOperator  # noqa: E402
from paper_1407_6486_b200.multigrid import MgConfig, plan_for  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--opts", default="")
    args = ap.parse_args()
    for kv in filter(None, args.opts.split(",")):
        k, v = kv.split("=")
        _capi.set_option(int(k), int(v))
    g = Grid(3, args.n)
    rng = np.random.default_rng(0)
    u = to_device(rng.standard_normal(g.shape))[0]
    b = to_device(rng.standard_normal(g.shape))[0]
    op = HeatOperator(g)
    lib = _capi.lib()
    s = torch.cuda.current_stream().cuda_stream
    sig = 1.0 / 512
    p = plan_for(op, MgConfig("jor-rb", 1.0, 1, 1))
    p.ensure(sig)
    ts = []
    for _ in range(args.reps + 2):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _capi.check(lib.pl_mg_vcycles(p.handle.value, u.data_ptr(), b.data_ptr(), sig, 1, 0, s))
        e.record()
        e.synchronize()
        ts.append(a.elapsed_time(e))
    print(f"n={args.n} V-cycle ms: median {np.median(ts[2:]):.4f} all {[round(t, 4) for t in ts]}")


if __name__ == "__main__":
    main()
