"""Interleaved in-process A/B of library options on one jor-rb V(1,1) cycle.

    python tools/mid_ab.py --n 64 --variants "" "7=7" "13=96" [--reps 200]

Every variant must set each key it touches (no reset between variants, e.g.
"7=15" against "7=7").  Each round times every variant once (CUDA events on the launching stream), so
clock and thermal drift hit all variants alike; prints the median per variant."""
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


def parse(v):
    return [tuple(int(x) for x in kv.split("=")) for kv in filter(None, v.split(","))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--variants", nargs="+", default=["7=15", "7=7"])
    args = ap.parse_args()
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
    times = {v: [] for v in args.variants}
    for rep in range(args.reps + 5):
        for v in args.variants:
            opts = parse(v)
            for k, val in opts:
                _capi.set_option(k, val)
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _capi.check(lib.pl_mg_vcycles(p.handle.value, u.data_ptr(), b.data_ptr(), sig, 1, 0, s))
            e.record()
            e.synchronize()
            if rep >= 5:
                times[v].append(a.elapsed_time(e))
    for v in args.variants:
        print(f"n={args.n} opts={v or 'default'}: median {np.median(times[v]) * 1e3:.1f} us")


if __name__ == "__main__":
    main()
