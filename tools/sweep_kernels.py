"""Per-launch CUDA-event timing of every kernel kind inside SDC sweeps of one
fine level (default: BASELINE config 3's 255^3, 8 sub-steps, jor-rb V(1,1)).

    python tools/sweep_kernels.py [--n 256] [--m 8] [--sweeps 3] [--opts K=V,...]

Prints, per kind and per launch size, launches, mean microseconds and the
algorithmic GB/s (SURVEY.md 8(d) bytes / mean launch time)."""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_6486_b200 import _capi  # noqa: E402
from paper_1407_6486_b200.heat import Grid, HeatOperator, seeded_field  # noqa: E402
from paper_1407_6486_b200.multigrid import FixedCycles, MgConfig  # noqa: E402
from paper_1407_6486_b200.quadrature import uniform_table  # noqa: E402
from paper_1407_6486_b200.sdc import NodeStates, sdc_sweep  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--m", type=int, default=8)
    ap.add_argument("--sweeps", type=int, default=3)
    ap.add_argument("--tau", action="store_true")
    ap.add_argument("--cubic", action="store_true", help="also time the cubic correction")
    ap.add_argument("--opts", default="")
    a = ap.parse_args()
    for kv in filter(None, a.opts.split(",")):
        k, v = kv.split("=")
        _capi.set_option(int(k), int(v))
    g = Grid(3, a.n)
    op = HeatOperator(g)
    table = uniform_table(a.m)
    u0 = torch.from_numpy(seeded_field(g)).cuda()
    tau = (torch.randn((a.m + 1,) + g.shape, dtype=torch.float64, device="cuda") * 1e-3
           if a.tau else None)
    cfg = MgConfig("jor-rb", 1.0, 1, 1)
    st = NodeStates.spread(op, table, u0)
    sdc_sweep(st, u0, 1.0 / 64, op, cfg, FixedCycles(1), tau)
    torch.cuda.synchronize()
    names = _capi.kind_names()
    _capi.timing_enable(names)
    from paper_1407_6486_b200.sdc import residual
    for _ in range(a.sweeps):
        sdc_sweep(st, u0, 1.0 / 64, op, cfg, FixedCycles(1), tau)
        residual(st, u0, 1.0 / 64, tau)          # the collocation residual after each sweep
    if a.cubic:      # the coarse correction's cubic interpolation (accumulate)
        from paper_1407_6486_b200 import transfers
        from paper_1407_6486_b200._device import to_device
        c = to_device(torch.randn(((a.n // 2) - 1,) * 3, dtype=torch.float64))[0]
        for _ in range(a.sweeps * a.m):
            transfers.interp_cubic_into(c, st.y[0], True)
    torch.cuda.synchronize()
    total = 0.0
    rows = []
    for name in names:
        for b, (cnt, ms) in sorted(_capi.timing_by_size(name).items(), reverse=True):
            us = 1e3 * ms / cnt
            total += ms
            rows.append((name, b, cnt, us, b / us / 1e3))
    _capi.timing_enable(None)
    print(f"{'kind':<16}{'MB/launch':>10}{'n':>6}{'us':>10}{'GB/s':>9}{'share':>8}")
    for name, b, cnt, us, gbs in rows:
        print(f"{name:<16}{b / 1e6:>10.1f}{cnt:>6}{us:>10.1f}{gbs:>9.0f}"
              f"{cnt * us / 1e3 / total:>8.3f}")
    print(f"total {total / a.sweeps:.3f} ms per sweep")


if __name__ == "__main__":
    main()
