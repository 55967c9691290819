"""Race / synchronisation probe of the shared-memory pipelines (GPU).

    python tools/race_probe.py [--part tma|mid|pfasst|big|all] [--stress N]

compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing
a reset), so this is the evidence instead: every kernel below is run with
the work split many different ways -- z-chunk floors 2..32, CTA targets
148..4096, forward/reverse chunk order, cooperative-kernel CTA counts --
while a second stream keeps other kernels in flight, and each result must
be bit-identical to the one-point kernels (no shared memory, no TMA).  A
missing barrier, a ring slot reused early or a wrong mbarrier phase shows
up as a differing value under some split / interleaving.  The same script
runs under compute-sanitizer where that tool is available.

Exercises, at sizes the sanitizer finishes in minutes: the TMA z-marching
kernels with their mbarrier rings and in-place shared-memory red/black
updates (k_zrb3 with both ring layouts, k_z1 apply / apply+rhs / residual /
Jacobi, k_z2, k_rfw, k_cubic5, k_chain_fw, engaged from 31^3 by
PL_OPT_ZMARCH_MIN_N), the cooperative small-level V-cycle (k_mid with its
grid.sync phases and the one-CTA shared-memory tail) at 63^3, and one
PFASST block of the same structure.  Each result is compared against the
one-point kernels, so a race that changed a value would also fail here.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1407_6486_b200 import _capi, hierarchy, sdc, transfers  # noqa: E402
from paper_1407_6486_b200._device import clone_field, to_device  # noqa: E402
from paper_1407_6486_b200.heat import Grid, HeatOperator, seeded_field  # noqa: E402
from paper_1407_6486_b200.hierarchy import Level  # noqa: E402
from paper_1407_6486_b200.multigrid import (FixedCycles, MgConfig, ShiftedOperator,  # noqa: E402
                                             v_cycle)
from paper_1407_6486_b200.pfasst import pfasst_run  # noqa: E402
from paper_1407_6486_b200.quadrature import uniform_table  # noqa: E402


STRESS = 1
SPLITS = [  # (z-chunk floor, CTA target, reverse-order mask, cooperative CTAs)
    (16, 1184, 3, 0), (2, 148, 0, 8), (4, 4096, 3, 32), (32, 296, 1, 148), (8, 592, 2, 0),
    (2, 4096, 0, 16), (16, 148, 3, 64), (4, 1184, 1, 0)]
_noise = {}


def _background():
    """Keep unrelated kernels in flight on a second stream."""
    if "s" not in _noise:
        _noise["s"] = torch.cuda.Stream()
        _noise["a"] = torch.randn(1 << 24, device="cuda", dtype=torch.float64)
    with torch.cuda.stream(_noise["s"]):
        for _ in range(4):
            _noise["a"].mul_(1.0000001).add_(1e-9)


def _split(i):
    zc, ctas, rev, mid = SPLITS[i % len(SPLITS)]
    _capi.set_option(_capi.OPT_ZC_FLOOR, zc)
    _capi.set_option(_capi.OPT_ZC_CTAS, ctas)
    _capi.set_option(_capi.OPT_ZREV, rev)
    _capi.set_option(_capi.OPT_MID_CTAS, mid)


def _reset():
    _capi.set_option(_capi.OPT_ZC_FLOOR, 16)
    _capi.set_option(_capi.OPT_ZC_CTAS, 148 * 8)
    _capi.set_option(_capi.OPT_ZREV, 3)
    _capi.set_option(_capi.OPT_MID_CTAS, 0)


def both(fn):
    """fn() with the one-point kernels, then STRESS x len(SPLITS) times with
    the TMA kernels (from 31^3) under every work split."""
    _capi.set_option(_capi.OPT_ZMARCH, 0)
    ref = fn()
    torch.cuda.synchronize()
    _capi.set_option(_capi.OPT_ZMARCH, 1)
    _capi.set_option(_capi.OPT_ZMARCH_MIN_N, 31)
    gots = []
    try:
        for i in range(STRESS * len(SPLITS)):
            _split(i)
            _background()
            gots.append(fn())
    finally:
        _reset()
        _capi.set_option(_capi.OPT_ZMARCH_MIN_N, 127)
    torch.cuda.synchronize()
    return gots, ref


def check(name, gots, ref):
    ref = ref if isinstance(ref, (list, tuple)) else [ref]
    bad = 0
    for got in gots:
        got = got if isinstance(got, (list, tuple)) else [got]
        bad += not all(torch.equal(a, b) for a, b in zip(got, ref))
    print(f"{name}: {len(gots) - bad}/{len(gots)} runs bit-identical", flush=True)
    if bad:
        raise SystemExit(f"{name} differs")


def part_tma(rng):
    g = Grid(3, 32)
    op = HeatOperator(g)
    u = to_device(rng.standard_normal(g.shape))[0]
    b = to_device(rng.standard_normal(g.shape))[0]
    for sm, om, pre, post in (("jor-rb", 1.0, 1, 1), ("jacobi", 2.0 / 3.0, 2, 2)):
        cfg = MgConfig(sm, om, pre, post)
        sop = ShiftedOperator(op, 0.01)
        rings = (0, 1, 4) if sm == "jor-rb" else (0,)
        for ring in rings:
            _capi.set_option(_capi.OPT_ZRB_RING, ring)
            check(f"v_cycle {sm} ring {ring}", *both(lambda: v_cycle(sop, u, b, cfg)))
        _capi.set_option(_capi.OPT_ZRB_RING, 0)
    c = to_device(rng.standard_normal((15,) * 3))[0]

    def cubic():
        f = clone_field(u)
        transfers.interp_cubic_into(c, f, True)
        return f
    check("interp_cubic (accumulate)", *both(cubic))
    check("interp_cubic", *both(lambda: transfers.interp_cubic(c)))
    fine = Level(op, uniform_table(4), MgConfig("jor-rb", 1.0, 1, 1), FixedCycles(1),
                 space_interp_order=4)
    coarse = Level(HeatOperator(Grid(3, 16)), uniform_table(2), MgConfig("jor-rb", 1.0, 1, 1),
                   FixedCycles(1), space_interp_order=4)
    y = rng.standard_normal((5,) + g.shape)

    def sweep_fas():
        st = sdc.NodeStates(fine.table, torch.from_numpy(y).cuda(),
                            torch.from_numpy(y).cuda())
        st.refresh(op)
        sdc.sdc_sweep(st, st.y[0].clone(), 1 / 64, op, fine.mg_cfg, fine.policy,
                      tau=torch.from_numpy(1e-3 * y).cuda())
        rs = hierarchy.restrict_state(st, fine, coarse)
        tau = hierarchy.compute_fas(st, rs, fine, coarse, 1 / 64,
                                    fine_tau=torch.from_numpy(1e-3 * y).cuda())
        new = sdc.NodeStates(coarse.table, rs.y + 1e-3, rs.f.clone())
        hierarchy.coarse_correction(st, rs, new, fine, coarse)
        return [st.y, st.f, rs.y, tau]
    check("sweep + restrict + FAS + correction", *both(sweep_fas))


def part_mid(rng):
    g = Grid(3, 64)
    u = to_device(rng.standard_normal(g.shape))[0]
    b = to_device(rng.standard_normal(g.shape))[0]
    sop = ShiftedOperator(HeatOperator(g), 0.013)
    cfg = MgConfig("jor-rb", 1.0, 1, 1)

    def vc():
        return v_cycle(sop, u, b, cfg)
    _capi.set_option(_capi.OPT_MID, 0)
    ref = vc()
    _capi.set_option(_capi.OPT_MID, 1)
    gots = []
    for i in range(STRESS * len(SPLITS)):
        _split(i)
        _background()
        for tail_n in (7, 15):
            _capi.set_option(_capi.OPT_MID_TAIL_N, tail_n)
            gots.append(vc())
    _capi.set_option(_capi.OPT_MID_TAIL_N, 15)
    _reset()
    torch.cuda.synchronize()
    check("cooperative mid V-cycle 63^3 (+ tail splits)", gots, ref)


def part_big(rng):
    """The production sizes: V(1,1) jor-rb cycles at 127^3 and 255^3 (6 + 3 rings
    in >= 32-plane chunks at 255^3) and the 255^3 cubic correction."""
    for n in (128, 256):
        g = Grid(3, n)
        u = to_device(rng.standard_normal(g.shape))[0]
        b = to_device(rng.standard_normal(g.shape))[0]
        sop = ShiftedOperator(HeatOperator(g), 1.0 / (4 * n))
        cfg = MgConfig("jor-rb", 1.0, 1, 1)
        check(f"v_cycle jor-rb {n - 1}^3", *both(lambda: v_cycle(sop, u, b, cfg)))
        c = to_device(rng.standard_normal((n // 2 - 1,) * 3))[0]

        def cubic():
            f = clone_field(u)
            transfers.interp_cubic_into(c, f, True)
            return f
        check(f"interp_cubic {n - 1}^3", *both(cubic))


def part_pfasst(rng):
    cfg = MgConfig("jor-rb", 1.0, 1, 1)
    levels = [Level(HeatOperator(Grid(3, n)), uniform_table(k - 1), cfg, FixedCycles(1),
                    space_interp_order=4) for n, k in ((32, 5), (16, 3))]
    u0 = torch.from_numpy(seeded_field(Grid(3, 32))).cuda()

    def run():
        return pfasst_run(levels, u0, 3 / 64, 3, tol=1e-9, max_iter=3).u
    check("pfasst block (rank streams)", *both(run))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="all", choices=["tma", "mid", "pfasst", "big", "all"])
    ap.add_argument("--stress", type=int, default=4, help="passes over the work splits")
    args = ap.parse_args()
    global STRESS
    STRESS = args.stress
    torch.cuda.set_device(0)
    rng = np.random.default_rng(2024)
    if args.part in ("tma", "all"):
        part_tma(rng)
    if args.part in ("mid", "all"):
        part_mid(rng)
    if args.part in ("pfasst", "all"):
        part_pfasst(rng)
    if args.part in ("big", "all"):
        part_big(rng)
    print("race probe done")


if __name__ == "__main__":
    main()
