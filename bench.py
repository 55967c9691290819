"""Benchmark: PFASST time-steps/s of the B200 hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
    python bench.py --impl reference ...      (the reference's CPU algorithm)

A *step* is one PFASST block of P = 8 time steps of the workload (one pass
of the hot path over the synthetic input), so ``value`` = 8 * K / elapsed.
The default workload is BASELINE config 3: 3-D heat, 255^3 / 127^3 / 63^3,
9/5/3 uniform nodes, jor-rb (omega = 1) V(1,1), 1 V-cycle per sub-step,
8 time ranks, dt = 1/64, tol 1e-10, max_iter 20.  Every
field (133 MB) exceeds L2 (126 MB), so no flush is needed between steps.

Printed JSON (rank 0, one line): value (device-resident input), e2e (host
buffers through the public API), roofline of the dominant kernel with CUDA
events inside the timed region, cpu_baseline (the oracle on a bounded
sample, extrapolated), clocks sampled during the timed region.
"""
from __future__ import annotations

import argparse
import faulthandler
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # BASELINE.json configs: grids, nodes, smoother, sweeps,
    # V-cycles per sub-step (or a ToTolerance policy), time ranks, dt, PFASST tol
    "cfg0": dict(dim=1, ns=(256, 128), nodes=(5, 3), smoother="jacobi", omega=2.0 / 3.0,
                 pre=2, post=2, cycles=None, policy=("tol", 1e-12), p=4, dt=1.0 / 32,
                 tol=1e-10, interp=4, u0="sine"),
    "cfg1": dict(dim=1, ns=(256, 128), nodes=(5, 3), smoother="jacobi", omega=2.0 / 3.0,
                 pre=2, post=2, cycles=1, p=4, dt=1.0 / 32, tol=1e-10, interp=4, u0="sine"),
    "cfg3": dict(dim=3, ns=(256, 128, 64), nodes=(9, 5, 3), smoother="jor-rb", omega=1.0,
                 pre=1, post=1, cycles=1, p=8, dt=1.0 / 64, tol=1e-10, interp=4),
    "cfg4": dict(dim=3, ns=(512, 256), nodes=(5, 3), smoother="jacobi", omega=2.0 / 3.0,
                 pre=2, post=2, cycles=1, p=8, dt=1.0 / 64, tol=1e-10, interp=4),
    "cfg2": dict(dim=2, ns=(1024, 512), nodes=(5, 3), smoother="jacobi", omega=2.0 / 3.0,
                 pre=2, post=2, cycles=1, p=8, dt=1.0 / 64, tol=1e-10, interp=4),
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm


def build_levels(w):
    from paper_1407_6486_b200.heat import Grid, HeatOperator
    from paper_1407_6486_b200.hierarchy import Level
    from paper_1407_6486_b200.multigrid import FixedCycles, MgConfig, ToTolerance
    from paper_1407_6486_b200.quadrature import uniform_table
    cfg = MgConfig(w["smoother"], w["omega"], w["pre"], w["post"])
    pol = ToTolerance(w["policy"][1]) if w.get("policy") else FixedCycles(w["cycles"])
    return [Level(HeatOperator(Grid(w["dim"], n)), uniform_table(k - 1), cfg, pol,
                  space_interp_order=w["interp"])
            for n, k in zip(w["ns"], w["nodes"])]


def initial_field(w):
    """u0 of the workload: sin(pi x) for the 1-D configs, the
    seeded Fourier-mode field otherwise."""
    from paper_1407_6486_b200.heat import Grid, initial_condition, seeded_field
    g = Grid(w["dim"], w["ns"][0])
    return initial_condition(g, 1) if w.get("u0") == "sine" else seeded_field(g)


def release_device_caches():
    """Drop the multigrid plans and scratch of the previous workload."""
    import gc

    import torch
    from paper_1407_6486_b200 import _device, multigrid, pfasst
    pfasst.release_engines()
    multigrid._plans.clear()
    _device.release_scratch()
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def measure_workload(name, steps=3, warmup=2):
    """PFASST time-steps/s of another BASELINE configuration on this GPU
    (device-resident u0, rank streams where they fit; CUDA events)."""
    import torch
    from paper_1407_6486_b200._device import to_device
    from paper_1407_6486_b200.pfasst import pfasst_run
    w = WORKLOADS[name]
    levels = build_levels(w)
    u0 = to_device(initial_field(w))[0]
    p, dt = w["p"], w["dt"]
    res = None
    for _ in range(warmup):
        res = pfasst_run(levels, u0, dt * p, p, tol=w["tol"], max_iter=20)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(steps):
        res = pfasst_run(levels, u0, dt * p, p, tol=w["tol"], max_iter=20)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    out = {"value": p / (ms / 1e3), "unit": "time-steps/s", "ms_per_step": ms, "steps": steps,
           "warmup": warmup, "grids": [n - 1 for n in w["ns"]], "dim": w["dim"],
           "nodes": list(w["nodes"]), "smoother": w["smoother"],
           "policy": (f"ToTolerance({w['policy'][1]:g})" if w.get("policy")
                      else f"FixedCycles({w['cycles']})"),
           "time_ranks": p, "rank_iterations": res.rank_iterations[0],
           "rank_vcycles": res.rank_vcycles[0]}
    del levels, u0, res
    release_device_caches()
    return out


def run_ours(args, w):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1407_6486_b200 import _capi
    from paper_1407_6486_b200.heat import Grid, seeded_field
    from paper_1407_6486_b200.pfasst import pfasst_run

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    for kv in filter(None, args.opts.split(",")):
        k, v = kv.split("=")
        _capi.set_option(int(k), int(v))
    if world > 1:
        # communicator set-up lines (ranks, NVLink/NVLS transport) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", init_method="env://",
                                device_id=torch.device("cuda", local))
    executor = "nccl" if world > 1 else "serial"
    levels = build_levels(w)
    p, dt = w["p"], w["dt"]
    from paper_1407_6486_b200._device import to_device
    u0_host = initial_field(w)
    u0_dev = to_device(u0_host)[0]            # device field in the library layout
    u0_pinned = torch.from_numpy(u0_host).pin_memory()

    streams = not args.no_streams

    def step(u0, streams=streams):
        return pfasst_run(levels, u0, dt * p, p, tol=w["tol"], max_iter=20, executor=executor,
                          streams=streams)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (plans, LU factors, allocations)
    res = None
    for _ in range(args.warmup):
        res = step(u0_dev)
    barrier()
    # which kernel dominates?  one untimed profiling block with events on all
    names = _capi.kind_names()
    _capi.timing_enable(names)
    step(u0_dev, streams=False)       # per-launch events: no cross-rank overlap
    barrier()
    per_kind = {n: _capi.timing_collect(n) for n in names}
    max_launch_bytes = {n: max(_capi.timing_by_size(n) or {0.0: None}) for n in names}
    _capi.timing_enable(None)
    total_ms = sum(v[1] for v in per_kind.values())
    dom_all = max(per_kind, key=lambda n: per_kind[n][1])
    # the roofline is quoted on the dominant HBM-bound kind: one whose largest
    # launch streams more than the L2 holds.  Kinds that only ever touch
    # L2-resident fields (the cooperative small-level V-cycle on <= 63^3) are
    # latency-bound; their share is reported beside, not against HBM.
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    hbm_kinds = [n for n in names if max_launch_bytes[n] > l2 and per_kind[n][0]]
    dom = max(hbm_kinds, key=lambda n: per_kind[n][1]) if hbm_kinds else dom_all

    # ---- timed region: device-resident input (sweeps replay as CUDA graphs)
    stream = torch.cuda.current_stream()
    _capi.stats_reset()
    barrier()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            res = step(u0_dev)
        t1.record(stream)
        barrier()
    ms = t0.elapsed_time(t1)
    stats = _capi.stats()
    launches = sum(v[0] for v in stats.values())
    alg_total = sum(v[1] for v in stats.values())
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- roofline pass: the same K steps again with CUDA events around every
    # launch of the dominant kernel (per-launch events need eager launches, so
    # this pass is timed separately; its step time is reported beside)
    _capi.timing_enable([dom])
    barrier()
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    r0.record(stream)
    for _ in range(args.steps):
        step(u0_dev, streams=False)
    r1.record(stream)
    barrier()
    ms_instr = r0.elapsed_time(r1)
    n_dom, ms_dom, bytes_dom = _capi.timing_collect(dom)
    by_size = _capi.timing_by_size(dom)
    _capi.timing_enable(None)

    # ---- e2e: host (pinned) buffers through the public API
    # (input from pinned host memory, result into a reused pinned host buffer:
    # both copies are inside the timed region, every step)
    out_pinned = torch.empty(tuple(u0_pinned.shape), dtype=torch.float64).pin_memory()
    barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        r = pfasst_run(levels, u0_pinned, dt * p, p, tol=w["tol"], max_iter=20,
                       executor=executor, streams=streams, out=out_pinned)
        assert r.u is out_pinned
    barrier()
    e2e_s = time.perf_counter() - te0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    out = None
    if rank == 0:
        peak, peak_src = peaks()
        steps_done = p * args.steps
        value = steps_done / (ms / 1e3)
        # the roofline is quoted on the dominant kind's fine-grid launches (the
        # largest per-launch byte count): one kernel at one size, comparable
        # with its ncu capture
        if by_size:
            b_top = max(by_size)
            c_top, t_top = by_size[b_top]
            achieved = b_top / ((t_top / c_top) / 1e3) / 1e9
        else:
            b_top = c_top = None
            achieved = (bytes_dom / n_dom) / ((ms_dom / n_dom) / 1e3) / 1e9 if n_dom else None
        traffic, traffic_src = ncu_traffic(dom)
        out = {
            "metric": "PFASST time-steps/s",
            "value": value, "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Fourier-mode u0, SURVEY.md 8(d))",
            "config": {"workload": args.workload, "grids": [n - 1 for n in w["ns"]],
                       "dim": w["dim"], "nodes": list(w["nodes"]), "smoother": w["smoother"],
                       "omega": w["omega"], "sweeps": [w["pre"], w["post"]],
                       "vcycles_per_substep": w["cycles"], "time_ranks": p, "dt": dt,
                       "tol": w["tol"], "max_iter": 20, "executor": executor,
                       "rank_streams": streams,
                       **({"options": args.opts} if args.opts else {}),
                       "parallelism": f"time{world}",
                       "l2": "fields (>=133 MB) exceed the 126 MB L2; no flush needed",
                       "rank_iterations": res.rank_iterations[0],
                       "rank_vcycles": res.rank_vcycles[0]},
            "e2e": {"value": steps_done / e2e_s, "unit": "time-steps/s",
                    "h2d_bytes_per_step": int(u0_host.nbytes),
                    "d2h_bytes_per_step": int(u0_host.nbytes)},
            "gpu_launches": launches,
            "dominant_kind": {"name": dom_all,
                              "share_of_step": round(per_kind[dom_all][1] / total_ms, 4),
                              "max_launch_mb": round(max_launch_bytes[dom_all] / 1e6, 1),
                              "note": ("the roofline kernel" if dom_all == dom else
                                       "latency-bound: every launch works on L2-resident "
                                       "fields (< L2 = %.0f MB); reported by share, the "
                                       "roofline is quoted on the dominant HBM-bound kind"
                                       % (l2 / 1e6))},
            "roofline": {"bound": "hbm", "kernel": f"{dom} @ {w['ns'][0] - 1}^{w['dim']}",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None,
                         "alg_bytes_per_launch": b_top, "launches": c_top,
                         "all_levels_achieved":
                             (bytes_dom / n_dom) / ((ms_dom / n_dom) / 1e3) / 1e9
                             if n_dom else None,
                         "per_level": {f"{b / 1e6:.1f}MB": {
                             "launches": c, "avg_us": 1e3 * t / c,
                             "gbs": b / (t / c / 1e3) / 1e9}
                             for b, (c, t) in sorted(by_size.items(), reverse=True)},
                         "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "launches_timed": n_dom,
                         "kernel_share_of_step": ms_dom / ms_instr if ms_instr else None,
                         "instrumented_ms_per_step": ms_instr / args.steps,
                         "profile_block_shares": {k: round(v[1] / total_ms, 4)
                                                  for k, v in per_kind.items() if v[0]}},
            "alg_gbs_whole_step": alg_total / (ms / 1e3) / 1e9,
            "clocks": clk.summary(),
        }
        out["vcycle"] = vcycle_rate(w)
    if world == 1 and not args.no_other_configs:
        # the other BASELINE configurations, a few blocks each (not the headline)
        release_device_caches()
        others = {}
        for name in ("cfg0", "cfg1", "cfg2", "cfg4"):
            if name == args.workload:
                continue
            try:
                others[name] = measure_workload(name)
            except Exception as exc:           # report, never hide the headline
                others[name] = {"error": repr(exc)[:200]}
        if out is not None:
            out["other_configs"] = others
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


NCU_KERNEL = {"jor_rb": "k_zrb3", "interp_cubic": "k_cubic5", "restrict": "k_rfw",
              "mg_mid": "k_mid"}


def ncu_traffic(kind):
    """DRAM bytes (read + write) per launch of the kind's fine-grid kernel from
    the latest committed ncu --set full capture (profiles/*/top255_full.txt),
    or (None, reason)."""
    import glob
    import re
    name = NCU_KERNEL.get(kind)
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                          "profiles", "*", "top255_full.txt")))
    if not name or not files:
        return None, "no ncu capture committed for this kernel"
    text = open(files[-1]).read()
    blocks = text.split("\n\n")
    for blk in blocks:
        if re.search(r"::%s[<(]" % name, blk):
            m = re.search(r"=> DRAM traffic ([0-9.]+) MB", blk)
            if m:
                rel = os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))
                return float(m.group(1)) * 1e6, f"{rel} (first {name} launch, 255^3)"
    return None, f"{name} not in {os.path.basename(files[-1])}"


def vcycle_rate(w, reps=10):
    """Standalone MG V-cycle DOF-updates/s at the workload's fine grid
    (solve(FixedCycles) semantics)."""
    import torch
    from paper_1407_6486_b200 import _capi
    from paper_1407_6486_b200.heat import Grid, HeatOperator, seeded_field
    from paper_1407_6486_b200.multigrid import MgConfig, ShiftedOperator, vcycles_into
    from paper_1407_6486_b200._device import clone_field, to_device
    g = Grid(w["dim"], w["ns"][0])
    u = to_device(seeded_field(g))[0]
    b = clone_field(u)
    cfg = MgConfig(w["smoother"], w["omega"], w["pre"], w["post"])
    sop = ShiftedOperator(HeatOperator(g), w["dt"] / (w["nodes"][0] - 1))
    for _ in range(3):
        vcycles_into(sop, u, b, cfg, 1)
    torch.cuda.synchronize()
    _capi.stats_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    vcycles_into(sop, u, b, cfg, reps)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alg = sum(v[1] for v in _capi.stats().values()) / reps
    return {"grid": list(g.shape), "ms_per_cycle": ms,
            "dof_updates_per_s": g.dof / (ms / 1e3), "alg_gbs": alg / (ms / 1e3) / 1e9}


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm (oracle port, numpy)
#
# A PFASST block is (K + P - 1) rank-iterations deep on the reference's
# threaded executor (one thread per time rank; rank n's iteration k waits for
# rank n-1's, pfasst.py:231-253), after a predictor of P coarsest sweeps and
# one interpolate_up (pfasst.py:166-181).  One rank-iteration at full size is
# split into units -- restrict + FAS per level, the coarsest sweep, per level
# the coarse correction and the sweep, and the finest sweep as its quadrature,
# one sub-step (x M) and the hand-off + residual -- and every unit is timed at
# full size on min(P, cores) single-threaded worker processes running it
# concurrently (each process is one time rank with its own state), so the
# memory-bandwidth contention is that of P concurrent ranks.  Then
#   block = (K + P - 1) * sum(units) + P * sweep_coarsest + sum(corrections)
# with K the GPU run's iteration count (20 for cfg3: no rank converges).


def cpu_units(w):
    """Unit names of one rank-iteration, in the order mlsdc_iteration runs
    them (hierarchy.py:166-203), and how often each occurs."""
    L = len(w["ns"])
    units = [f"down{l}" for l in range(L - 1)] + [f"sweep{L - 1}"]
    for l in range(L - 2, -1, -1):
        units.append(f"corr{l}")
        if l > 0:
            units.append(f"sweep{l}")
    units += ["quad0", "sub0", "resid0"]
    mult = {u: 1 for u in units}
    mult["sub0"] = w["nodes"][0] - 1
    return units, mult


class _CpuRank:
    """One time rank's full-size state on the oracle, and the units of a
    rank-iteration restated from oracle primitives (mlsdc_iteration and
    sdc_sweep split where the units cut them)."""

    def __init__(self, w):
        import numpy as np
        from oracle import pintlab_oracle as O
        self.O, self.np, self.w = O, np, w
        self.dt = w["dt"]
        pol = O.ToTol(w["policy"][1]) if w.get("policy") else O.Fixed(w["cycles"])
        self.lv = [O.Lvl(O.Op(w["dim"], n), O.uniform_table(k - 1),
                         O.Mg(w["smoother"], w["omega"], w["pre"], w["post"]), pol,
                         w["interp"])
                   for n, k in zip(w["ns"], w["nodes"])]
        u0 = (O.sine_mode(w["dim"], w["ns"][0], 1) if w.get("u0") == "sine"
              else O.seeded_field(w["dim"], w["ns"][0]))
        self.ts = O.Step.spread(self.lv, u0)
        self.old = [s.copy() for s in self.ts.states]
        self.s = None

    def run(self, unit):
        O, np, ts, lv, dt = self.O, self.np, self.ts, self.lv, self.dt
        kind, l = unit[:-1], int(unit[-1])
        if kind == "down":               # hierarchy.py:177-186
            r = O.restrict_state(ts.states[l], lv[l], lv[l + 1])
            ts.tau[l + 1] = O.compute_fas(ts.states[l], r, lv[l], lv[l + 1], dt,
                                          fine_tau=ts.tau[l])
            self.old[l + 1] = r.copy()
            ts.states[l + 1] = r
            ts.y0[l + 1] = r.y[0].copy()
        elif kind == "sweep":            # sdc.py:84-114
            O._sweep_level(ts, l, dt, None)
        elif kind == "corr":             # hierarchy.py:196-198
            O.coarse_correction(ts.states[l], self.old[l + 1], ts.states[l + 1], lv[l],
                                lv[l + 1])
            ts.y0[l] = ts.states[l].y[0].copy()
        elif kind == "quad":             # sdc.py:93-97
            st, q = ts.states[0], ts.states[0].table.q
            self.s = dt * np.tensordot(q[1:] - q[:-1], st.f, axes=(1, 0))
            st.y[0] = ts.y0[0]
            st.f[0] = O.heat_apply(lv[0].op, ts.y0[0])
        elif kind == "sub":              # sdc.py:98-113, a middle sub-step
            st, m = ts.states[0], (self.w["nodes"][0] - 1) // 2
            if self.s is None:
                self.run("quad0")
            dtm = float(st.table.gammas[m]) * dt
            rhs = st.y[m] - dtm * st.f[m + 1] + self.s[m]
            if ts.tau[0] is not None:
                rhs = rhs + (ts.tau[0][m + 1] - ts.tau[0][m])
            u, _, _ = O.mg_solve(lv[0].op, dtm, st.y[m + 1].copy(), rhs, lv[0].cfg,
                                 lv[0].policy)
            st.y[m + 1] = u
            st.f[m + 1] = O.heat_apply(lv[0].op, u)
        elif kind == "resid":            # pfasst.py:189-200: hand-off + residual
            st = ts.states[0]
            st.y[0] = ts.y0[0]
            st.f[0] = O.heat_apply(lv[0].op, ts.y0[0])
            O.residual(st, ts.y0[0], dt)
        else:
            raise ValueError(unit)


def _cpu_worker(conn, w):
    t0 = time.perf_counter()
    rank = _CpuRank(w)
    conn.send(time.perf_counter() - t0)
    while True:
        unit = conn.recv()
        if unit is None:
            break
        t0 = time.perf_counter()
        rank.run(unit)
        conn.send(time.perf_counter() - t0)
    conn.close()


def _mem_available():
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


class CpuRanks:
    """min(P, cores) worker processes (spawned, single-threaded BLAS), each
    holding one time rank's state; ``time(unit)`` runs the unit on all of
    them at once and returns the wall time."""

    def __init__(self, w, max_procs=None):
        import multiprocessing as mp
        self.cores = os.cpu_count() or 1
        n = max(1, min(w["p"], self.cores, max_procs or w["p"]))
        # bound by memory: about 3 (M+1) + 8 fine fields per process
        per = 8.0 * (w["ns"][0] - 1) ** w["dim"] * (3 * w["nodes"][0] + 8)
        avail = _mem_available()
        if avail:
            n = max(1, min(n, int(0.7 * avail // per)))
        self.procs_n = n
        saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                                 "MKL_NUM_THREADS", "CUDA_VISIBLE_DEVICES")}
        os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
                          CUDA_VISIBLE_DEVICES="")
        ctx = mp.get_context("spawn")
        self.conns, self.procs = [], []
        try:
            for _ in range(n):
                a, b = ctx.Pipe()
                pr = ctx.Process(target=_cpu_worker, args=(b, w), daemon=True)
                pr.start()
                self.conns.append(a)
                self.procs.append(pr)
        finally:
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        self.setup_s = max(c.recv() for c in self.conns)

    def time(self, unit):
        t0 = time.perf_counter()
        for c in self.conns:
            c.send(unit)
        for c in self.conns:
            c.recv()
        return time.perf_counter() - t0

    def close(self):
        for c in self.conns:
            try:
                c.send(None)
            except Exception:
                pass
        for pr in self.procs:
            pr.join(timeout=10)

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def host_info():
    import numpy as np
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import scipy
        sv = scipy.__version__
    except Exception:
        sv = None
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "blas_threads": 1,
            "numpy": np.__version__, "scipy": sv}


def cpu_block_estimate(w, unit_s, iters):
    """(seconds per block, seconds per rank-iteration) from the per-unit
    concurrent wall times."""
    units, mult = cpu_units(w)
    t_ri = sum(unit_s[u] * mult[u] for u in units)
    L = len(w["ns"])
    predictor = w["p"] * unit_s[f"sweep{L - 1}"] + sum(unit_s[f"corr{l}"]
                                                        for l in range(L - 1))
    return (iters + w["p"] - 1) * t_ri + predictor, t_ri


def run_reference(args, w, iters=None, passes=None, max_procs=None):
    """The reference's algorithm (oracle port) on this host's cores: each
    step times one unit of a rank-iteration (round robin) on the concurrent
    rank processes; ``passes`` (the cpu_baseline leg) times every unit that
    many times instead."""
    rank, world, _ = env_rank()
    if rank != 0:
        return None
    iters = iters or 20
    units, _ = cpu_units(w)
    samples = {u: [] for u in units}
    with CpuRanks(w, max_procs) as pool:
        if passes:
            for _ in range(passes):
                for u in units:
                    samples[u].append(pool.time(u))
            steps_note = f"{passes} pass(es) over the {len(units)} units"
        else:
            for i in range(args.warmup + args.steps):
                u = units[i % len(units)]
                t = pool.time(u)
                if i >= args.warmup:
                    samples[u].append(t)
            missing = [u for u in units if not samples[u]]
            for u in missing:          # fewer timed steps than units
                samples[u].append(pool.time(u))
            steps_note = (f"{args.steps} timed steps, one unit each (round robin)" +
                          (f"; {len(missing)} units timed after the loop" if missing else ""))
        nproc, setup_s = pool.procs_n, pool.setup_s
    all_t = [t for v in samples.values() for t in v]
    unit_s = {u: statistics.mean(v) for u, v in samples.items()}
    block_s, t_ri = cpu_block_estimate(w, unit_s, iters)
    value = w["p"] / block_s
    grid = f"{w['ns'][0] - 1}^{w['dim']}"
    sample = (f"full-size ({grid}) units of one rank-iteration of the oracle port, each run "
              f"concurrently on {nproc} single-threaded processes (one time rank each): "
              f"{steps_note}; rank-iteration {t_ri:.1f} s; block = (K + P - 1) = "
              f"{iters + w['p'] - 1} rank-iterations + predictor = {block_s:.0f} s "
              f"(threaded-executor wavefront bound, pfasst.py:231-253)")
    return {"impl": "reference", "metric": "PFASST time-steps/s", "value": value,
            "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup,
            # wall time of one timed step (one unit on every rank process);
            # ``value`` is P / the block time those units add up to
            "ms_per_step": 1e3 * statistics.mean(all_t),
            "higher_is_better": True, "dtype": "f64",
            "data": "synthetic (seeded Fourier-mode u0, SURVEY.md 8(d))",
            "config": {"workload": args.workload},
            "cpu_baseline": {"value": value, "unit": "time-steps/s", "cores": nproc,
                             "kind": "port", "sample": sample,
                             "unit_seconds": {u: round(t, 3) for u, t in unit_s.items()},
                             "rank_iteration_s": t_ri, "block_s": block_s,
                             "setup_s": setup_s, "host": host_info()},
            "e2e": {"value": value, "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true",
                    help="skip the short runs of the other BASELINE configurations")
    ap.add_argument("--no-streams", action="store_true",
                    help="issue all time ranks on one stream (A/B of the wavefront overlap)")
    ap.add_argument("--opts", default="", help="pl_set_option pairs KEY=VAL,... (A/B only)")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        out = run_reference(args, w)
        if out is not None:
            print(json.dumps(out))
        return
    out = run_ours(args, w)
    if out is not None:
        if not args.no_cpu_baseline and out["n_gpus"] == 1:
            ref = run_reference(argparse.Namespace(warmup=0, steps=0, workload=args.workload),
                                w, iters=max(out["config"]["rank_iterations"]), passes=1)
            out["cpu_baseline"] = dict(ref["cpu_baseline"])
        print(json.dumps(out))


if __name__ == "__main__":
    main()
