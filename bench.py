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
    # name: (dim, ns, nodes, smoother, omega, pre, post, cycles, P, dt, tol)
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
    from paper_1407_6486_b200.multigrid import FixedCycles, MgConfig
    from paper_1407_6486_b200.quadrature import uniform_table
    cfg = MgConfig(w["smoother"], w["omega"], w["pre"], w["post"])
    return [Level(HeatOperator(Grid(w["dim"], n)), uniform_table(k - 1), cfg,
                  FixedCycles(w["cycles"]), space_interp_order=w["interp"])
            for n, k in zip(w["ns"], w["nodes"])]


def alg_bytes_of_one_substep(w):
    """Algorithmic bytes (SURVEY.md 8(d) model, counted by the runtime) of one
    fine-level sub-step: rhs + V-cycles + f refresh."""
    import torch
    from paper_1407_6486_b200 import _capi
    from paper_1407_6486_b200.heat import Grid, HeatOperator, seeded_field
    from paper_1407_6486_b200.multigrid import MgConfig, ShiftedOperator, vcycles_into
    from paper_1407_6486_b200._device import clone_field, to_device
    g = Grid(w["dim"], w["ns"][0])
    op = HeatOperator(g)
    u = to_device(seeded_field(g))[0]
    b = clone_field(u)
    cfg = MgConfig(w["smoother"], w["omega"], w["pre"], w["post"])
    sop = ShiftedOperator(op, w["dt"] / (w["nodes"][0] - 1))
    vcycles_into(sop, u, b, cfg, w["cycles"])        # warm (plans, LU)
    torch.cuda.synchronize()
    _capi.stats_reset()
    vcycles_into(sop, u, b, cfg, w["cycles"])
    torch.cuda.synchronize()
    st = _capi.stats()
    return sum(v[1] for v in st.values()) + (32.0 + 16.0) * g.dof


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
        dist.init_process_group("nccl", init_method="env://")
    executor = "nccl" if world > 1 else "serial"
    levels = build_levels(w)
    p, dt = w["p"], w["dt"]
    from paper_1407_6486_b200._device import to_device
    u0_host = seeded_field(Grid(w["dim"], w["ns"][0]))
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
    barrier()
    te0 = time.perf_counter()
    for _ in range(args.steps):
        r = pfasst_run(levels, u0_pinned, dt * p, p, tol=w["tol"], max_iter=20,
                       executor=executor, streams=streams)
        _ = r.u if isinstance(r.u, np.ndarray) else r.u.cpu()
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
            "metric": "PFASST time-steps/s (MG V-cycle DOF-updates/s and HBM GB/s in "
                      "'vcycle' / 'roofline')",
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
        out["block_over_sample"] = (alg_total / args.steps) / alg_bytes_of_one_substep(w)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


NCU_KERNEL = {"jor_rb": "k_zrb3", "interp_cubic": "k_cubic4", "restrict": "k_rfw",
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


def oracle_sample(w):
    """One fine-level sub-step of the workload via the oracle: rhs build,
    FixedCycles V-cycles, f refresh (sdc.py:102-112).  Returns seconds."""
    import numpy as np
    from oracle import pintlab_oracle as O
    op = O.Op(w["dim"], w["ns"][0])
    u = O.seeded_field(w["dim"], w["ns"][0])
    f = O.heat_apply(op, u)
    s = np.zeros_like(u)
    dtm = w["dt"] / (w["nodes"][0] - 1)
    cfg = O.Mg(w["smoother"], w["omega"], w["pre"], w["post"])
    t0 = time.perf_counter()
    rhs = u - dtm * f + s
    v, _, _ = O.mg_solve(op, dtm, u.copy(), rhs, cfg, O.Fixed(w["cycles"]))
    O.heat_apply(op, v)
    return time.perf_counter() - t0


def cpu_extrapolate(w, sample_s, threads, samples, block_alg_bytes, sample_alg_bytes):
    """Time-steps/s of the reference algorithm on this host, extrapolated from
    the measured sub-step samples by algorithmic bytes."""
    per_sample = sample_s / samples * threads      # seconds per sample per thread
    block_s = per_sample * block_alg_bytes / sample_alg_bytes / threads
    return w["p"] / block_s


def run_reference(args, w, ratio=None):
    rank, world, _ = env_rank()
    if rank != 0:
        return None
    threads = max(1, min(8, os.cpu_count() or 1))
    # algorithmic bytes of a whole block over those of one sample (the same
    # model the GPU arm counts): live from the GPU arm, else its recorded value
    model = {"block_over_sample": ratio} if ratio else BLOCK_MODEL[args.workload]
    # one single-threaded worker PROCESS per core (spawned: numpy/scipy BLAS
    # called from several threads of one process aborted once with a heap
    # error); a round's time is its slowest worker's sample (they run together)
    import concurrent.futures as cf
    import multiprocessing as mp
    saved = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                             "MKL_NUM_THREADS", "CUDA_VISIBLE_DEVICES")}
    os.environ.update(OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
                      CUDA_VISIBLE_DEVICES="")
    vals = []
    try:
        with cf.ProcessPoolExecutor(max_workers=threads,
                                    mp_context=mp.get_context("spawn")) as pool:
            for i in range(args.warmup + args.steps):
                wall = max(pool.map(oracle_sample, [w] * threads))
                if i >= args.warmup:
                    vals.append(wall)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    wall = sum(vals)
    samples = threads * len(vals)
    value = w["p"] / (wall / samples * model["block_over_sample"])
    return {"impl": "reference", "metric": "PFASST time-steps/s", "value": value,
            "unit": "time-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
            "config": {"workload": args.workload},
            "cpu_baseline": {"value": value, "unit": "time-steps/s", "cores": threads,
                             "kind": "port",
                             "sample": f"{samples} fine sub-steps (rhs + {w['cycles']} V-cycle "
                                       f"+ f refresh at {w['ns'][0] - 1}^{w['dim']}) on "
                                       f"{threads} single-threaded processes; block time "
                                       f"extrapolated x"
                                       f"{model['block_over_sample']:.1f} by algorithmic bytes"},
            "e2e": {"value": value, "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


# block / sample algorithmic-byte ratios measured by the GPU arm (the runtime's
# byte counter over one block vs one fine sub-step); refreshed by --calibrate
BLOCK_MODEL = {
    "cfg3": {"block_over_sample": 2230.4},     # profiles/r01/bench.json (GPU arm, live)
    "cfg4": {"block_over_sample": 1048.1},
    "cfg2": {"block_over_sample": 1124.9},
}


def main():
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
            ref = run_reference(argparse.Namespace(warmup=0, steps=1, workload=args.workload),
                                w, out["block_over_sample"])
            cb = dict(ref["cpu_baseline"])
            out["cpu_baseline"] = cb
        print(json.dumps(out))


if __name__ == "__main__":
    main()
