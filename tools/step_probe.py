"""Per-block timing probe for the default bench workload: host enqueue time
of each pfasst_run block (no sync) vs the device time of the block.

    python tools/step_probe.py [--steps 8] [--no-streams] [--opts K=V,...]"""
from __future__ import annotations

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1407_6486_b200 import _capi  # noqa: E402
from paper_1407_6486_b200._device import to_device  # noqa: E402
from paper_1407_6486_b200.heat import Grid, seeded_field  # noqa: E402
from paper_1407_6486_b200.pfasst import pfasst_run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--no-streams", action="store_true")
    ap.add_argument("--opts", default="")
    ap.add_argument("--nosync", action="store_true",
                    help="experiment: never wait for residuals (every rank runs max_iter)")
    a = ap.parse_args()
    if a.nosync:
        from paper_1407_6486_b200 import pfasst
        pfasst.DeviceEngine.read = lambda self, n, handle: float("inf")
    for kv in filter(None, a.opts.split(",")):
        k, v = kv.split("=")
        _capi.set_option(int(k), int(v))
    w = bench.WORKLOADS["cfg3"]
    levels = bench.build_levels(w)
    u0 = to_device(seeded_field(Grid(w["dim"], w["ns"][0])))[0]
    p, dt = w["p"], w["dt"]
    for i in range(3 + a.steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        pfasst_run(levels, u0, dt * p, p, tol=w["tol"], max_iter=20, streams=not a.no_streams)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"block {i}: host enqueue {1e3 * (t1 - t0):8.1f} ms  device {e0.elapsed_time(e1):8.1f} ms"
              f"  wall {1e3 * (t2 - t0):8.1f} ms", flush=True)


if __name__ == "__main__":
    main()
