"""Wall time of consecutive PFASST blocks of a bench workload (default
BASELINE config 3), with the SM clock, board power and throttle reasons after
each: the steady-state block time next to bench.py's average.

    python tools/block_times.py [--workload cfg3] [--blocks 12] [--no-streams]"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1407_6486_b200._device import to_device  # noqa: E402
from paper_1407_6486_b200.pfasst import pfasst_run  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--blocks", type=int, default=12)
    ap.add_argument("--no-streams", action="store_true")
    a = ap.parse_args()
    w = bench.WORKLOADS[a.workload]
    levels = bench.build_levels(w)
    u0 = to_device(bench.initial_field(w))[0]
    p, dt = w["p"], w["dt"]
    q = "clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active"
    for i in range(a.blocks):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pfasst_run(levels, u0, dt * p, p, tol=w["tol"], max_iter=20, streams=not a.no_streams)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        smi = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"],
                             capture_output=True, text=True).stdout.strip()
        print(f"block {i}: {ms:8.1f} ms  {p / ms * 1e3:6.2f} time-steps/s   {smi}", flush=True)


if __name__ == "__main__":
    main()
