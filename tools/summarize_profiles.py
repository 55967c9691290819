"""Summarise gpurun_out/ ncu artefacts into profiles/<round>/ (text, committed).

    python tools/summarize_profiles.py r01
"""
import collections
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")


def launch_list(dst):
    path = os.path.join(OUT, "launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0] != "ID"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = re.sub(r"\(.*", "", r[4]).replace("pl::<unnamed>::", "")
        key = f"{name} grid={r[8]}"
        agg[key][0] += 1
        agg[key][1] += float(r[14]) / 1e3
    tot = sum(v[1] for v in agg.values())
    with open(dst, "w") as fh:
        fh.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none -s 30000 -c 4000\n"
                 f"# python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs (rank streams; {len(rows)} launches, "
                 f"{tot:.1f} us, cold-cache serialised: compare SHARES)\n")
        fh.write(f"{'share':>7s} {'us':>10s} {'n':>5s}  kernel\n")
        for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"{us / tot:7.2%} {us:10.1f} {n:5d}  {k}\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size"]


def full_capture(rep, dst, note):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    with open(dst, "w") as fh:
        fh.write(f"# {note}\n# ncu --set full --clock-control none (report {os.path.basename(rep)})\n")
        for r in rows[2:]:
            fh.write(f"\n{r[idx['Kernel Name']]}\n")
            for w in WANT:
                if w in idx:
                    fh.write(f"  {w:62s} {r[idx[w]]:>14s} {rows[1][idx[w]]}\n")
            try:
                rd = float(r[idx["dram__bytes_read.sum"]])
                wr = float(r[idx["dram__bytes_write.sum"]])
                us = float(r[idx["gpu__time_duration.sum"]])
                unit = rows[1][idx["dram__bytes_read.sum"]]
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}.get(unit, 1)
                tu = rows[1][idx["gpu__time_duration.sum"]]
                tscale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}.get(tu, 1e-6)
                fh.write(f"  => DRAM traffic {(rd + wr) * scale / 1e6:.1f} MB, "
                         f"{(rd + wr) * scale / (us * tscale) / 1e9:.0f} GB/s\n")
            except Exception:
                pass


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    dst = os.path.join(ROOT, "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        launch_list(os.path.join(dst, "launch_list_summary.txt"))
    caps = {"top255_full.ncu-rep": "top kernels at 255^3 (k_zrb3 one-barrier red-black sweep, "
                                   "k_rfw residual+restriction, k_cubic5 cubic correction, "
                                   "k_mid cooperative small levels)",
            "other255_full.ncu-rep": "the other fine-level kernels at 255^3 in kernel_bench's order "
                                     "(restrict_state: k_chain_fw + coarse k_z1 applies; FAS: "
                                     "k_chain_fw_wide + k_chain; then the correction, the residual and "
                                     "one SDC sweep as far as the launch count reaches)",
            "zrb255_full.ncu-rep": "dominant kernel: fused red-black sweep (TMA), 255^3 "
                                   "(first launch: with fused prolongation? see kernel name)",
            "jacobi512.ncu-rep": "round-1 baseline: one-point-per-thread Jacobi sweep, 511^3",
            "zmarch512.ncu-rep": "cp.async z-marching Jacobi sweep, 511^3 (before TMA)",
            "zjac512.ncu-rep": "TMA z-marching Jacobi sweep, 511^3",
            "zrb512.ncu-rep": "TMA fused red-black sweep, 511^3 (before the divergence fix)"}
    for rep, note in caps.items():
        p = os.path.join(OUT, rep)
        if os.path.exists(p):
            full_capture(p, os.path.join(dst, rep.replace(".ncu-rep", ".txt")), note)
    for src, name in (("bench_full.json", "bench.json"),
                      ("bench_nostreams.json", "bench_single_stream.json")):
        b = os.path.join(OUT, src)
        if os.path.exists(b) and os.path.getsize(b):
            json.dump(json.load(open(b)), open(os.path.join(dst, name), "w"), indent=1)


if __name__ == "__main__":
    main()
