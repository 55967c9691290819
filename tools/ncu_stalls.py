"""Stall and instruction-mix summary of one kernel in an `ncu --set full
--import-source on` report (the tables DESIGN.md section 9 quotes).

    python tools/ncu_stalls.py gpurun_out/top255_full.ncu-rep [kernel index] [top N]

Prints, for the chosen launch: duration, registers, warp instructions, issue
utilisation, the warp-state stall reasons above 0.3 warp-cycles per issued
instruction, the dynamic opcode mix, and the N SASS instructions that hold
the most stall samples with their dominant reasons."""
import collections
import csv
import subprocess
import sys


def table(rep, page, kid=None):
    cmd = ["ncu", "-i", rep, "--page", page, "--csv"]
    if kid is not None:
        cmd += ["--kernel-id", f":::{kid}"]
    return list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))


def main():
    rep = sys.argv[1]
    which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    top_n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    rows = table(rep, "raw")
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    for n, r in enumerate(rows[2:]):
        print(n, r[idx["Kernel Name"]][:60], r[idx["gpu__time_duration.sum"]], "us  regs",
              r[idx["launch__registers_per_thread"]], " inst", r[idx["smsp__inst_executed.sum"]],
              " issue", r[idx["smsp__issue_active.avg.pct_of_peak_sustained_active"]][:5], "%")
        if n == which:
            for h in hdr:
                if "issue_stalled" in h and "pcsamp" not in h and float(r[idx[h]]) > 0.3:
                    print("     ", h.split("issue_stalled_")[1].split("_per")[0],
                          round(float(r[idx[h]]), 2))
    rows = table(rep, "source", which + 1)
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
    if not starts:
        return
    hdr = rows[starts[0]]
    end = starts[1] - 1 if len(starts) > 1 else len(rows)
    idx = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[starts[0] + 1:end] if len(r) > 10 and r[0].startswith("0x")]
    ex = [int(r[idx["Instructions Executed"]]) for r in data]
    smp = [int(r[idx["# Samples"]]) for r in data]
    ops = collections.Counter()
    for r, e in zip(data, ex):
        w = r[idx["Source"]].split()
        ops[(w[1] if w[0].startswith("@") else w[0]).split(".")[0]] += e
    tot, tsm = sum(ex) or 1, sum(smp) or 1
    print("opcode mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(12)))
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    for i in sorted(sorted(range(len(data)), key=lambda i: -smp[i])[:top_n]):
        r = data[i]
        why = sorted(((h[6:], int(r[idx[h]])) for h in stalls if int(r[idx[h]]) > 0),
                     key=lambda kv: -kv[1])[:2]
        print(f"{i:5d} {100 * smp[i] / tsm:5.1f}%  {r[idx['Source']].strip()[:58]:58s} {why}")


if __name__ == "__main__":
    main()
