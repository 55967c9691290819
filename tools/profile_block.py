"""Per-kernel-kind, per-level time breakdown of one PFASST block (CUDA events
around every launch).  python tools/profile_block.py [workload]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_1407_6486_b200 import _capi  # noqa: E402
from paper_1407_6486_b200._device import to_device  # noqa: E402
from paper_1407_6486_b200.heat import Grid, seeded_field  # noqa: E402
from paper_1407_6486_b200.pfasst import pfasst_run  # noqa: E402

w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]
levels = bench.build_levels(w)
u0 = to_device(seeded_field(Grid(w["dim"], w["ns"][0])))[0]
run = lambda: pfasst_run(levels, u0, w["dt"] * w["p"], w["p"], tol=w["tol"], max_iter=20)
run()
torch.cuda.synchronize()
names = _capi.kind_names()
_capi.timing_enable(names)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1)
rows = []
for n in names:
    for b, (c, t) in _capi.timing_by_size(n).items():
        rows.append((t, n, b, c))
_capi.timing_enable(None)
rows.sort(reverse=True)
acc = 0.0
print(f"block {total:.1f} ms (timed launches sum {sum(r[0] for r in rows):.1f} ms)")
print(f"{'kind':14s} {'MB/launch':>10s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s} {'GB/s':>8s}")
for t, n, b, c in rows[:40]:
    acc += t
    print(f"{n:14s} {b/1e6:10.2f} {c:8d} {t:9.2f} {t/total:6.1%} {1e3*t/c:8.1f} {b/(t/c/1e3)/1e9:8.1f}")
