"""Where one level-phase apply spends its time (CUPTI kernel records, PDL off so
records do not overlap): subtree-task launches, device-descriptor phases, small
phases.  python tools/apply_breakdown.py CFG"""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

os.environ["RSC_APPLY_NO_PDL"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
DeviceApply.FLOW = False
ap = DeviceApply(F)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
z = E.empty(A.n)
ap(r, z)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as kp:
    ap._run_program()
    torch.cuda.synchronize()
kev = [e for e in kp.events() if e.device_type.name == "CUDA"]
tot = sum(e.device_time for e in kev)
by = {}
for e in kev:
    k = e.name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    d = by.setdefault(k, [0, 0.0, []])
    d[0] += 1
    d[1] += e.device_time
    d[2].append(e.device_time)
print(f"kernel records {len(kev)}, sum {tot / 1e3:.3f} ms")
for k, (n, t, ts) in sorted(by.items(), key=lambda kv: -kv[1][1]):
    ts = np.asarray(ts)
    print(f"{k[:60]:60s} n={n:5d} sum={t / 1e3:7.3f} ms  median={np.median(ts):7.1f} us  max={ts.max():8.1f} us")
# the per-phase sizes of the level phases (bytes of matrix)
sizes = np.array([sum(8 * it[1] * it[2] for it in ph.items) for ph in ap.phases])
print("level phases", len(sizes), "bytes", sizes.sum() / 1e9, "GB; phases > 64 MB:", int((sizes > 64e6).sum()),
      "holding", sizes[sizes > 64e6].sum() / 1e9, "GB")
tb = sum(8 * it[1] * it[2] for bw, lst in ap.tasks.items() for _, ph in lst for it in ph.items)
print("subtree tasks bytes", tb / 1e9, "GB (both sweeps)")
# records in launch order: forward tasks, the phases (one launch each when device
# descriptors, else ceil(items / 224)), backward tasks
recs = [e.device_time for e in kev]
k = 1 if ap.task_dev.get(False) is not None else 0
print("forward tasks %.1f us" % recs[0] if k else "no forward tasks")
rowsz = []
for li, ph in enumerate(ap.phases):
    n = len(ph.items)
    nl = 1 if li in ap.dev else max(1, -(-n // 224))
    t = sum(recs[k:k + nl])
    k += nl
    b = sum(8 * it[1] * it[2] * (0.5 if it[8] & 6 and it[1] == it[2] else 1.0) for it in ph.items)
    rowsz.append((t, b, n))
print("backward tasks %.1f us" % recs[k] if k < len(recs) else "no backward tasks")
rowsz = np.array(rowsz)
for lo, hi in [(0, 1e6), (1e6, 4e6), (4e6, 16e6), (16e6, 64e6), (64e6, 1e12)]:
    m = (rowsz[:, 1] >= lo) & (rowsz[:, 1] < hi)
    if m.any():
        print(f"phases {lo / 1e6:6.0f}-{hi / 1e6:6.0f} MB: {m.sum():4d}  {rowsz[m, 0].sum() / 1e3:7.3f} ms  "
              f"{rowsz[m, 1].sum() / max(rowsz[m, 0].sum(), 1e-9) / 1e3:7.0f} GB/s (triangles at half)")
