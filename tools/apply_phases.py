"""Per-phase device time of one preconditioner apply (CUPTI kernel records of an
eager run) with each phase's matrix bytes: where the apply's time goes."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200.benchsparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
z = E.empty(A.n)
F.apply_device(r, z)
ap = F._apply
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as kp:
    ap._run_program()
    torch.cuda.synchronize()
kev = [e for e in kp.events() if e.device_type.name == "CUDA"]
gem = [e for e in kev if "gemv" in e.name or "trsv" in e.name]
print("phases", len(ap.phases), "kernel records", len(gem), "all", len(kev))
tot_t = sum(e.device_time for e in gem)
rows = []
for ph, e in zip(ap.phases, gem):
    byts = sum(8 * it[1] * it[2] for it in ph.items)
    rows.append((e.device_time, byts, len(ph.items)))
tot_b = sum(b for _, b, _ in rows)
print(f"sum kernel time {tot_t / 1e3:.3f} ms, matrix bytes {tot_b / 1e9:.3f} GB -> {tot_b / tot_t / 1e3:.1f} GB/s")
rows_sorted = sorted(rows, reverse=True)
for t, b, n in rows_sorted[:25]:
    print(f"{t:8.1f} us  {b / 1e6:8.2f} MB  {b / t / 1e3 if t else 0:7.1f} GB/s  problems {n}")
small = [x for x in rows if x[1] < 4e6]
print(f"phases < 4 MB: {len(small)} taking {sum(x[0] for x in small) / 1e3:.3f} ms")
