"""Duration distribution of one kernel's launches in one factorization (CUPTI)."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid, pat = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
d = np.array([e.device_time for e in prof.events() if e.device_type.name == "CUDA" and pat in e.name])
d.sort()
print(f"{pat}: {d.size} launches, total {d.sum() / 1e3:.1f} ms, median {np.median(d):.1f} us")
for q in (0.5, 0.9, 0.99, 1.0):
    print(f"  q{q}: {d[min(int(q * d.size), d.size - 1)]:.1f} us")
c = np.cumsum(d[::-1])
for k in (10, 100, 1000):
    print(f"  top {k}: {c[min(k, d.size) - 1] / 1e3:.1f} ms")
