"""Inclusive device time per factorization section (engine.region timing)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
E.PROFILE = E.KernelProfile()
t0 = time.perf_counter()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tags = E.PROFILE.by_tag()
E.PROFILE = None
print(f"wall {wall:.3f}s (timed run, events add overhead)")
for k, (n, t, fl) in sorted(tags.items(), key=lambda x: -x[1][1]):
    print(f"  {t * 1e3:9.1f} ms  n={n:6d}  {fl / 1e9:9.1f} GF  {fl / max(t, 1e-12) / 1e12:6.2f} TF/s  {k}")
