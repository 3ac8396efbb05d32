"""Factorize once, then time N preconditioner applies (CUDA events) and print
algorithmic bytes/s (stored scalars x 8 B x 2 sweeps per apply)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402

cfg, grid, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 10
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
z = E.empty(A.n)
for _ in range(5):
    F.apply_device(r, z)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(reps):
    F.apply_device(r, z)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / reps
byts = 2 * 8 * F.stats.stored_scalars
print(f"apply {ms:.3f} ms  stored {F.stats.stored_scalars}  {byts / ms / 1e6:.1f} GB/s (algorithmic)")
