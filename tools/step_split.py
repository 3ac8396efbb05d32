"""Split of one bench step (sparse config): graph-replayed factorization, apply
program refresh, PCG loop -- CUDA events + host timers, after warm-up."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.benchsparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve_device  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
bd = E.to_dev(np.random.default_rng(0).standard_normal(A.n))
A.device_csr()
F = None
for _ in range(3):
    F = None
    F = factorize(A, prepared=prep)
    x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
torch.cuda.synchronize()
for _ in range(2):
    F = None
    t0 = time.perf_counter()
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    z = E.empty(A.n)
    F.apply_device(bd, z)  # first apply: program refresh
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    F.apply_device(bd, z)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"factorize {t1 - t0:.3f}s (numeric phase {F.stats.phase_times['numeric']:.3f}) first apply {t2 - t1:.4f}s "
          f"apply {t3 - t2:.4f}s pcg {t4 - t3:.3f}s its {rep.iterations}")
