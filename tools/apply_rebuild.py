"""Cost of (re)building the preconditioner-apply program for a new factor (what a
refactorization pays when its kept ranks differ from the cached program's)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.benchsparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
prep = prepare(A, SolverConfig(**KNOBS), coords)
F = factorize(A, prepared=prep)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
for rep in range(2):
    torch.cuda.synchronize()
    pr = cProfile.Profile() if rep == 1 else None
    t0 = time.perf_counter()
    if pr:
        pr.enable()
    ap = DeviceApply(F)
    torch.cuda.synchronize()
    if pr:
        pr.disable()
    t1 = time.perf_counter()
    ts = []
    for i in range(ap.GRAPH_AFTER + 3):
        a = time.perf_counter()
        ap(r)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - a)
    print(f"build {t1 - t0:.3f}s  applies " + " ".join(f"{x * 1e3:.1f}" for x in ts) + " ms", flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
