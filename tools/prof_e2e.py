"""cProfile of the one-shot public API (factorize + pcg_solve) on a sparse config."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
b = np.random.default_rng(0).standard_normal(A.n)
import torch  # noqa: E402

F = factorize(A, SolverConfig(**KNOBS), coords=coords)  # warm (kernel attributes, allocator)
x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6)
del F
torch.cuda.synchronize()
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
t1 = time.perf_counter()
x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6)
pr.disable()
t2 = time.perf_counter()
print(f"factorize {t1 - t:.2f}s  pcg {t2 - t1:.2f}s  phases {F.stats.phase_times}")
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
st.sort_stats("cumulative").print_stats(40)
