"""Wall-clock breakdown of factorize + pcg on one config (host vs device)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
t0 = time.perf_counter()
prep = prepare(A, SolverConfig(**KNOBS), coords)
t1 = time.perf_counter()
print(f"n={A.n} prepare {t1 - t0:.2f}s (ordering {prep[0].t_ordering:.2f} symbolic {prep[0].t_symbolic:.2f})")
b = np.random.default_rng(0).standard_normal(A.n)
for it in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6)
    t2 = time.perf_counter()
    print(f"numeric {t1 - t0:.3f}s pcg {t2 - t1:.3f}s its {rep.iterations} relres {rep.relative_residual:.2e} "
          f"work {F.stats.model_gflop:.1f} GF launches {F.stats.gpu_launches} ranks {len(F.ranks)} "
          f"restarts {F.stats.restarts} stored {F.stats.stored_scalars}")
pr = cProfile.Profile()
pr.enable()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
