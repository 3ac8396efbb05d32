"""Debug helper: GPU factor + apply + short PCG vs the oracle on a mid-size grid."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import numeric as on  # noqa: E402
from paper_1507_05593_b200.benchsparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
torch.cuda.synchronize()
r = np.random.default_rng(1).standard_normal(A.n)
z = F.apply(r)
b = np.random.default_rng(0).standard_normal(A.n)
t0 = time.perf_counter()
x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6, max_iter=30)
print("gpu pcg its", rep.iterations, "relres", rep.relative_residual, "t", time.perf_counter() - t0, flush=True)
if A.n <= 40000:
    Fo = on.factorize(A, on.Config(**KNOBS), coords=coords)
    zo = Fo.apply(r)
    print("apply relerr vs oracle", np.linalg.norm(z - zo) / np.linalg.norm(zo))
    print("ranks equal", sorted(F.ranks.items()) == sorted(Fo.ranks.items()))
    xo, repo = on.pcg(A, b, Fo, tol=1e-6)
    print("oracle its", repo.iterations, "x relerr", np.linalg.norm(x - xo) / np.linalg.norm(xo))
