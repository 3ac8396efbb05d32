"""cProfile of one graph-replayed factorize() (host work around the replay)."""
import cProfile
import os
import pstats
import sys

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
F = None
for _ in range(3):
    F = None
    F = factorize(A, prepared=prep)
    x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
torch.cuda.synchronize()
F = None
pr = cProfile.Profile()
pr.enable()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
