"""One numeric factorization (+ one preconditioner apply) of a sparse config, for
ncu launch lists: the symbolic plan is prepared first, then factorize runs once."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
torch.cuda.synchronize()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
z = F.apply(np.ones(A.n))
torch.cuda.synchronize()
print("ok", F.stats.gpu_launches)
