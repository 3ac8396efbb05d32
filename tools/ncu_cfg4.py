"""ncu driver for the sparse configs: the profiled region (cudaProfilerStart/Stop,
run ncu with --profile-from-start off) is one piece of a factor+PCG step.

    python tools/ncu_cfg4.py apply   [cfg]   one preconditioner apply + one SpMV + 2 PCG iterations
    python tools/ncu_cfg4.py numeric [cfg]   one eager numeric factorization (prepared plan)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
import paper_1507_05593_b200.factor as FM  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve_device  # noqa: E402

mode = sys.argv[1]
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
A, coords = _problem(cfg, GRID[cfg])
conf = SolverConfig(**KNOBS)
prep = prepare(A, conf, coords)
FM.GRAPH_REFACTOR = False  # every pass eager: the launches ncu sees are the sweep's own
F = factorize(A, prepared=prep)
b = E.to_dev(np.random.default_rng(0).standard_normal(A.n))
z = E.empty(A.n)
y = E.empty(A.n)
S = A.device_csr()
for _ in range(3):
    F.apply_device(b, z)
torch.cuda.synchronize()
if mode == "apply":
    F._apply.graph = None
    F._apply.calls = -10**9  # stay eager (the graph replay would hide the launches from -k filters)
    torch.cuda.profiler.start()
    F.apply_device(b, z)
    E.spmv(S, b, y)
    pcg_solve_device(A, b, preconditioner=F, tol=1e-6, max_iter=2)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
elif mode == "numeric":
    F = None
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("ok", mode, cfg, F.stats.stored_scalars)
