"""cProfile of prepare() (ordering + symbolic + plan) on a sparse config."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
t = time.perf_counter()
A, coords = _problem(cfg, grid)
print(f"generator {time.perf_counter() - t:.2f}s")
import torch  # noqa: E402
torch.zeros(1, device="cuda")
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
prep = prepare(A, SolverConfig(**KNOBS), coords)
pr.disable()
print(f"prepare {time.perf_counter() - t:.2f}s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
