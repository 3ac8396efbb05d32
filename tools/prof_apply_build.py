"""cProfile of building the apply program (DeviceApply) of a config's factor: the
first-PCG host cost of the one-shot API.  python tools/prof_apply_build.py CFG"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
import torch  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
torch.cuda.synchronize()
t = time.perf_counter()
ap = DeviceApply(F)
torch.cuda.synchronize()
print(f"DeviceApply build {time.perf_counter() - t:.3f}s phases {len(ap.phases)}")
pr = cProfile.Profile()
pr.enable()
ap = DeviceApply(F)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
