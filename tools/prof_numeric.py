"""cProfile of one eager numeric pass (prepared plan, no graph): the host cost of
the one-shot factorize's sweep.  python tools/prof_numeric.py CFG"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
import paper_1507_05593_b200.factor as FM  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402
import torch  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
t = time.perf_counter()
prep = prepare(A, SolverConfig(**KNOBS), coords)
print(f"prepare {time.perf_counter() - t:.2f}s")
FM.GRAPH_REFACTOR = False
F = factorize(A, prepared=prep)
del F
torch.cuda.synchronize()
t = time.perf_counter()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
print(f"eager numeric (no profiler) {time.perf_counter() - t:.3f}s  phases {F.stats.phase_times}")
del F
pr = cProfile.Profile()
pr.enable()
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(40)
st.sort_stats("cumulative").print_stats(40)
