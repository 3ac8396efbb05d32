"""GPU busy fraction of one factorization (torch.profiler / CUPTI kernel activity)."""
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    t0 = time.perf_counter()
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
busy = sum(e.device_time for e in ev) / 1e6 if ev else 0.0
byname = {}
for e in ev:
    k = e.name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "").split("(")[0][:60]
    byname[k] = byname.get(k, 0.0) + e.device_time / 1e3
print(f"wall {wall:.3f}s  kernel-sum {busy:.3f}s  ({100 * busy / wall:.0f}% busy)  kernels {len(ev)}")
for k, v in sorted(byname.items(), key=lambda x: -x[1])[:20]:
    print(f"  {v:9.1f} ms  {k}")
