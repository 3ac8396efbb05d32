"""Step-to-step variance of factorize + device PCG on one config: device time of
each part (CUDA events) and host time, with/without the cyclic GC frozen."""
import gc
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402
from paper_1507_05593_b200.pcg import pcg_solve_device  # noqa: E402

cfg = int(sys.argv[1])
freeze = len(sys.argv) > 2 and sys.argv[2] == "freeze"
A, coords = _problem(cfg, GRID[cfg])
prep = prepare(A, SolverConfig(**KNOBS), coords)
bd = E.to_dev(np.random.default_rng(0).standard_normal(A.n))
A.device_csr()
if freeze:
    gc.collect()
    gc.freeze()
gcs = []
gc.callbacks.append(lambda phase, info: gcs.append((phase, info["generation"], time.perf_counter())))
F = None


class step_var_prev:
    ap = None


for it in range(8):
    F = None
    torch.cuda.synchronize()
    n0 = len(gcs)
    t0 = time.perf_counter()
    F = factorize(A, prepared=prep)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ap = getattr(F, "_apply", None)
    same = ap is not None and ap is getattr(step_var_prev, "ap", None)
    step_var_prev.ap = ap
    t4 = time.perf_counter()
    F.apply_device(bd, x)  # one more apply, timed on the host (graph replay or re-capture)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    g = gcs[n0:]
    gen2 = sum(1 for p, gen, _ in g if p == "start" and gen == 2)
    gct = sum(b[2] - a[2] for a, b in zip(g[::2], g[1::2]))
    print(f"{'freeze' if freeze else 'gc'} step {it}: factorize host {t1 - t0:.3f} +sync {t2 - t1:.3f}  pcg {t3 - t2:.3f} "
          f"({rep.iterations} its; program {'reused' if same else 'new'}, next apply {1e3 * (t5 - t4):.1f} ms, "
          f"pcg phases {getattr(rep, 'wall_times', None)})  gc runs {len(g) // 2} (gen2 {gen2}) {gct:.3f}s", flush=True)
