"""Apply with the diagonal trees' flattened inverses vs the lock-step Alg. 4 waves:
time per application, phases, refresh (explicit inverses) time, agreement.
python tools/apply_treeinv.py CFG [GRID]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402

cfg = int(sys.argv[1])
grid = int(sys.argv[2]) if len(sys.argv) > 2 else GRID[cfg]
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
ref = None
for inv in (False, True):
    DeviceApply.TREE_INV = inv
    ap = DeviceApply(F)
    z = E.empty(A.n)
    for _ in range(5):
        ap(r, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ap(r, z)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    for _ in range(3):  # the third call replays the refresh graph
        ap.refresh_inverses()
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e0.record()
        ap.refresh_inverses()
        e1.record()
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        tr = e0.elapsed_time(e1)
    ap(r, z)
    torch.cuda.synchronize()
    zz = z.cpu().numpy()  # after the graph-replayed refresh
    if ref is None:
        ref = zz
    err = float(np.linalg.norm(zz - ref) / np.linalg.norm(ref))
    byt = 16.0 * F.stats.stored_scalars + 48.0 * A.n
    print(f"tree_inv {int(inv)}: phases {len(ap.launches):5d}  apply {t:.3f} ms  {byt / t / 1e6:.0f} GB/s  "
          f"refresh {tr:.2f} ms (host {1e3 * (h1 - h0):.2f} ms)  rel diff vs waves {err:.2e}", flush=True)
