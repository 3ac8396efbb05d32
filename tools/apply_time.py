"""Apply (preconditioner) time vs the subtree-task size threshold, with a check
against the all-phases program.  python tools/apply_time.py CFG [MB ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402

cfg = int(sys.argv[1])
mbs = [float(x) for x in sys.argv[2:]] or [0.0, 0.5, 1, 2, 4, 8]
A, coords = _problem(cfg, GRID[cfg])
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
ref = None
for mb in mbs:
    DeviceApply.TASK_BYTES = int(mb * (1 << 20))
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
    zz = z.cpu().numpy()
    if ref is None:
        ref = zz
    err = float(np.abs(zz - ref).max() / np.abs(ref).max())
    byt = 16.0 * F.stats.stored_scalars + 48.0 * A.n
    print(f"task_mb {mb:5.2f}: tasks {ap.n_tasks:6d} phases {len(ap.launches):5d}  apply {t:.3f} ms  "
          f"{byt / t / 1e6:.0f} GB/s  maxrel vs first {err:.2e}", flush=True)
