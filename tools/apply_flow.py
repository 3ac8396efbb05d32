"""Preconditioner apply: the dataflow program (one persistent launch) vs the level
phases + subtree tasks, CUDA-event times and the max difference of the results.
python tools/apply_flow.py CFG [GRID]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
import time  # noqa: E402

cfg = int(sys.argv[1])
grid = int(sys.argv[2]) if len(sys.argv) > 2 else GRID[cfg]
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
byt = 16.0 * F.stats.stored_scalars + 48.0 * A.n
out = {}
for flow in (False, True, False, True):
    DeviceApply.FLOW = flow
    t0 = time.perf_counter()
    ap = DeviceApply(F)
    tb = time.perf_counter() - t0
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
    out[flow] = z.cpu().numpy()
    extra = (f"ops {ap.flow_nops} items {ap.flow_items} edges {ap.flow_edges}" if flow else
             f"phases {len(ap.launches)} tasks {ap.n_tasks}")
    print(f"flow={flow!s:5}: apply {t:.3f} ms = {byt / t / 1e6:.0f} GB/s  build {tb:.2f} s  {extra}", flush=True)
d = np.abs(out[True] - out[False]).max() / np.abs(out[False]).max()
print(f"max |flow - phases| / max|z| = {d:.2e}")
