"""Bandwidth of the apply's batched GEMV kernel on representative shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import _lib  # noqa: E402
from paper_1507_05593_b200._lib import int_array, ptr_array  # noqa: E402

lib = _lib.load()


def run(shapes, mode, reps=20):
    Ms = [torch.randn(r, c, dtype=torch.float64, device="cuda") for r, c in shapes]
    xs = [torch.randn(r if mode & 1 else c, dtype=torch.float64, device="cuda") for r, c in shapes]
    ys = [torch.zeros(c if mode & 1 else r, dtype=torch.float64, device="cuda") for r, c in shapes]
    n = len(shapes)
    arrs = [ptr_array([m.data_ptr() for m in Ms]), int_array([s[0] for s in shapes]), int_array([s[1] for s in shapes]),
            int_array([s[1] for s in shapes]), ptr_array([x.data_ptr() for x in xs]), ptr_array([0] * n),
            ptr_array([y.data_ptr() for y in ys]), ptr_array([0] * n)]
    args = [n] + [a.ctypes.data for a in arrs] + [mode, 1.0, torch.cuda.current_stream().cuda_stream]
    lib.rsc_gemv_batched(*args)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        lib.rsc_gemv_batched(*args)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    byts = sum(8 * r * c for r, c in shapes)
    return ms, byts / ms / 1e6


for name, shapes in (("1 x 20000x64", [(20000, 64)]), ("1 x 4096x4096", [(4096, 4096)]),
                     ("500 x 2000x60", [(2000, 60)] * 500), ("100 x 8000x200", [(8000, 200)] * 100),
                     ("2000 x 300x40", [(300, 40)] * 2000)):
    for mode in (0, 1):
        ms, gbs = run(shapes, mode)
        print(f"{name:16s} mode {mode}: {ms*1e3:8.1f} us  {gbs:7.1f} GB/s")
