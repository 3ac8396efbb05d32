"""Grouped GEMM on the large config[4] sweep shapes (the 1e10+ flop launches run at
~18 TF/s in the shape census): transpose / atomic / gather effects, vs cuBLAS."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_sparse_micro import bench  # noqa: E402

for (n, M, N, K) in ((2, 1016, 1016, 6342), (8, 1016, 513, 6337), (4, 684, 338, 3171), (16, 256, 256, 2048)):
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    B = torch.randn(K, N, dtype=torch.float64, device="cuda")
    torch.matmul(A, B)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        for _ in range(n):
            torch.matmul(A, B)
    e.record()
    torch.cuda.synchronize()
    cub = 2.0 * n * M * N * K / (s.elapsed_time(e) / 5) / 1e9
    for ta in (False, True):
        base = bench(n, M, N, K, ta, reps=5)
        at = bench(n, M, N, K, ta, atomic=True, reps=5)
        ga = bench(n, M, N, K, ta, atomic=True, gather=True, reps=5)
        print(f"{n}x M{M} N{N} K{K} TA={int(ta)}: plain {base:5.1f}  atomic {at:5.1f}  atomic+gather {ga:5.1f}  "
              f"cuBLAS(serial) {cub:5.1f} TF/s", flush=True)
