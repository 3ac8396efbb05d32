"""Microbenchmark of the grouped DMMA GEMM on the config[1] shapes (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402

nb = 512
LO = torch.randn(nb, 2048, 256, dtype=torch.float64, device="cuda")
Om = torch.randn(nb, 2048, 58, dtype=torch.float64, device="cuda")
G = torch.empty(nb, 256, 58, dtype=torch.float64, device="cuda")
H = torch.empty(nb, 2048, 58, dtype=torch.float64, device="cuda")
X = torch.randn(nb, 2048, 192, dtype=torch.float64, device="cuda")
Lt = torch.randn(nb, 64, 192, dtype=torch.float64, device="cuda")
Y = torch.randn(nb, 2048, 64, dtype=torch.float64, device="cuda")


def t(fn, flops, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return ms, flops / ms / 1e9


lib = os.environ.get("RSC_B200_LIB", "default")
r1 = t(lambda: E.gemm_strided_batched(LO, Om, G, transA=True, splitk=8), 2.0 * nb * 2048 * 256 * 58)
r2 = t(lambda: E.gemm_strided_batched(LO, G, H), 2.0 * nb * 2048 * 256 * 58)
r3 = t(lambda: E.gemm_strided_batched(X, Lt, Y, transB=True, alpha=-1.0, beta=1.0), 2.0 * nb * 2048 * 64 * 192)
big = torch.randn(4096, 4096, dtype=torch.float64, device="cuda")
C = torch.empty(4096, 4096, dtype=torch.float64, device="cuda")
r4 = t(lambda: E.gemm(big, big, C), 2.0 * 4096**3, reps=3)
print(f"{lib}: LOtOm {r1[0]:.3f}ms {r1[1]:.1f}TF | LO_G {r2[0]:.3f}ms {r2[1]:.1f}TF | "
      f"trsm-like {r3[0]:.3f}ms {r3[1]:.1f}TF | 4096^3 {r4[0]:.3f}ms {r4[1]:.1f}TF")
