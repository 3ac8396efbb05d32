"""config[1] L_O^T X product: split-K sweep (CUDA events)."""
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
for sk in (1, 2, 4, 8, 16):
    f = lambda: E.gemm_strided_batched(LO, Om, G, transA=True, splitk=sk)
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    print(f"splitk {sk:2d}: {ms:.3f} ms  {2.0*nb*2048*256*58/ms/1e9:.1f} TF/s")
