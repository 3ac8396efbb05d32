"""Time config[1]'s four sketch products with the library named by RSC_B200_LIB."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402

nb, n, m, r = 512, 256, 2048, 58
LO = torch.randn(nb, m, n, dtype=torch.float64, device="cuda")
Om = torch.randn(nb, m, r, dtype=torch.float64, device="cuda")
G = torch.empty(nb, n, r, dtype=torch.float64, device="cuda")
H = torch.empty(nb, m, r, dtype=torch.float64, device="cuda")
sk = max(1, min(m // 256, 16))
ops = [("LOt_Om", lambda: E.gemm_strided_batched(LO, Om, G, transA=True, splitk=sk)),
       ("LO_G", lambda: E.gemm_strided_batched(LO, G, H))]
res = []
for name, fn in ops:
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    res.append(f"{name} {ms:.3f} ms {2.0 * nb * m * n * r / ms / 1e9:.2f} TF/s")
print(os.path.basename(os.environ.get("RSC_B200_LIB", "default")), " | ".join(res))
