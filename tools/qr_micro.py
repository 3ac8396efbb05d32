"""Time rsc_qrcp_batched on a given sketch shape (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402

m, k, cnt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(0)
G0 = [E.to_dev(rng.standard_normal((m, k)) @ np.diag(np.logspace(0, -8, k))) for _ in range(cnt)]
Gs = [g.clone() for g in G0]
Qs = [E.empty(m, k) for _ in range(cnt)]
rank = E.zeros(cnt, dtype=E.I32)
E.ensure_gemm_workspace()


def run():
    for g, g0 in zip(Gs, G0):
        g.copy_(g0)
    return E.qrcp_batched([g.data_ptr() for g in Gs], [m] * cnt, [k] * cnt, [k] * cnt, [q.data_ptr() for q in Qs],
                          [k] * cnt, rank)


w = run()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(3):
    w = run()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 3
print(f"qrcp {cnt} x {m}x{k}: {ms:.2f} ms  ({ms*1e3/k:.1f} us per column)  ranks {sorted(set(rank.cpu().tolist()))}")
