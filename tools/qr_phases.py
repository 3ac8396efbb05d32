"""RSC_QR_TIMING=1: clock64 cycles per phase of the cluster QRCP (CTA 0, matrix 0)."""
import ctypes
import os
import subprocess
import sys

os.environ["RSC_QR_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_05593_b200 import _lib  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402

m, k, cnt = (int(x) for x in sys.argv[1:4])
lib = _lib.load()
rng = np.random.default_rng(0)
Gs = [E.to_dev(rng.standard_normal((m, k)) @ np.diag(np.logspace(0, -8, k))) for _ in range(cnt)]
Qs = [E.empty(m, k) for _ in range(cnt)]
rank = E.zeros(cnt, dtype=E.I32)
buf = (ctypes.c_ulonglong * 32)()
E.qrcp_batched([g.data_ptr() for g in Gs], [m] * cnt, [k] * cnt, [k] * cnt, [q.data_ptr() for q in Qs], [k] * cnt, rank)
torch.cuda.synchronize()
lib.rsc_qr_phase_cycles(buf, 1)
Gs = [E.to_dev(rng.standard_normal((m, k)) @ np.diag(np.logspace(0, -8, k))) for _ in range(cnt)]
E.qrcp_batched([g.data_ptr() for g in Gs], [m] * cnt, [k] * cnt, [k] * cnt, [q.data_ptr() for q in Qs], [k] * cnt, rank)
torch.cuda.synchronize()
lib.rsc_qr_phase_cycles(buf, 1)
steps = min(m, k)
names = ["pivot", "reflector", "barrier1", "update", "barrier2"]
tot = sum(buf[i] for i in range(5))
for i, nm in enumerate(names):
    print(f"{nm:10s} {buf[i] / steps:9.0f} cycles/step  {100 * buf[i] / max(tot, 1):5.1f}%")
print(f"total      {tot / steps:9.0f} cycles/step")
print("per-warp update cycles/step, CTA 0:", [int(buf[8 + w] / steps) for w in range(8)])
print("per-warp update cycles/step, CTA 1:", [int(buf[16 + w] / steps) for w in range(8)])
