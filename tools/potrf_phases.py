"""RSC_POTRF_TIMING=1: clock64 cycles per phase of the fused POTRF (CTA 0)."""
import ctypes
import os
import sys

os.environ["RSC_POTRF_TIMING"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1507_05593_b200 import _lib  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402

n, cnt = int(sys.argv[1]), int(sys.argv[2])
lib = _lib.load()
rng = np.random.default_rng(0)
G = rng.standard_normal((n, n))
S = G @ G.T / n + np.eye(n)
As = [E.to_dev(S) for _ in range(cnt)]
Ds = [E.empty(n, 64) for _ in range(cnt)]
info = E.zeros(cnt, dtype=E.I32)
buf = (ctypes.c_ulonglong * 8)()
for it in range(2):
    for a in As:
        a.copy_(torch.from_numpy(S))
    torch.cuda.synchronize()
    lib.rsc_potrf_phase_cycles(buf, 1)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    E.potrf_batched([a.data_ptr() for a in As], [n] * cnt, [n] * cnt, [d.data_ptr() for d in Ds], info)
    e.record()
    torch.cuda.synchronize()
lib.rsc_potrf_phase_cycles(buf, 1)
names = {7: "loop top->1", 0: "update (1)", 1: "diag (2)", 2: "out+clean", 3: "unused"}
tot = sum(buf[i] for i in (7, 0, 1, 2))
print(f"n={n} x{cnt}: {s.elapsed_time(e):.3f} ms; CTA0 cycles {tot}")
for i in (0, 1, 2, 7):
    print(f"  {names[i]:12s} {buf[i]:10d} cycles {100 * buf[i] / max(tot, 1):5.1f}%")
