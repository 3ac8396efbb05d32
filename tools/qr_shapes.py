"""Shape census + synchronous timing of the batched QRCP calls of one numeric pass."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05593_b200.engine as E  # noqa: E402
import paper_1507_05593_b200.factor as FM  # noqa: E402
import paper_1507_05593_b200.numeric as NM  # noqa: E402
from paper_1507_05593_b200.benchsparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
FM.GRAPH_REFACTOR = False
F = factorize(A, prepared=prep)
log = []
orig = E.qrcp_batched


def logged(Gp, m, k, ldg, Qp, ldq, rank, alloc=None):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = orig(Gp, m, k, ldg, Qp, ldq, rank, alloc)
    e.record()
    torch.cuda.synchronize()
    log.append((np.asarray(m), np.asarray(k), s.elapsed_time(e)))
    return r


NM.E.qrcp_batched = logged
F = None
F = factorize(A, prepared=prep)
tot = sum(l[2] for l in log)
print(f"QR calls {len(log)}  total {tot:.1f} ms")
for m, k, ms in sorted(log, key=lambda x: -x[2])[:15]:
    reg = ((m <= 256) & (k <= 64)).sum()
    sm = ((~((m <= 256) & (k <= 64))) & ((m | 1) * k * 8 + 40 * k <= 220 * 1024)).sum()
    big = len(m) - reg - sm
    print(f"  {ms:7.2f} ms  n={len(m):4d} (reg {reg}, smem {sm}, coop {big})  max m {m.max()} max k {k.max()}  "
          f"median m {int(np.median(m))} k {int(np.median(k))}")
