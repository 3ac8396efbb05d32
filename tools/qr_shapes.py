"""Shape census + synchronous timing of the batched QRCP calls of one numeric pass."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05593_b200.engine as E  # noqa: E402
import paper_1507_05593_b200.factor as FM  # noqa: E402
import paper_1507_05593_b200.numeric as NM  # noqa: E402
from bench_sparse import KNOBS, _problem  # noqa: E402
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
    if os.environ.get("QR_COND"):
        for gp, mm, kk, ll in zip(Gp, m, k, ldg):
            if mm * kk >= 64 * 64:
                t = _dev_view(int(gp), int(mm), int(kk), int(ll))
                sv = torch.linalg.svdvals(t)
                conds.append((int(mm), int(kk), float(sv[0] / sv[-1])))
    r = orig(Gp, m, k, ldg, Qp, ldq, rank, alloc)
    e.record()
    torch.cuda.synchronize()
    log.append((np.asarray(m), np.asarray(k), s.elapsed_time(e)))
    return r


conds = []


class _CAI:
    def __init__(self, ptr, shape, strides):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False),
                                         "strides": strides, "version": 3}


def _dev_view(ptr, m, k, ld):
    return torch.as_tensor(_CAI(ptr, (m, k), (8 * ld, 8)), device="cuda").clone()


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
    o = np.argsort(-(m.astype(np.int64) * k * k))[:6]
    print("      largest (m,k):", " ".join(f"({int(m[x])},{int(k[x])})" for x in o))

if conds:
    c = np.array([x[2] for x in conds])
    sz = np.array([x[0] * x[1] for x in conds], dtype=float)
    for lim in (1e4, 1e6, 1e8, 1e10, 1e12):
        print(f"  cond <= {lim:.0e}: {int((c <= lim).sum())} of {c.size} sketches, {100 * sz[c <= lim].sum() / sz.sum():.0f}% of entries")
