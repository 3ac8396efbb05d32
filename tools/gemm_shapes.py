"""Shape census of the grouped GEMM launches of one numeric pass (eager)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05593_b200.engine as E  # noqa: E402
import paper_1507_05593_b200.factor as FM  # noqa: E402
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
prep = prepare(A, SolverConfig(**KNOBS), coords)
FM.GRAPH_REFACTOR = False
F = factorize(A, prepared=prep)
log = []
orig = E.gemm_grouped


def logged(probs, transA=False, transB=False):
    p = np.ascontiguousarray(probs, dtype=E.GEMM_DTYPE)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = orig(probs, transA, transB)
    e.record()
    torch.cuda.synchronize()
    log.append((p.copy(), transA, transB, s.elapsed_time(e) * 1e-3))
    return r


E.gemm_grouped = logged
import paper_1507_05593_b200.numeric as NM  # noqa: E402
NM.E.gemm_grouped = logged
F = None
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
M = np.concatenate([l[0]["M"] for l in log]).astype(float)
N = np.concatenate([l[0]["N"] for l in log]).astype(float)
K = np.concatenate([l[0]["K"] for l in log]).astype(float)
B = np.concatenate([l[0]["batch"] for l in log]).astype(float)
at = np.concatenate([l[0]["atomic"] for l in log])
fl = 2 * M * N * K * B
tiles = np.ceil(M / 64) * np.ceil(N / 64) * B
padded = tiles * 64 * 64 * np.ceil(K / 16) * 16 * 2
print(f"launch groups {len(log)}  problems {M.size}  flops {fl.sum()/1e9:.1f} GF  padded-DMMA work {padded.sum()/1e9:.1f} GF "
      f"(useful {100*fl.sum()/padded.sum():.0f}%)  atomic share of flops {100*fl[at==1].sum()/fl.sum():.0f}%")
for name, v in (("M", M), ("N", N), ("K", K)):
    w = np.average(v, weights=fl)
    print(f"  flop-weighted mean {name} = {w:.0f};  pct of flops with {name}<64: {100*fl[v<64].sum()/fl.sum():.0f}%")
edges = [0, 1e5, 1e6, 1e7, 1e8, 1e12]
h = np.histogram(fl, bins=edges, weights=fl)[0]
print("  flops by problem size (flop):", {f"<{e:.0e}": f"{100*x/fl.sum():.0f}%" for e, x in zip(edges[1:], h)})
per = [(l[0].size, float((2*l[0]["M"].astype(float)*l[0]["N"]*l[0]["K"]*l[0]["batch"]).sum()),
        float((np.ceil(l[0]["M"]/64)*np.ceil(l[0]["N"]/64)*l[0]["batch"]).sum()), l[1], l[2]) for l in log]
ctas = np.array([p[2] for p in per])
print(f"  CTAs per launch: median {np.median(ctas):.0f}, launches with < 148 CTAs: {(ctas<148).sum()} of {len(ctas)}, "
      f"their flops {100*sum(p[1] for p in per if p[2]<148)/fl.sum():.0f}%")

tm = np.array([l[3] for l in log])
fls = np.array([p[1] for p in per])
print(f"  sum of per-call GEMM time {tm.sum()*1e3:.1f} ms -> {fls.sum()/tm.sum()/1e12:.2f} TF/s")
for lo, hi in ((0, 1e8), (1e8, 1e9), (1e9, 1e10), (1e10, 1e13)):
    sel = (fls >= lo) & (fls < hi)
    if sel.any():
        print(f"  calls with {lo:.0e}..{hi:.0e} flop: {sel.sum():4d} calls, {tm[sel].sum()*1e3:7.1f} ms, "
              f"{fls[sel].sum()/1e9:7.1f} GF, {fls[sel].sum()/max(tm[sel].sum(),1e-9)/1e12:5.2f} TF/s")
for ta, tb in ((False, False), (True, False), (False, True)):
    sel = np.array([(l[1] == ta and l[2] == tb) for l in log])
    if sel.any():
        print(f"  TA={ta:d} TB={tb:d}: {sel.sum()} calls {tm[sel].sum()*1e3:.1f} ms {fls[sel].sum()/1e9:.1f} GF "
              f"{fls[sel].sum()/tm[sel].sum()/1e12:.2f} TF/s")
# load balance: a launch cannot finish before its longest CTA (its largest K, in
# 16-wide k-steps) nor before total tile-steps / (740 concurrent CTAs)
lb_sum, ideal_sum = 0.0, 0.0
for l in log:
    p = l[0]
    tiles = (np.ceil(p["M"] / 64) * np.ceil(p["N"] / 64) * p["batch"]).astype(float)
    ksteps = np.ceil(p["K"] / 16).astype(float)
    total = float((tiles * ksteps).sum())
    lb = max(total / 740.0, float(ksteps.max()))
    lb_sum += lb
    ideal_sum += total / 740.0
print(f"  launch-time lower bound from the longest CTA vs perfect balance: {lb_sum:.0f} vs {ideal_sum:.0f} "
      f"k-step units ({lb_sum/ideal_sum:.2f}x)")
rows = []
for l in log:
    p = l[0]
    tiles = (np.ceil(p["M"] / 64) * np.ceil(p["N"] / 64) * p["batch"]).astype(float)
    ksteps = np.ceil(p["K"] / 16).astype(float)
    total = float((tiles * ksteps).sum())
    lb = max(total / 740.0, float(ksteps.max()))
    i = int(np.argmax(ksteps))
    rows.append((lb - total / 740.0, len(p), int(p["M"][i]), int(p["N"][i]), int(p["K"][i]), int(p["atomic"][i]),
                 float(p["beta"][i]), l[1], l[2], total / 740.0))
rows.sort(reverse=True)
print("  worst launches (excess k-steps, nprob, M N K atomic beta of the longest, TA TB, balanced):")
for r in rows[:12]:
    print("   ", r)
