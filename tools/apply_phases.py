"""Per-phase device time of one preconditioner apply (CUPTI kernel records of an
eager run) with each phase's matrix bytes: where the apply's time goes."""
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402

cfg, grid = int(sys.argv[1]), int(sys.argv[2])
A, coords = _problem(cfg, grid)
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
z = E.empty(A.n)
F.apply_device(r, z)
ap = F._apply
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as kp:
    ap._run_program()
    torch.cuda.synchronize()
kev = [e for e in kp.events() if e.device_type.name == "CUDA"]
gem = [e for e in kev if "gemv" in e.name]
GMAXP = int(os.environ.get("GMAXP", "224"))  # csrc/apply.cu GMAXP
print("phases", len(ap.phases), "gemv kernel records", len(gem), "all", len(kev),
      "(set RSC_APPLY_NO_PDL=1: with PDL a record includes the wait for the previous phase)")
rows, k = [], 0
for ph in ap.phases:
    live = [it for it in ph.items if it[1] > 0 and it[2] > 0]
    n_all = len(ph.items)  # phases of >= DEV_MIN problems run as one device-descriptor launch
    nl = (1 if n_all >= ap.DEV_MIN else max(1, -(-len(live) // GMAXP))) if live else 0
    t = sum(e.device_time for e in gem[k:k + nl])
    k += nl
    byts = sum(8 * it[1] * it[2] for it in live)
    big = max((8 * it[1] * it[2] for it in live), default=0)
    modes = "".join(sorted({str(it[8]) for it in live}))
    rows.append((t, byts, len(live), big, modes))
tot_t = sum(r[0] for r in rows)
tot_b = sum(r[1] for r in rows)
print(f"matched {k} of {len(gem)} records; sum kernel time {tot_t / 1e3:.3f} ms, matrix bytes {tot_b / 1e9:.3f} GB "
      f"-> {tot_b / max(tot_t, 1e-9) / 1e3:.1f} GB/s")
edges = [0, 1e5, 1e6, 4e6, 16e6, 64e6, 1e12]
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = [r for r in rows if lo <= r[1] < hi]
    if sel:
        tt = sum(r[0] for r in sel)
        bb = sum(r[1] for r in sel)
        print(f"phases {lo / 1e6:7.1f}-{hi / 1e6:7.1f} MB: {len(sel):4d} phases {tt / 1e3:7.3f} ms "
              f"({tt / len(sel):6.1f} us each) {bb / max(tt, 1e-9) / 1e3:7.1f} GB/s")
for t, b, n, big, modes in sorted(rows, reverse=True)[:20]:
    print(f"{t:8.1f} us  {b / 1e6:8.2f} MB  {b / t / 1e3 if t else 0:7.1f} GB/s  problems {n:4d}  largest {big / 1e6:7.2f} MB  modes {modes}")
