"""Compare an eager numeric pass with a captured+replayed one, unit by unit."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200.factor import SolverConfig, prepare, DenseTri, DevLR, DeviceTree  # noqa
from paper_1507_05593_b200.numeric import LevelPass  # noqa
from paper_1507_05593_b200.problems import laplacian_3d  # noqa

A, coords = laplacian_3d(int(sys.argv[1]) if len(sys.argv) > 1 else 14)
cfg = SolverConfig(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=64, power_iters=1, seed=0)
sym, plan, cfg, *_ = prepare(A, cfg, coords)
pe = LevelPass(plan, cfg, cfg.alpha_d)
pe.run()
pg = LevelPass(plan, cfg, cfg.alpha_d)
pg.capture()
pg.replay()
torch.cuda.synchronize()


def arr(x):
    if x is None:
        return None
    if isinstance(x, DenseTri):
        return x.L.cpu().numpy()
    if isinstance(x, DevLR):
        return (x.V.cpu().numpy() @ x.U.cpu().numpy().T)
    if isinstance(x, DeviceTree):
        return None
    return x.cpu().numpy()


bad = 0
for u, (a, b) in enumerate(zip(pe.units, pg.units)):
    for attr in ("diag", "off"):
        xa, xb = arr(getattr(a, attr, None)), arr(getattr(b, attr, None))
        if xa is None or xb is None:
            continue
        d = np.abs(xa - xb).max() / max(np.abs(xa).max(), 1e-300)
        if d > 1e-8:
            print("unit", u, a.kind if hasattr(a, "kind") else type(a).__name__, attr, xa.shape, f"{d:.2e}")
            bad += 1
            if bad > 12:
                sys.exit(0)
print("done, mismatches:", bad, "ranks equal:", pe.ranks == pg.ranks)

from paper_1507_05593_b200 import factorize  # noqa: E402

r = np.random.default_rng(1).standard_normal(A.n)
Fe = factorize(A, cfg, coords=coords)
prep = prepare(A, cfg, coords)
Fg = factorize(A, prepared=prep)
ze, zg = Fe.apply(r), Fg.apply(r)
print("apply relerr eager vs graph", np.linalg.norm(ze - zg) / np.linalg.norm(ze))
Fg._apply = None
Fg._entry = None
zg2 = Fg.apply(r)
print("graph factor, fresh apply program", np.linalg.norm(ze - zg2) / np.linalg.norm(ze))
bad = 0
for u, (a, b) in enumerate(zip(Fe.units, Fg.units)):
    for attr in ("diag", "off", "tri", "Y"):
        xa, xb = arr(getattr(a, attr, None)), arr(getattr(b, attr, None))
        if xa is None or xb is None:
            continue
        d = np.abs(xa - xb).max() / max(np.abs(xa).max(), 1e-300)
        if d > 1e-8:
            print("F unit", u, type(a).__name__, attr, xa.shape, f"{d:.2e}")
            bad += 1
print("factor mismatches", bad, Fe.ranks == Fg.ranks, Fe.stats.stored_scalars, Fg.stats.stored_scalars)
