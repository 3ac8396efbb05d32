"""Kept-rank and factor digests of one factorization per config (bit-identity A/B of
two library builds: RSC_B200_LIB=... python tools/digest.py 2 3 4)."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import fullsize as FS  # noqa: E402
import torch  # noqa: E402

from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

for cfg in [int(x) for x in sys.argv[1:]]:
    A, coords = _problem(cfg, GRID[cfg])
    prep = prepare(A, SolverConfig(**KNOBS), coords)
    F = factorize(A, prepared=prep)
    del F
    torch.cuda.synchronize()
    t = time.perf_counter()
    F = factorize(A, prepared=prep)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    rl = FS.rank_list(F)
    rh = hashlib.sha256(repr(rl).encode()).hexdigest()[:16]
    print(f"cfg{cfg} ranks {rh} factor {FS.factor_digest(F)} sum_ranks {sum(r for *_, r in rl)} numeric {dt:.3f}s", flush=True)
