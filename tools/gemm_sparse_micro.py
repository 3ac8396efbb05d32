"""Grouped GEMM on sparse-sweep-like shapes: effect of atomics, gathers, scatters."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402

rng = np.random.default_rng(0)


def bench(nprob, M, N, K, transA=False, atomic=False, gather=False, scatter=False, reps=10):
    As = [torch.randn(K, M) if transA else torch.randn(M, K) for _ in range(nprob)]
    As = [a.double().cuda() for a in As]
    Bs = [torch.randn(K + 64, N, dtype=torch.float64, device="cuda") for _ in range(nprob)]
    Cs = [torch.zeros(M + 64, N, dtype=torch.float64, device="cuda") for _ in range(nprob)]
    idx = [torch.from_numpy(rng.permutation(K + 64)[:K].astype(np.int32)).cuda() for _ in range(nprob)]
    cidx = [torch.from_numpy(rng.permutation(M + 64)[:M].astype(np.int32)).cuda() for _ in range(nprob)]
    p = E.gemm_problems(nprob)
    p["A"] = [a.data_ptr() for a in As]
    p["B"] = [b.data_ptr() for b in Bs]
    p["C"] = [c.data_ptr() for c in Cs]
    p["M"], p["N"], p["K"] = M, N, K
    p["lda"] = M if transA else K
    p["ldb"], p["ldc"], p["batch"], p["alpha"] = N, N, 1, 1.0
    p["beta"] = 1.0
    p["atomic"] = int(atomic)
    if gather:
        p["b_rows"] = [i.data_ptr() for i in idx]
    if scatter:
        p["c_rows"] = [i.data_ptr() for i in cidx]
    E.gemm_grouped(p, transA, False)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        E.gemm_grouped(p, transA, False)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return 2.0 * nprob * M * N * K / ms / 1e9


if __name__ == "__main__":
    for (n, M, N, K) in ((150, 512, 256, 448), (150, 512, 64, 448), (150, 2048, 128, 96), (150, 128, 128, 2048)):
        for ta in (False, True):
            base = bench(n, M, N, K, ta)
            at = bench(n, M, N, K, ta, atomic=True)
            ga = bench(n, M, N, K, ta, gather=True)
            sc = bench(n, M, N, K, ta, atomic=True, scatter=True)
            print(f"{n}x M{M} N{N} K{K} TA={int(ta)}: plain {base:5.1f}  atomic {at:5.1f}  gather {ga:5.1f}  "
                  f"atomic+scatter {sc:5.1f} TF/s")
