"""Multi-rank sharded factorization vs the single-GPU factorization (run under
torchrun; RSC_DIST_BACKEND=gloo lets several ranks share one GPU -- host-staged
collectives, no kernel waits on another rank).  Rank 0 prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import factorize, pcg_solve  # noqa: E402
from paper_1507_05593_b200.distributed import factorize_distributed, unit_ranks  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig  # noqa: E402
from paper_1507_05593_b200.problems import elasticity_3d, laplacian_3d  # noqa: E402


def main():
    backend = os.environ.get("RSC_DIST_BACKEND", "nccl")
    dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    out = {}
    cases = [("l3d16_td48", laplacian_3d(16), dict(tau_o=16, tau_d=48, oversample=4)),
             ("l3d20", laplacian_3d(20), dict(tau_o=32, tau_d=64, oversample=10)),
             ("el7", elasticity_3d(7, strip_zeros=True), dict(tau_o=16, tau_d=32, oversample=4))]
    for name, (A, coords), kw in cases:
        cfg = SolverConfig(**kw)
        Fd = factorize_distributed(A, cfg, coords=coords)
        F1 = factorize(A, cfg, coords=coords)
        owners = unit_ranks(F1.sym, world)
        b = np.random.default_rng(0).standard_normal(A.n)
        z1, zd = F1.apply(b), Fd.apply(b)
        F2 = factorize(A, cfg, coords=coords)  # run-to-run noise of the single-GPU factor (atomic sums)
        z2 = F2.apply(b)
        x1, r1 = pcg_solve(A, b, preconditioner=F1, tol=1e-6)
        xd, rd = pcg_solve(A, b, preconditioner=Fd, tol=1e-6)
        x2, _ = pcg_solve(A, b, preconditioner=F2, tol=1e-6)
        mism = sorted(set(F1.ranks.items()) ^ set(Fd.ranks.items()))
        out[name] = {
            "n": A.n,
            "owned_units": int((owners == rank).sum()), "top_units": int((owners == -1).sum()),
            "ranks_equal": F1.ranks == Fd.ranks, "rank_mismatches": len(mism) // 2,
            "stored_equal": F1.stats.stored_scalars == Fd.stats.stored_scalars,
            "counters_equal": (F1.stats.compressed_offdiag, F1.stats.compressed_diag, F1.stats.dense_fallback)
            == (Fd.stats.compressed_offdiag, Fd.stats.compressed_diag, Fd.stats.dense_fallback),
            "model_gflop": [F1.stats.model_gflop, Fd.stats.model_gflop],
            "apply_relerr": float(np.linalg.norm(zd - z1) / np.linalg.norm(z1)),
            "apply_relerr_self": float(np.linalg.norm(z2 - z1) / np.linalg.norm(z1)),
            "pcg_its": [r1.iterations, rd.iterations],
            "x_relerr": float(np.linalg.norm(xd - x1) / np.linalg.norm(x1)),
            "x_relerr_self": float(np.linalg.norm(x2 - x1) / np.linalg.norm(x1)),
            "exchanged_bytes": Fd.dist["exchanged_bytes"],
            "factor_bytes_total": 8 * F1.stats.stored_scalars,
            "local_units": len(Fd.dist["local_units"]), "kept_units": len(Fd.dunits),
        }
    if rank == 0:
        print(json.dumps({"world": world, "backend": backend, "cases": out}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
