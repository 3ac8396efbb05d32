"""Full-size determinism + parity probe on the GPU box (exploratory; the pinned
version is tests/test_fullsize_gpu.py).

    python tools/fullsize_check.py 2 3 4   [--runs 3]

Per config: one-shot factorize, then prepare() + 2 refactorizations (eager, then
graph replay); reports whether kept ranks / apply(r) bits agree across runs, the
rank mismatches against tests/golden/full_cfgN.npz with their reference decision
margins, PCG iterations / x error and the shared-probe Hutchinson residual.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fullsize as FS  # noqa: E402
from paper_1507_05593_b200 import factorize, pcg_solve  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, prepare  # noqa: E402
from paper_1507_05593_b200.problems import config_problem  # noqa: E402


def main():
    cfgs = [int(a) for a in sys.argv[1:] if a.isdigit()]
    out = {}
    for cfg in cfgs:
        A, coords = config_problem(cfg)
        g = FS.fixture(cfg)
        conf = SolverConfig(**FS.KNOBS)
        r = np.random.default_rng(1).standard_normal(A.n)
        res = {"n": A.n}
        runs = []
        t = time.perf_counter()
        F = factorize(A, conf, coords=coords)
        res["oneshot_s"] = time.perf_counter() - t
        runs.append((FS.rank_list(F), F.apply(r), FS.factor_digest(F)))
        prep = prepare(A, conf, coords)
        for i in range(2):
            t = time.perf_counter()
            F2 = factorize(A, prepared=prep)
            res[f"refactor{i}_s"] = time.perf_counter() - t
            runs.append((FS.rank_list(F2), F2.apply(r), FS.factor_digest(F2)))
            del F2
        res["ranks_identical"] = all(x[0] == runs[0][0] for x in runs)
        res["factor_digest_identical"] = all(x[2] == runs[0][2] for x in runs)
        res["apply_bits_identical"] = all(np.array_equal(x[1], runs[0][1]) for x in runs)
        res["apply_maxrel_between_runs"] = max(float(np.abs(x[1] - runs[0][1]).max() / np.abs(runs[0][1]).max())
                                                for x in runs)
        res["nblocks"] = len(runs[0][0])
        if g is not None:
            res["symbolic_sha_equal"] = bool(
                np.array_equal(FS.sha(F.perm.forward.astype(np.int64)), g["perm_sha"])
                and np.array_equal(FS.sha(F.partition.starts.astype(np.int64)), g["starts_sha"])
                and np.array_equal(FS.sha(np.concatenate(F.partition.rows).astype(np.int64)), g["rows_sha"]))
            d = FS.rank_diff(F, g)
            res["rank_mismatches"] = len(d)
            res["rank_mismatch_detail"] = d[:40]
            res["stored_scalars"] = [F.stored_scalars(), int(g["stored_scalars"][0])]
            b = np.random.default_rng(0).standard_normal(A.n)
            t = time.perf_counter()
            x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6)
            res["pcg_s"] = time.perf_counter() - t
            res["pcg_iters"] = [rep.iterations, int(g["pcg_iters"][0])]
            res["x_relerr"] = float(np.linalg.norm(x - g["pcg_x"]) / np.linalg.norm(g["pcg_x"]))
            t = time.perf_counter()
            h = FS.hutchinson(A, F)
            res["hutch"] = [h, float(g["resid_hutch"][0])]
            res["hutch_rel"] = abs(h - float(g["resid_hutch"][0])) / float(g["resid_hutch"][0])
            res["hutch_s"] = time.perf_counter() - t
        out[cfg] = res
        print(json.dumps({cfg: res}, default=str), flush=True)
        del F, runs


if __name__ == "__main__":
    main()
