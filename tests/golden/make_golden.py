"""Generate the golden fixtures by running the REFERENCE implementation itself.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py [section ...]

Sections: kernels, cfg1, symbolic, factor.  Outputs tests/golden/<section>*.npz.
The fixtures pin (a) the oracle restatement (tests/test_oracle_golden.py) and
(b) the GPU path's symbolic plan (tests/test_symbolic.py) on hosts without the
reference.  Inputs are seeded generators, so fixtures stay small.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import rschol as rs  # noqa: E402
from rschol import factor as rfactor  # noqa: E402
from rschol import problems as rprob  # noqa: E402

# the benchmark knob mapping of SURVEY §8(d)
KNOBS = dict(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=256, power_iters=1, seed=0,
             interior_blocks=True, max_restarts=10)


def sec_kernels():
    rng = np.random.default_rng(7)
    out = {}
    for n in (1, 7, 23, 50, 64, 65, 130, 256):
        M = rng.standard_normal((n, n))
        M = M @ M.T + n * np.eye(n)
        out[f"chol_in_{n}"] = M
        out[f"chol_out_{n}"] = rs.dense_cholesky(M)
    L = np.tril(rng.standard_normal((150, 150))) + 12 * np.eye(150)
    B = rng.standard_normal((150, 37))
    out["tri_L"] = L
    out["tri_B"] = B
    out["tri_left"] = rs.tri_solve(L, B)
    out["tri_left_t"] = rs.tri_solve(L, B, transpose=True)
    out["tri_right_t"] = rs.tri_solve(L, B.T, transpose=True, side="right")
    out["tri_right"] = rs.tri_solve(L, B.T, side="right")
    for tag, (m, k) in {"a": (300, 40), "b": (64, 90), "c": (256, 58)}.items():
        G = rng.standard_normal((m, k))
        if tag == "c":  # rank-deficient sketch: 30 strong directions + tiny noise
            G = rng.standard_normal((m, 30)) @ rng.standard_normal((30, k)) + 1e-15 * G
        out[f"orth_in_{tag}"] = G
        out[f"orth_out_{tag}"] = rs.orthonormalize(G)
    Bl = rng.standard_normal((200, 12)) @ rng.standard_normal((12, 90)) + 1e-9 * rng.standard_normal((200, 90))
    V, U = rs.low_rank_approx(Bl, 30, power_iters=1, seed=5)
    out["lra_in"] = Bl
    out["lra_V"] = V
    out["lra_U"] = U
    out["gauss_7x3_99"] = rs.gaussian_matrix(7, 3, 99)
    out["block_seed_0_0_5"] = np.array([rfactor._block_seed(0, 0, 5)], dtype=np.uint64)
    out["block_seed_0_1_9_3"] = np.array([rfactor._block_seed(0, 1, 9, 3)], dtype=np.uint64)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def sec_cfg1(nb=4):
    """Config[1] composition on the first `nb` blocks of the seeded batch."""
    from paper_1507_05593_b200.problems import batched_supernodes  # generator pinned below

    D, B = batched_supernodes(nb=nb)
    out = {"D0": D[0], "B0_head": B[0, :8]}
    for i in range(nb):
        LD = rs.dense_cholesky(D[i])
        LO = rs.tri_solve(LD, B[i].T).T
        V, U = rs.low_rank_approx(LO, 58, power_iters=1, seed=rfactor._block_seed(0, 0, i))
        out[f"rank_{i}"] = np.array([U.shape[1]])
        out[f"LD_{i}"] = LD
        out[f"VUt_{i}_head"] = (V @ U.T)[:64]
        out[f"LO_{i}_head"] = LO[:64]
    np.savez_compressed(os.path.join(OUT, "cfg1.npz"), **out)


INF = float("inf")
# name -> (generator, args, strip zeros, knob overrides, keep dense_lower)
FACTOR_CASES = {
    "l2d16_exact": ("laplacian_2d", (16,), False, dict(tau_o=INF), True),
    "l3d8_small": ("laplacian_3d", (8,), False, dict(tau_o=16, tau_d=32, oversample=4), True),
    "l3d12": ("laplacian_3d", (12,), False, dict(tau_d=64), True),
    "l3d16": ("laplacian_3d", (16,), False, dict(tau_d=64), False),
    "el5": ("elasticity_3d", (5,), True, dict(tau_o=16, tau_d=32, oversample=4), True),
    "el7": ("elasticity_3d", (7,), True, dict(tau_d=64), False),
    "cfg0": ("laplacian_2d", (128,), False, dict(), False),
    "l3d24": ("laplacian_3d", (24,), False, dict(), False),
    "l3d16_noint": ("laplacian_3d", (16,), False, dict(tau_d=64, interior_blocks=False), False),
    "l3d20_td32": ("laplacian_3d", (20,), False, dict(tau_o=16, tau_d=32, oversample=4), False),
    "el9_td48": ("elasticity_3d", (9,), True, dict(tau_o=24, tau_d=48, oversample=6), False),
}


def _strip(A):
    keep = A.values != 0.0
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.col_ptr))
    return rs.SparseSpdMatrix.from_coo(A.n, A.row_idx[keep], cols[keep], A.values[keep])


def _units_code(units):
    """(kind, first, last) per unit: kind 0 interior [members j0..j1], 1 node j."""
    out = []
    for kind, obj in units:
        if kind == "interior":
            ids = [m.j for m in obj.members]
            out.append((0, ids[0], ids[-1]))
        else:
            out.append((1, obj.j, obj.j))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


def sec_factor():
    """Symbolic plan + numeric results of the reference on small instances."""
    for name, (gen, args, strip, over, keep_dense) in FACTOR_CASES.items():
        A, coords = getattr(rprob, gen)(*args)
        if strip:
            A = _strip(A)
        cfg = rs.SolverConfig(**dict(KNOBS, **over))
        F = rs.factorize(A, cfg, coords=coords)
        part = F.partition
        rows = part.rows
        out = {
            "perm": F.perm.forward,
            "starts": part.starts,
            "is_sep": part.is_separator,
            "rows_ptr": np.concatenate([[0], np.cumsum([r.size for r in rows])]).astype(np.int64),
            "rows_idx": np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, np.int64),
            "units": _units_code(F.units),
            "stored_scalars": np.array([F.stored_scalars()]),
            "restarts": np.array([F.stats.restarts]),
            "counts": np.array([F.stats.compressed_offdiag, F.stats.compressed_diag, F.stats.dense_fallback]),
        }
        # diagonal-tree leaf sizes per tree node and kept ranks of compressed blocks
        ranks = []
        for kind, obj in F.units:
            if kind != "node":
                continue
            if isinstance(obj.offdiag, rs.LowRankBlock):
                ranks.append((obj.j, -1, obj.offdiag.rank))
            if isinstance(obj.diag, rs.DiagBlockTree):
                for s in obj.diag.inorder_ids():
                    b = obj.diag.blocks[s]
                    if isinstance(b, rs.LowRankBlock):
                        ranks.append((obj.j, s, b.rank))
                out[f"leaves_{obj.j}"] = np.array(
                    [obj.diag.nodes[s].hi - obj.diag.nodes[s].lo for s in obj.diag.leaf_ids()])
        out["ranks"] = np.array(ranks, dtype=np.int64).reshape(-1, 3)
        r = np.random.default_rng(1).standard_normal(A.n)
        out["apply_r"] = F.apply(r)
        b = np.random.default_rng(0).standard_normal(A.n)
        x, rep = rs.pcg_solve(A, b, preconditioner=F, tol=1e-6)
        out["pcg_x"] = x
        out["pcg_iters"] = np.array([rep.iterations])
        out["pcg_hist"] = np.array(rep.relative_residual_history)
        if keep_dense:
            L = F.dense_lower()
            Bm = rs.permute_symmetric(A, F.perm).dense()
            out["L_dense"] = L
            out["resid"] = np.array([np.linalg.norm(L @ L.T - Bm) / np.linalg.norm(A.dense())])
        np.savez_compressed(os.path.join(OUT, f"factor_{name}.npz"), **out)
        print(" ", name, A.n, "iters", rep.iterations, "ranks", len(ranks))


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))
    secs = sys.argv[1:] or ["kernels", "cfg1"]
    for s in secs:
        globals()[f"sec_{s}"]()
        print("wrote", s)
