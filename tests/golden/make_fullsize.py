"""Full-size reference fixtures for the BASELINE configs ("missing" item 1).

Runs the REFERENCE implementation (/root/reference/pkg/src/rschol) on configs 2, 3, 4 at
their BASELINE sizes, and the config[1] composition on all 512 blocks, and pins what the
north-star parity bars are about:

* symbolic structure: sha256 of perm / supernode starts / concatenated row structures;
* every pivoted-QR decision, in call order, tagged (kind, j, s): m, k, kept rank and the
  decision margins |R_ii| / cutoff of the last kept and the first dropped column
  (ref kernels.py:77-82; cutoff = max(m,k) eps |R_00|);
* kept-rank census per compressed block, stored scalars, counters, restarts;
* PCG: iterations, relative-residual history, solution x (pcg.py:64-135, tol 1e-6,
  b = default_rng(0).standard_normal(n));
* a shared-probe Hutchinson estimate of ||PAP^T - L L^T||_F: probes
  Z = default_rng(HUTCH_SEED).standard_normal((n, HUTCH_K)) in the permuted ordering;
  the GPU test multiplies its own factor by the SAME Z.

Usage (build container only; the reference does not exist on the GPU box):

    OMP_NUM_THREADS=1 python tests/golden/make_fullsize.py cfg1 | full2 | full3 | full4

Config[3]'s generator is ours (the reference has none); the matrix is
handed to the reference as a plain lower CSC.  Config[4] is the reference generator
with stored zeros stripped (SURVEY finding 6), done identically on both sides.
"""

import hashlib
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(OUT)))

import rschol as rs  # noqa: E402
from rschol import diagblocks as rdiag  # noqa: E402
from rschol import factor as rfactor  # noqa: E402
from rschol import kernels as rkernels  # noqa: E402
from rschol import problems as rprob  # noqa: E402
import scipy.linalg as sla  # noqa: E402

KNOBS = dict(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=256, power_iters=1, seed=0,
             interior_blocks=True, max_restarts=10)
HUTCH_SEED = 20251020
HUTCH_K = 8
EPS = np.finfo(np.float64).eps


def sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8).copy()


# --- QR decision recorder --------------------------------------------------------------
_QR = []
_TAG = [(-1, -1, -1)]


def _record(G):
    G = np.asarray(G, dtype=np.float64)
    m, k = G.shape
    if k == 0 or m == 0:
        _QR.append(_TAG[-1] + (m, k, 0, np.nan, np.nan))
        return
    R = sla.qr(G, mode="r", pivoting=True, check_finite=False)[0]
    d = np.abs(np.diag(R))
    cut = max(m, k) * EPS * d[0]
    kept = int(np.sum(d > cut))
    last = d[kept - 1] / cut if kept > 0 else np.nan
    first = d[kept] / cut if kept < d.size else np.nan
    _QR.append(_TAG[-1] + (m, k, kept, last, first))


def _wrap_orth(orig):
    def orth(G):
        _record(G)
        return orig(G)
    return orth


def _wrap_off(orig):
    def f(A, j, L, rank, **kw):
        _TAG.append((0, j, -1))
        try:
            return orig(A, j, L, rank, **kw)
        finally:
            _TAG.pop()
    return f


def _wrap_diag(orig):
    def f(A, L, j, s, rank, **kw):
        _TAG.append((1, j, s))
        try:
            return orig(A, L, j, s, rank, **kw)
        finally:
            _TAG.pop()
    return f


rfactor.orthonormalize = _wrap_orth(rfactor.orthonormalize)
rdiag.orthonormalize = _wrap_orth(rdiag.orthonormalize)
rkernels.orthonormalize = _wrap_orth(rkernels.orthonormalize)
rfactor.approximate_off_diagonal = _wrap_off(rfactor.approximate_off_diagonal)
rdiag.approximate_diagonal_block = _wrap_diag(rdiag.approximate_diagonal_block)
_orig_pass = rfactor._numeric_pass


def _pass(*a, **kw):
    _QR.clear()  # only the accepted (last) pass's decisions are kept
    return _orig_pass(*a, **kw)


rfactor._numeric_pass = _pass


# --- L multiply on the reference factor (test infrastructure only) --------------------
def lower_mul(F, X, transpose=False):
    """Y = L X (or L^T X) for the reference factor, in the permuted ordering.  Block
    layout as in RankStructuredFactor.dense_lower (ref factor.py:243-266)."""
    Y = np.zeros_like(X)

    def blk(rr, cc, M, lowrank=None):
        # block M (dense) or lowrank (V, U) occupying rows rr, cols cc
        if lowrank is not None:
            if transpose:
                Y[cc] += lowrank.rmatmat(X[rr])
            else:
                Y[rr] += lowrank.matmat(X[cc])
        elif transpose:
            Y[cc] += M.T @ X[rr]
        else:
            Y[rr] += M @ X[cc]

    for kind, obj in F.units:
        if kind == "interior":
            for m in obj.members:
                mc = np.arange(m.c0, m.c1)
                blk(mc, mc, np.tril(m.diag))
                if m.nrows_in_block:
                    blk(m.rows[: m.nrows_in_block], mc, m.offdiag)
            if obj.off_rows.size:
                # L(off, C_B) = coupling L_B^{-T}
                if transpose:
                    Y[obj.c0:obj.c1] += obj.solve(obj.coupling.T @ X[obj.off_rows], transpose=False)
                else:
                    Y[obj.off_rows] += obj.coupling @ obj.solve(X[obj.c0:obj.c1], transpose=True)
            continue
        c0 = obj.c0
        if isinstance(obj.diag, rs.DiagBlockTree):
            tree = obj.diag
            for s, node in tree.nodes.items():
                content = tree.blocks[s]
                (r0, r1), (k0, k1) = tree.col_span(s)
                rr, cc = np.arange(c0 + r0, c0 + r1), np.arange(c0 + k0, c0 + k1)
                if node.is_leaf:
                    blk(rr, cc, np.tril(content))
                elif isinstance(content, rs.LowRankBlock):
                    blk(rr, cc, None, content)
                else:
                    blk(rr, cc, content)
        else:
            cc = np.arange(obj.c0, obj.c1)
            blk(cc, cc, np.tril(obj.diag))
        if obj.rows.size and obj.offdiag is not None:
            cc = np.arange(obj.c0, obj.c1)
            if isinstance(obj.offdiag, rs.LowRankBlock):
                blk(obj.rows, cc, None, obj.offdiag)
            else:
                blk(obj.rows, cc, obj.offdiag)
    return Y


def _strip(A):
    keep = A.values != 0.0
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.col_ptr))
    return rs.SparseSpdMatrix.from_coo(A.n, A.row_idx[keep], cols[keep], A.values[keep])


def _problem(cfg):
    if cfg == 2:
        return rprob.laplacian_3d(64)
    if cfg == 4:
        A, c = rprob.elasticity_3d(65)
        return _strip(A), c
    if cfg == 3:
        from paper_1507_05593_b200.problems import diffusion_fv_3d

        A, c = diffusion_fv_3d(96)
        return rs.SparseSpdMatrix(A.n, A.col_ptr, A.row_idx, A.values), c.xyz
    raise ValueError(cfg)


def full(cfg):
    t0 = time.perf_counter()
    A, coords = _problem(cfg)
    F = rs.factorize(A, rs.SolverConfig(**KNOBS), coords=coords)
    tf = time.perf_counter() - t0
    part = F.partition
    rows = part.rows
    out = {
        "n": np.array([A.n]),
        "nnz_lower": np.array([A.row_idx.size]),
        "perm_sha": sha(F.perm.forward.astype(np.int64)),
        "starts_sha": sha(part.starts.astype(np.int64)),
        "rows_sha": sha(np.concatenate(rows).astype(np.int64)),
        "nsupernodes": np.array([part.count]),
        "nunits": np.array([len(F.units)]),
        "stored_scalars": np.array([F.stored_scalars()]),
        "restarts": np.array([F.stats.restarts]),
        "counts": np.array([F.stats.compressed_offdiag, F.stats.compressed_diag, F.stats.dense_fallback]),
        "phase_times": np.array([F.stats.phase_times.get(k, np.nan) for k in ("ordering", "symbolic", "numeric", "total")]),
    }
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
    out["ranks"] = np.array(ranks, dtype=np.int64).reshape(-1, 3)
    q = np.array(_QR, dtype=np.float64).reshape(-1, 8)
    out["qr_tag"] = q[:, :6].astype(np.int64)  # kind, j, s, m, k, kept
    out["qr_margin"] = q[:, 6:]  # |R| / cutoff: last kept, first dropped
    print(f"cfg{cfg}: n={A.n} factor {tf:.1f}s qr calls {len(_QR)} stored {out['stored_scalars'][0]}", flush=True)

    b = np.random.default_rng(0).standard_normal(A.n)
    t1 = time.perf_counter()
    x, rep = rs.pcg_solve(A, b, preconditioner=F, tol=1e-6)
    out["pcg_seconds"] = np.array([time.perf_counter() - t1])
    out["pcg_x"] = x
    out["pcg_iters"] = np.array([rep.iterations])
    out["pcg_hist"] = np.array(rep.relative_residual_history)
    print(f"cfg{cfg}: pcg {rep.iterations} its {out['pcg_seconds'][0]:.1f}s", flush=True)

    Bm = rs.permute_symmetric(A, F.perm)
    Bfull = Bm.to_csr_full()
    Z = np.random.default_rng(HUTCH_SEED).standard_normal((A.n, HUTCH_K))
    LtZ = lower_mul(F, Z, transpose=True)
    EZ = Bfull @ Z - lower_mul(F, LtZ)
    out["hutch_ez_col"] = np.linalg.norm(EZ, axis=0)
    out["hutch_az_col"] = np.linalg.norm(Bfull @ Z, axis=0)
    out["hutch_ltz_col"] = np.linalg.norm(LtZ, axis=0)
    out["a_fro"] = np.array([np.sqrt(np.sum(Bfull.data ** 2))])
    out["resid_hutch"] = np.array([np.linalg.norm(EZ) / np.sqrt(HUTCH_K) / out["a_fro"][0]])
    print(f"cfg{cfg}: hutchinson resid {out['resid_hutch'][0]:.4e}", flush=True)
    np.savez_compressed(os.path.join(OUT, f"full_cfg{cfg}.npz"), **out)


def cfg1():
    """All 512 config[1] blocks through the reference kernels."""
    from paper_1507_05593_b200.problems import batched_supernodes

    D, B = batched_supernodes(nb=512)
    w = np.random.default_rng(HUTCH_SEED).standard_normal(256)
    ranks, ld_diag, fro, vuw = [], [], [], []
    for i in range(512):
        LD = rs.dense_cholesky(D[i])
        LO = rs.tri_solve(LD, B[i].T).T
        V, U = rs.low_rank_approx(LO, 58, power_iters=1, seed=rfactor._block_seed(0, 0, i))
        ranks.append(U.shape[1])
        ld_diag.append(np.diag(LD))
        fro.append((np.linalg.norm(LD), np.linalg.norm(LO), np.linalg.norm(V @ U.T)))
        vuw.append((V @ (U.T @ w))[:64])
    q = np.array(_QR, dtype=np.float64).reshape(-1, 8)
    np.savez_compressed(os.path.join(OUT, "full_cfg1.npz"), ranks=np.array(ranks), ld_diag=np.array(ld_diag),
                        fro=np.array(fro), vuw_head=np.array(vuw), qr_margin=q[:, 6:])
    print("cfg1: ranks", sorted(set(ranks)))


if __name__ == "__main__":
    for s in sys.argv[1:]:
        if s == "cfg1":
            cfg1()
        else:
            full(int(s.replace("full", "")))
