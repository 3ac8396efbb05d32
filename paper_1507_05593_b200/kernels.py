"""Dense building blocks with the reference contracts, computed on the B200.

Drop-in for rschol.kernels (reference pkg/src/rschol/kernels.py): same names,
arguments, return shapes and exceptions.  Host numpy arrays in and out; the
arithmetic runs in librsc_b200.so (FP64 DMMA POTRF/TRSM, pivoted Householder QR).
`gaussian_matrix` stays on the host on purpose: the sketches must be the
reference's own PCG64 stream, uploaded unchanged.
"""

import numpy as np
import torch

from . import engine as E
from .errors import IndefiniteError, SingularDiagonal

__all__ = ["dense_cholesky", "tri_solve", "orthonormalize", "gaussian_matrix", "low_rank_approx"]


def _dinv_for(n):
    return E.empty(max(n, 1), 64)


def dense_cholesky(M):
    """Lower Cholesky factor (lower triangle read); kernels.py:22-39.

    Raises IndefiniteError(pivot) with the 0-based index of the first
    non-positive pivot, never perturbs.
    """
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("dense_cholesky needs a square matrix")
    n = M.shape[0]
    if n == 0:
        return np.zeros((0, 0))
    A = E.to_dev(M)
    Dinv = _dinv_for(n)
    info = E.zeros(1, dtype=E.I32)
    E.potrf_batched([A.data_ptr()], [n], [n], [Dinv.data_ptr()], info)
    bad = int(info.item())
    if bad > 0:
        raise IndefiniteError(bad - 1)
    return A.cpu().numpy()


def _device_tri(L):
    n = L.shape[0]
    Ld = E.to_dev(np.tril(L))
    Dinv = _dinv_for(n)
    E.trtri_diag_batched([Ld.data_ptr()], [n], [n], [Dinv.data_ptr()])
    return Ld, Dinv


def tri_solve(L, B, transpose=False, side="left"):
    """Solve with a dense lower triangle; kernels.py:42-64.

    side="left":  L X = B   (L^T X = B with transpose)
    side="right": X L = B   (X L^T = B with transpose)
    """
    L = np.asarray(L, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    if L.shape[0] and np.any(np.diag(L) == 0.0):
        raise SingularDiagonal("zero on triangular diagonal")
    if L.shape[0] == 0:
        return B.copy()
    if side not in ("left", "right"):
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    n = L.shape[0]
    vec = B.ndim == 1
    B2 = B.reshape(-1, 1) if vec else B
    Ld, Dinv = _device_tri(L)
    if side == "left":
        X = E.to_dev(B2)
        E.trsm_batched("left", 1 if transpose else 0, [Ld.data_ptr()], [n], [n], [Dinv.data_ptr()],
                       [X.data_ptr()], [X.shape[1]], [E.ld(X)])
        out = X.cpu().numpy()
    elif transpose:
        X = E.to_dev(B2)  # X L^T = B
        E.trsm_batched("right", 1, [Ld.data_ptr()], [n], [n], [Dinv.data_ptr()], [X.data_ptr()],
                       [X.shape[0]], [E.ld(X)])
        out = X.cpu().numpy()
    else:
        Xt = E.to_dev(np.ascontiguousarray(B2.T))  # X L = B  <=>  L^T X^T = B^T
        E.trsm_batched("left", 1, [Ld.data_ptr()], [n], [n], [Dinv.data_ptr()], [Xt.data_ptr()],
                       [Xt.shape[1]], [E.ld(Xt)])
        out = np.ascontiguousarray(Xt.cpu().numpy().T)
    return out[:, 0] if vec else out


def orthonormalize(G):
    """Orthonormal basis of range(G) by pivoted QR with the reference cutoff;
    kernels.py:67-82.  Dependent columns are dropped."""
    G = np.asarray(G, dtype=np.float64)
    m, k = G.shape
    if k == 0 or m == 0:
        return np.zeros((m, 0))
    Gd = E.to_dev(G)
    Q = E.empty(m, k)
    rank = E.zeros(1, dtype=E.I32)
    work = E.qrcp_batched([Gd.data_ptr()], [m], [k], [k], [Q.data_ptr()], [k], rank)
    r = int(rank.item())
    del work
    return np.ascontiguousarray(Q[:, :r].cpu().numpy())


def gaussian_matrix(m, n, seed):
    """Seeded m x n standard normals from PCG64 (kernels.py:85-92), generated on
    the host so the stream is bit-identical to the reference's."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((m, n))


def low_rank_approx(B, rank, power_iters=0, seed=0):
    """Randomized range finder B ~ V U^T for an explicit B; kernels.py:95-113."""
    B = np.asarray(B, dtype=np.float64)
    m, n = B.shape
    rank = min(rank, m, n)
    Om = gaussian_matrix(m, rank, seed)
    if m == 0 or n == 0 or rank == 0:
        return np.zeros((m, 0)), np.zeros((n, 0))
    Bd = E.to_dev(B)
    G = E.empty(n, rank)
    E.gemm(Bd, E.to_dev(Om), G, transA=True)
    H = E.empty(m, rank)
    for _ in range(power_iters):
        E.gemm(Bd, G, H)
        E.gemm(Bd, H, G, transA=True)
    Q = E.empty(n, rank)
    rk = E.zeros(1, dtype=E.I32)
    work = E.qrcp_batched([G.data_ptr()], [n], [rank], [rank], [Q.data_ptr()], [rank], rk)
    r = int(rk.item())
    del work
    U = Q[:, :r].contiguous()
    V = E.empty(m, r)
    if r:
        E.gemm(Bd, U, V)
    return V.cpu().numpy(), U.cpu().numpy()
