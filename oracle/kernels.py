"""Dense kernels restated on LAPACK via scipy (reference kernels.py:22-113).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py)."""

import numpy as np
import scipy.linalg as sla
from scipy.linalg import lapack


class OracleIndefinite(Exception):
    def __init__(self, pivot):
        self.pivot = pivot
        super().__init__(f"indefinite at pivot {pivot}")


def chol(M):
    """kernels.py:22-39: dpotrf lower+clean, info>0 -> pivot info-1."""
    M = np.asarray(M, dtype=np.float64)
    if M.shape[0] == 0:
        return np.zeros((0, 0))
    c, info = lapack.dpotrf(M, lower=1, clean=1, overwrite_a=0)
    if info > 0:
        raise OracleIndefinite(int(info) - 1)
    return c


def trisolve(L, B, transpose=False, side="left"):
    """kernels.py:42-64."""
    if L.shape[0] == 0:
        return np.array(B, dtype=np.float64, copy=True)
    if side == "left":
        return sla.solve_triangular(L, B, lower=True, trans=1 if transpose else 0, check_finite=False)
    return sla.solve_triangular(L, B.T, lower=True, trans=0 if transpose else 1, check_finite=False).T


def orth(G):
    """kernels.py:67-82: pivoted QR, keep |R_ii| > max(m,k) eps |R_00|."""
    G = np.asarray(G, dtype=np.float64)
    m, k = G.shape
    if m == 0 or k == 0:
        return np.zeros((m, 0))
    Q, R, _ = sla.qr(G, mode="economic", pivoting=True, check_finite=False)
    d = np.abs(np.diag(R))
    if d.size == 0 or d[0] == 0.0:
        return np.zeros((m, 0))
    r = int(np.sum(d > max(m, k) * np.finfo(np.float64).eps * d[0]))
    return np.ascontiguousarray(Q[:, :r])


def gauss(m, n, seed):
    """kernels.py:85-92."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((m, n))


def block_seed(master, *tags):
    """factor.py:324-326."""
    return int(np.random.SeedSequence((int(master),) + tuple(int(t) for t in tags)).generate_state(1, np.uint64)[0])


def range_finder(B, rank, power_iters=0, seed=0):
    """kernels.py:95-113 (low_rank_approx)."""
    m, n = B.shape
    rank = min(rank, m, n)
    G = B.T @ gauss(m, rank, seed)
    for _ in range(power_iters):
        G = B.T @ (B @ G)
    U = orth(G)
    return B @ U, U


def cfg1_block(D, B, rank, power_iters, seed):
    """Config[1] per-block composition:
    chol -> L_O = B L_D^{-T} (factor.py:414 idiom) -> low_rank_approx."""
    LD = chol(D)
    LO = trisolve(LD, B.T).T
    V, U = range_finder(LO, rank, power_iters, seed)
    return LD, LO, V, U
