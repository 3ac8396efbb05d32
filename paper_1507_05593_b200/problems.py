"""Synthetic SPD problems of the five BASELINE configs (matrix + coordinates).

laplacian_2d / laplacian_3d / elasticity_3d reproduce the reference generators
(pkg/src/rschol/problems.py:21-64,147-230) value-for-value, including the order in
which duplicate element contributions are summed (pinned by tests/golden).
diffusion_fv_3d is the config[3] generator, which the reference lacks (SURVEY
§8(d)): cell-centred 7-point finite volumes, kappa = exp(sigma g), harmonic face
transmissibilities, Dirichlet walls with transmissibility 2 kappa_i.
batched_supernodes is the config[1] input.
"""

import numpy as np

from .sparse import SparseSpdMatrix, strip_explicit_zeros

__all__ = [
    "Coordinates",
    "laplacian_2d",
    "laplacian_3d",
    "elasticity_3d",
    "diffusion_fv_3d",
    "batched_supernodes",
    "config_problem",
]


class Coordinates:
    """Per-index 3-D positions (the reference's IndexCoordinates, ordering.py:375-389)."""

    def __init__(self, xyz, source="geometric-file", converged=True):
        self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        if self.xyz.ndim != 2 or self.xyz.shape[1] != 3:
            from .errors import MissingCoordinates

            raise MissingCoordinates("coordinates must be (n, 3)")
        self.source = source
        self.converged = converged

    @property
    def n(self):
        return self.xyz.shape[0]


def _stencil_pairs(shape):
    """Lower-triangle (row, col) pairs of nearest neighbours along each axis of a
    lexicographic grid (last axis fastest), axis by axis."""
    idx = np.arange(int(np.prod(shape))).reshape(shape)
    out = []
    for ax in range(len(shape)):
        hi = np.take(idx, np.arange(1, shape[ax]), axis=ax).ravel()
        lo = np.take(idx, np.arange(0, shape[ax] - 1), axis=ax).ravel()
        out.append((np.maximum(hi, lo), np.minimum(hi, lo)))
    return idx, out


def _grid_laplacian(shape, diag):
    n = int(np.prod(shape))
    idx, pairs = _stencil_pairs(shape)
    rows = [idx.ravel()] + [p[0] for p in pairs]
    cols = [idx.ravel()] + [p[1] for p in pairs]
    vals = [np.full(n, float(diag))] + [np.full(p[0].size, -1.0) for p in pairs]
    A = SparseSpdMatrix.from_coo(n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    pos = np.stack(np.unravel_index(np.arange(n), shape), axis=1).astype(float)
    if pos.shape[1] == 2:
        pos = np.column_stack([pos, np.zeros(n)])
    return A, Coordinates(pos)


def laplacian_2d(N):
    """5-point Dirichlet Laplacian on an N x N grid (config[0] at N=128)."""
    if N < 2:
        raise ValueError("N must be at least 2")
    return _grid_laplacian((N, N), 4.0)


def laplacian_3d(N):
    """7-point Dirichlet Laplacian on an N^3 grid (config[2] at N=64)."""
    if N < 2:
        raise ValueError("N must be at least 2")
    return _grid_laplacian((N, N, N), 6.0)


def diffusion_fv_3d(N, sigma=2.0, seed=0):
    """Config[3]: cell-centred FV diffusion, kappa = exp(sigma g), g ~ N(0,1) per cell
    from default_rng(seed); interior faces 2 k_i k_j / (k_i + k_j), wall faces 2 k_i."""
    if N < 2:
        raise ValueError("N must be at least 2")
    shape = (N, N, N)
    n = N**3
    g = np.random.default_rng(seed).standard_normal(shape)
    kap = np.exp(sigma * g).ravel()
    idx, pairs = _stencil_pairs(shape)
    diag = np.zeros(n)
    rows, cols, vals = [], [], []
    for r, c in pairs:
        t = 2.0 * kap[r] * kap[c] / (kap[r] + kap[c])
        np.add.at(diag, r, t)
        np.add.at(diag, c, t)
        rows.append(r)
        cols.append(c)
        vals.append(-t)
    # Dirichlet walls: each cell on a boundary face gets 2 kappa_i per wall face
    coord = np.unravel_index(np.arange(n), shape)
    walls = np.zeros(n)
    for ax in range(3):
        walls += (coord[ax] == 0).astype(float) + (coord[ax] == N - 1).astype(float)
    diag += 2.0 * kap * walls
    A = SparseSpdMatrix.from_coo(n, np.concatenate([np.arange(n)] + rows),
                                 np.concatenate([np.arange(n)] + cols), np.concatenate([diag] + vals))
    pos = np.stack(coord, axis=1).astype(float)
    return A, Coordinates(pos)


def _hex_stiffness(h, lam, mu):
    """Trilinear 8-node brick stiffness, 2x2x2 Gauss (problems.py:147-188 contract)."""
    gauss = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    corner = np.array([[a, b, c] for a in (0, 1) for b in (0, 1) for c in (0, 1)], dtype=np.float64)
    sgn = 2.0 * corner - 1.0
    Dm = np.zeros((6, 6))
    Dm[:3, :3] = lam
    Dm[np.arange(3), np.arange(3)] += 2.0 * mu
    Dm[3:, 3:] = mu * np.eye(3)
    K = np.zeros((24, 24))
    jac = (h / 2.0) ** 3
    for gx in gauss:
        for gy in gauss:
            for gz in gauss:
                pt = np.array([gx, gy, gz])
                dN = np.empty((8, 3))
                for a in range(3):
                    f = np.ones(8)
                    for bb in range(3):
                        f = f * (sgn[:, bb] / 2.0) if bb == a else f * ((1.0 + sgn[:, bb] * pt[bb]) / 2.0)
                    dN[:, a] = f
                dN = dN * (2.0 / h)
                Bm = np.zeros((6, 24))
                for node in range(8):
                    bx, by, bz = dN[node]
                    c = 3 * node
                    Bm[0, c], Bm[1, c + 1], Bm[2, c + 2] = bx, by, bz
                    Bm[3, c + 1], Bm[3, c + 2] = bz, by
                    Bm[4, c], Bm[4, c + 2] = bz, bx
                    Bm[5, c], Bm[5, c + 1] = by, bx
                K += Bm.T @ Dm @ Bm * jac
    return K, corner


def elasticity_3d(N, young=1.0, poisson=0.3, strip_zeros=False):
    """Linear elasticity on an N^3-node hex grid with the x=0 face clamped
    (config[4] at N=65, with strip_zeros=True -- SURVEY §8(d))."""
    if N < 2:
        raise ValueError("N must be at least 2")
    lam = young * poisson / ((1 + poisson) * (1 - 2 * poisson))
    mu = young / (2 * (1 + poisson))
    h = 1.0 / (N - 1)
    K, corner = _hex_stiffness(h, lam, mu)
    nodes = np.arange(N**3).reshape(N, N, N)
    xnode = np.unravel_index(np.arange(N**3), (N, N, N))[0]
    free_nodes = np.nonzero(xnode > 0)[0]
    free = np.full(N**3, -1, dtype=np.int64)
    free[free_nodes] = np.arange(free_nodes.size)
    ndof = 3 * free_nodes.size
    e = N - 1
    ex, ey, ez = (a.ravel() for a in np.meshgrid(range(e), range(e), range(e), indexing="ij"))
    conn = np.empty((ex.size, 8), dtype=np.int64)
    for a, (ci, cj, ck) in enumerate(corner.astype(int)):
        conn[:, a] = nodes[ex + ci, ey + cj, ez + ck]
    base = np.repeat(3 * free[conn], 3, axis=1)
    dofs = base + np.tile(np.arange(3), 8)[None, :]
    dofs[base < 0] = -1
    ii = np.repeat(dofs, 24, axis=1).ravel()
    jj = np.tile(dofs, (1, 24)).ravel()
    vv = np.tile(K.ravel(), ex.size)
    keep = (ii >= 0) & (jj >= 0) & (ii >= jj)
    A = SparseSpdMatrix.from_coo(ndof, ii[keep], jj[keep], vv[keep])
    if strip_zeros:
        A = strip_explicit_zeros(A)
    x, y, z = np.unravel_index(free_nodes, (N, N, N))
    xyz = np.column_stack([x, y, z]).astype(float) * h
    return A, Coordinates(np.repeat(xyz, 3, axis=0))


def batched_supernodes(nb=512, n=256, m=2048, true_rank=48, noise=1e-6, seed=0):
    """Config[1] inputs: per block i (draw order D then B, block by block, from
    default_rng(seed)): D = G G^T / n + I,  B = X Y + noise * Z with X m x true_rank,
    Y true_rank x n."""
    rng = np.random.default_rng(seed)
    D = np.empty((nb, n, n))
    B = np.empty((nb, m, n))
    for i in range(nb):
        G = rng.standard_normal((n, n))
        D[i] = G @ G.T / n + np.eye(n)
        B[i] = rng.standard_normal((m, true_rank)) @ rng.standard_normal((true_rank, n)) + noise * rng.standard_normal(
            (m, n)
        )
    return D, B


def config_problem(cfg, scale=None):
    """(A, coords) for config 0, 2, 3, 4 at full size (or `scale` grid points)."""
    if cfg == 0:
        return laplacian_2d(scale or 128)
    if cfg == 2:
        return laplacian_3d(scale or 64)
    if cfg == 3:
        return diffusion_fv_3d(scale or 96)
    if cfg == 4:
        return elasticity_3d(scale or 65, strip_zeros=True)
    raise ValueError(f"config {cfg} has no sparse problem")
