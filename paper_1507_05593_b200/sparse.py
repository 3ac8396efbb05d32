"""Host sparse containers of the rschol API (reference pkg/src/rschol/sparse.py).

`SparseSpdMatrix` keeps the reference's storage contract (lower-triangle CSC,
0-based, strictly increasing rows, positive diagonal, read-only arrays) and
adds a cached device copy of the full symmetric CSR (`device_csr()`), which is
what the GPU SpMV and block extraction read.  Any object exposing
`n, col_ptr, row_idx, values` (e.g. the reference's own matrix class) is
accepted by `as_spd()`.
"""

import numpy as np
import scipy.sparse as sp

from .errors import DimensionMismatch, MissingDiagonal, NonPositiveDiagonal, ParseError

__all__ = ["SparseSpdMatrix", "Permutation", "permute_symmetric", "as_spd", "strip_explicit_zeros"]


class SparseSpdMatrix:
    """Lower-triangle CSC storage of an SPD matrix (sparse.py:33-130)."""

    def __init__(self, n, col_ptr, row_idx, values, validate=True):
        self.n = int(n)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        if validate:
            self._validate()
        for a in (self.col_ptr, self.row_idx, self.values):
            a.setflags(write=False)
        self._csr_full = None
        self._csc_lower = None
        self._dev = None

    def _validate(self):
        n = self.n
        cp, ri, v = self.col_ptr, self.row_idx, self.values
        if cp.shape != (n + 1,):
            raise DimensionMismatch("col_ptr must have length n+1")
        if n and np.any(np.diff(cp) < 0):
            raise ParseError("col_ptr must be nondecreasing")
        if ri.shape[0] != v.shape[0]:
            raise DimensionMismatch("row_idx and values must have equal length")
        if n == 0:
            return
        counts = np.diff(cp)
        empty = np.nonzero(counts == 0)[0]
        if empty.size:
            raise MissingDiagonal(f"diagonal entry ({empty[0]},{empty[0]}) missing")
        first = ri[cp[:-1]]
        bad = np.nonzero(first != np.arange(n))[0]
        if bad.size:
            raise MissingDiagonal(f"diagonal entry ({bad[0]},{bad[0]}) missing")
        # strictly increasing within each column: successive entries of one column
        same_col = np.ones(ri.shape[0], dtype=bool)
        same_col[cp[1:-1]] = False
        same_col[0] = False
        d = np.diff(ri)
        if np.any(d[same_col[1:]] <= 0):
            col = int(np.searchsorted(cp, np.nonzero((d <= 0) & same_col[1:])[0][0] + 1, side="right") - 1)
            raise ParseError(f"row indices not strictly increasing in column {col}")
        if ri.size and ri.max() >= n:
            raise ParseError("row index out of range")
        dv = v[cp[:-1]]
        nonpos = np.nonzero(dv <= 0.0)[0]
        if nonpos.size:
            j = int(nonpos[0])
            raise NonPositiveDiagonal(f"a[{j},{j}] = {dv[j]} <= 0")

    @property
    def nnz_lower(self):
        return int(self.values.shape[0])

    def diagonal(self):
        return self.values[self.col_ptr[:-1]].copy()

    def to_csc_lower(self):
        if self._csc_lower is None:
            self._csc_lower = sp.csc_matrix((self.values, self.row_idx, self.col_ptr), shape=(self.n, self.n))
        return self._csc_lower

    def to_csr_full(self):
        """Full symmetric CSR (both triangles, stored zeros dropped), cached, indices
        sorted -- one O(nnz) C++ pass (rsc_sym_full_csr) instead of scipy's
        add + convert + sort."""
        if self._csr_full is None:
            self._csr_full = full_csr(self, adjacency=False)
        return self._csr_full

    def device_csr(self):
        """Device copy of the full CSR (uploaded once, cached like _csr_full)."""
        if self._dev is None:
            from . import engine

            self._dev = engine.DeviceCSR.from_scipy(self.to_csr_full())
        return self._dev

    def dense(self):
        return self.to_csr_full().toarray()

    def matvec(self, x):
        return self.to_csr_full() @ x

    @classmethod
    def from_coo(cls, n, rows, cols, vals):
        """Lower-triangle triples (upper ones mirrored, duplicates summed)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        lo_r = np.maximum(rows, cols)
        lo_c = np.minimum(rows, cols)
        m = sp.coo_matrix((vals, (lo_r, lo_c)), shape=(n, n)).tocsc()
        m.sum_duplicates()
        m.sort_indices()
        return cls(n, m.indptr, m.indices, m.data)

    @classmethod
    def from_dense(cls, M):
        M = np.asarray(M, dtype=np.float64)
        r, c = np.nonzero(np.tril(M))
        return cls.from_coo(M.shape[0], r, c, M[r, c])

    def __repr__(self):
        return f"SparseSpdMatrix(n={self.n}, nnz_lower={self.nnz_lower})"


def as_spd(A):
    """Accept our matrix or any duck-typed lower-CSC SPD matrix (e.g. rschol's)."""
    if isinstance(A, SparseSpdMatrix):
        return A
    return SparseSpdMatrix(A.n, A.col_ptr, A.row_idx, A.values, validate=False)


def strip_explicit_zeros(A):
    """Drop stored zeros (mandatory input normalization for the elasticity
    generator); keeps the diagonal."""
    keep = A.values != 0.0
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.col_ptr))
    return SparseSpdMatrix.from_coo(A.n, A.row_idx[keep], cols[keep], A.values[keep])


class Permutation:
    """Bijection with forward (old->new) and inverse maps (sparse.py:133-168)."""

    def __init__(self, forward):
        self.forward = np.ascontiguousarray(forward, dtype=np.int64)
        n = self.forward.shape[0]
        if n and (self.forward.min() < 0 or self.forward.max() >= n):
            raise DimensionMismatch("forward map is not a bijection on 0..n-1")
        inv = np.full(n, -1, dtype=np.int64)
        inv[self.forward] = np.arange(n, dtype=np.int64)
        if n and np.any(inv < 0):
            raise DimensionMismatch("forward map has repeated images")
        self.inverse = inv
        self.forward.setflags(write=False)
        self.inverse.setflags(write=False)

    @property
    def n(self):
        return self.forward.shape[0]

    @classmethod
    def identity(cls, n):
        return cls(np.arange(n, dtype=np.int64))

    def compose(self, other):
        return Permutation(other.forward[self.forward])

    def __eq__(self, other):
        return isinstance(other, Permutation) and np.array_equal(self.forward, other.forward)

    def __repr__(self):
        return f"Permutation(n={self.n})"


def full_csr(A, adjacency=False):
    """scipy CSR of the symmetric full matrix (adjacency=True: without the diagonal)."""
    from . import _lib

    n = A.n
    cp = np.ascontiguousarray(A.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.row_idx, dtype=np.int64)
    va = np.ascontiguousarray(A.values, dtype=np.float64)
    cap = 2 * ri.size
    indptr = np.empty(n + 1, dtype=np.int64)
    indices = np.empty(max(cap, 1), dtype=np.int64)
    data = np.empty(max(cap, 1), dtype=np.float64)
    nnz = _lib.load().rsc_sym_full_csr(n, cp.ctypes.data, ri.ctypes.data, va.ctypes.data, int(adjacency),
                                       indptr.ctypes.data, indices.ctypes.data, data.ctypes.data)
    if nnz < 0:
        raise RuntimeError(f"rsc_sym_full_csr failed ({nnz})")
    it = np.int32 if nnz < 2**31 - 1 else np.int64
    m = sp.csr_matrix((data[:nnz], indices[:nnz].astype(it), indptr.astype(it)), shape=(n, n))
    m.has_sorted_indices = True
    return m


def _permuted_lower(A, p):
    """Lower-storage (row, col) of every entry of A under p, sorted by (col, row),
    and the source position of each: one counting pass by column plus a per-column
    row sort in C++ (rsc_sym_permute_lower) instead of a 2-key lexsort."""
    from . import _lib

    n = A.n
    nnz = int(A.row_idx.size)
    r = np.empty(nnz, dtype=np.int64)
    c = np.empty(nnz, dtype=np.int64)
    order = np.empty(nnz, dtype=np.int64)
    if n == 0 or nnz == 0:
        return r, c, np.arange(nnz, dtype=np.int64)
    cp = np.ascontiguousarray(A.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.row_idx, dtype=np.int64)
    pp = np.ascontiguousarray(p, dtype=np.int64)
    _lib.check(_lib.load().rsc_sym_permute_lower(n, cp.ctypes.data, ri.ctypes.data, pp.ctypes.data, r.ctypes.data,
                                                 c.ctypes.data, order.ctypes.data), "rsc_sym_permute_lower")
    return r, c, order


def permute_symmetric(A, perm):
    """B[p(i), p(j)] = A[i, j], kept in lower storage (sparse.py:171-189)."""
    if perm.n != A.n:
        raise DimensionMismatch(f"permutation size {perm.n} != matrix size {A.n}")
    r, c, order = _permuted_lower(A, perm.forward)
    v = A.values[order]
    col_ptr = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(c, minlength=A.n), out=col_ptr[1:])
    return SparseSpdMatrix(A.n, col_ptr, r, v, validate=False)
