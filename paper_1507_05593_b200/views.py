"""Reference-shaped views of the device factor (rschol's factor object model).

rschol exposes the factor as `RankStructuredFactor.nodes` (one SupernodeFactor per
supernode), `.interior` (InteriorBlock per subdomain) and `.units` ((kind, obj)
tuples in sweep order) (reference factor.py:155-172, blocks.py:8-80,
interior.py:29-102, diagblocks.py:54-131).  The B200 factor keeps every block in
HBM; these classes present the same attributes and methods over it and copy a
block to the host only when it is read (numpy arrays, like the reference's).
"""

import numpy as np

__all__ = ["LowRankBlock", "SupernodeFactor", "DiagBlockNode", "DiagBlockTree", "InteriorBlock", "UpdateSource"]


def _host(t):
    return t.detach().cpu().numpy() if t is not None else None


class LowRankBlock:
    """V U^T with U orthonormal (blocks.py:8-45); V, U fetched from HBM on first use."""

    __slots__ = ("_dev", "_V", "_U", "_utu")

    def __init__(self, V, U=None):
        if U is None:  # from a device DevLR
            self._dev, self._V, self._U = V, None, None
        else:
            self._dev, self._V, self._U = None, np.ascontiguousarray(V, dtype=np.float64), \
                np.ascontiguousarray(U, dtype=np.float64)
        self._utu = None

    @property
    def V(self):
        if self._V is None:
            self._V = _host(self._dev.V)
        return self._V

    @property
    def U(self):
        if self._U is None:
            self._U = _host(self._dev.U)
        return self._U

    @property
    def rank(self):
        return self._dev.k if self._dev is not None else self._U.shape[1]

    @property
    def utu(self):
        if self._utu is None:
            self._utu = self.U.T @ self.U
        return self._utu

    def matmat(self, X):
        return self.V @ (self.U.T @ X)

    def rmatmat(self, X):
        return self.U @ (self.V.T @ X)

    def dense(self):
        return self.V @ self.U.T

    def scalars(self):
        return self.rank * (self._dev.V.shape[0] + self._dev.U.shape[0]) if self._dev is not None \
            else self.V.size + self.U.size


class DiagBlockNode:
    """Tree node of a hierarchical diagonal (diagblocks.py:30-51)."""

    __slots__ = ("s", "lo", "hi", "split", "left", "right", "parent")

    def __init__(self, nd):
        self.s, self.lo, self.hi, self.split = nd.s, nd.lo, nd.hi, nd.split
        self.left = self.right = self.parent = None

    @property
    def is_leaf(self):
        return self.split is None


class DiagBlockTree:
    """In-order block tree of one supernode's diagonal (diagblocks.py:54-131): dense
    lower leaves, LowRankBlock or dense couplings at internal nodes."""

    def __init__(self, shape, dev_tree=None):
        self.ncols, self.g0 = shape.ncols, shape.g0
        self._shape = shape
        self.nodes = {s: DiagBlockNode(nd) for s, nd in shape.nodes.items()}
        for s, nd in shape.nodes.items():
            v = self.nodes[s]
            v.left = self.nodes[nd.left.s] if nd.left is not None else None
            v.right = self.nodes[nd.right.s] if nd.right is not None else None
            v.parent = self.nodes[nd.parent.s] if nd.parent is not None else None
        self.root = self.nodes[shape.root.s]
        self._dev = dev_tree
        self._blocks = None

    @property
    def blocks(self):
        if self._blocks is None:
            from .factor import DevLR

            out = {}
            if self._dev is not None:
                for s, b in self._dev.blocks.items():
                    if self.nodes[s].is_leaf:
                        out[s] = np.tril(_host(b.L))
                    elif isinstance(b, DevLR):
                        out[s] = LowRankBlock(b)
                    else:
                        out[s] = _host(b)
            self._blocks = out
        return self._blocks

    @property
    def block_count(self):
        return len(self.nodes)

    def node(self, s):
        return self.nodes[s]

    def inorder_ids(self):
        return sorted(self.nodes)

    def leaf_ids(self):
        return [s for s in self.inorder_ids() if self.nodes[s].is_leaf]

    def path_above(self, s):
        return self._shape.path_above(s)

    def col_span(self, s):
        return self._shape.span(s)

    def assemble_dense(self):
        L = np.zeros((self.ncols, self.ncols))
        for s, nd in self.nodes.items():
            b = self.blocks[s]
            (r0, r1), (c0, c1) = self.col_span(s)
            L[r0:r1, c0:c1] = np.tril(b) if nd.is_leaf else (b.dense() if isinstance(b, LowRankBlock) else b)
        return L

    def stored_scalars(self):
        total = 0
        for s, nd in self.nodes.items():
            b = self.blocks.get(s)
            if b is None:
                continue
            if nd.is_leaf:
                k = nd.hi - nd.lo
                total += k * (k + 1) // 2
            elif isinstance(b, LowRankBlock):
                total += b.scalars()
            else:
                total += b.size
        return total


class SupernodeFactor:
    """Numeric content of one supernode (blocks.py:48-80)."""

    __slots__ = ("j", "c0", "c1", "rows", "_diag", "_off", "nrows_in_block", "interior_id", "_dev")

    def __init__(self, j, c0, c1, rows, diag=None, offdiag=None, nrows_in_block=None, interior_id=-1):
        self.j, self.c0, self.c1, self.rows = j, c0, c1, rows
        self._diag, self._off = diag, offdiag
        self.nrows_in_block, self.interior_id = nrows_in_block, interior_id
        self._dev = None

    @property
    def ncols(self):
        return self.c1 - self.c0

    @property
    def source_rows(self):
        return self.rows if self.nrows_in_block is None else self.rows[: self.nrows_in_block]

    @property
    def diag(self):
        if callable(self._diag):
            self._diag = self._diag()
        return self._diag

    @diag.setter
    def diag(self, v):
        self._diag = v

    @property
    def offdiag(self):
        if callable(self._off):
            self._off = self._off()
        return self._off

    @offdiag.setter
    def offdiag(self, v):
        self._off = v


class UpdateSource:
    """One left-looking update source (blocks.py:83-100): a factored supernode
    (kind "node") or an interior block (kind "interior"); order = first column."""

    __slots__ = ("kind", "rows", "order", "node", "block")

    def __init__(self, kind, rows, order, node=None, block=None):
        self.kind, self.rows, self.order, self.node, self.block = kind, rows, order, node, block

    def __lt__(self, other):
        return self.order < other.order


class InteriorBlock:
    """Exact factor of one subdomain (interior.py:29-102), over the device's dense
    L_B: members carry their diagonal triangles and in-block rows; `coupling` is the
    sparse A(off_rows, C_B)."""

    def __init__(self, block_id, unit, partition, B):
        self.id = block_id
        self.c0, self.c1 = unit.c0, unit.c1
        self.off_rows = unit.off_rows
        self._unit = unit
        self._part = partition
        self._B = B
        self._members = None
        self._coupling = None
        self._LB = None

    @property
    def ncols(self):
        return self.c1 - self.c0

    def _lb(self):
        if self._LB is None:
            self._LB = np.tril(_host(self._unit.diag.L))
        return self._LB

    @property
    def members(self):
        if self._members is None:
            out = []
            for j in self._unit.members:
                j0, j1 = self._part.cols(j)
                rows = self._part.rows[j]
                nib = int(np.searchsorted(rows, self.c1))

                def diag(j0=j0, j1=j1):
                    return self._lb()[j0 - self.c0:j1 - self.c0, j0 - self.c0:j1 - self.c0].copy()

                def off(j0=j0, j1=j1, rr=rows[:nib]):
                    return self._lb()[np.ix_(rr - self.c0, np.arange(j0 - self.c0, j1 - self.c0))]

                out.append(SupernodeFactor(j, j0, j1, rows, diag, off, nib, self.id))
            self._members = out
        return self._members

    @property
    def coupling(self):
        if self._coupling is None:
            full = self._B.to_csr_full()
            self._coupling = full[self.off_rows, self.c0:self.c1].tocsr()
        return self._coupling

    def solve(self, G, transpose=False):
        """Triangular solve with the in-block factor L_B (interior.py:50-75), on the
        device (the dense L_B and its inverse diagonal blocks live in HBM)."""
        from . import engine as E
        from .errors import ShapeMismatch

        G = np.asarray(G, dtype=np.float64)
        vec = G.ndim == 1
        X = G.reshape(-1, 1) if vec else G
        if X.shape[0] != self.ncols:
            raise ShapeMismatch(f"expected {self.ncols} rows, got {X.shape[0]}")
        Xd = E.to_dev(np.ascontiguousarray(X))
        self._unit.diag.solve(Xd, transpose=transpose)
        out = Xd.cpu().numpy()
        return out[:, 0] if vec else out

    def factor_rows(self, A, rows):
        """L(rows, C_B) = A(rows, C_B) L_B^{-T} (interior.py:77-82)."""
        rows = np.asarray(rows, dtype=np.int64)
        X = A.to_csr_full()[rows, self.c0:self.c1].toarray()
        return self.solve(X.T).T

    def multiply(self, A, R, C, G, transpose=False):
        """L(R, C_B) L(C, C_B)^T G (interior.py:84-95)."""
        from . import engine as E

        if transpose:
            R, C = C, R
        full = A.to_csr_full()
        AC = E.to_dev(full[np.asarray(C, dtype=np.int64), self.c0:self.c1].toarray())
        AR = E.to_dev(full[np.asarray(R, dtype=np.int64), self.c0:self.c1].toarray())
        Gd = E.to_dev(np.ascontiguousarray(np.asarray(G, dtype=np.float64).reshape(AC.shape[0], -1)))
        T = E.empty(self.ncols, Gd.shape[1])
        E.gemm(AC, Gd, T, transA=True)
        self._unit.diag.solve(T, transpose=False)
        self._unit.diag.solve(T, transpose=True)
        W = E.empty(AR.shape[0], Gd.shape[1])
        E.gemm(AR, T, W)
        out = W.cpu().numpy()
        return out[:, 0] if np.ndim(G) == 1 else out

    def stored_scalars(self):
        return self._unit._stored
