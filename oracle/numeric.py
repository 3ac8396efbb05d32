"""CPU restatement of the reference numeric factorization, preconditioner apply
and PCG -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows /root/reference/pkg/src/rschol line by line in behaviour (not in text):
  factorize / restart loop       factor.py:642-740
  _numeric_pass + buckets        factor.py:538-639
  _assemble_schur                factor.py:372-399
  off_diagonal_multiply[_trans]  factor.py:427-483
  approximate_off_diagonal       factor.py:486-505
  interior blocks                interior.py:29-156
  diagonal trees (Algs. 4-6)     diagblocks.py:132-370
  apply (_forward/_backward)     factor.py:175-218
  stored_scalars / dense_lower   factor.py:222-267
  pcg                            pcg.py:64-135
The symbolic plan (ordering, supernodes, units) comes from
paper_1507_05593_b200.symbolic.analyze, which tests/test_symbolic.py pins
bit-exactly against the reference's own symbolic output.
"""

import math
import time
from dataclasses import dataclass, field

import numpy as np

from .kernels import OracleIndefinite, block_seed, chol, gauss, orth, trisolve

DENSE_FALLBACK = 0.75

# Algorithmic work census: when COUNT is a dict, every operation of
# the reference algorithm adds its flops under a category; _CAT is the category of
# the enclosing compression (off-diagonal / diagonal-tree sketch products).
COUNT = None
_CAT = ["off_sketch"]


def _f(cat, val):
    if COUNT is not None:
        COUNT[cat] = COUNT.get(cat, 0.0) + float(val)


def _nnzL(blk):
    return sum((m.c1 - m.c0) * (m.c1 - m.c0 + 1) // 2 + (m.c1 - m.c0) * (m.nib or 0) for m in blk.members)


def _nnz(full, rows, c0, c1):
    return full[np.asarray(rows, dtype=np.int64), c0:c1].nnz


@dataclass
class Config:
    tau_o: float = 400
    tau_d: int = 256
    alpha_o: float = 1.0
    alpha_d: float = 0.5
    oversample: int = 8
    power_iters: int = 1
    seed: int = 0
    interior_blocks: bool = True
    max_restarts: int = 10
    alpha_d_growth: float = 1.25


class TooManyRestarts(Exception):
    pass


def block_rank(m, n, alpha, p):
    k = min(int(m), int(n))
    if k <= 0:
        return 0
    return min(int(math.ceil(alpha * math.sqrt(k) * math.log2(k))) + int(p), k)


class LR:
    """V U^T with cached U^T U (blocks.py:8-45)."""

    def __init__(self, V, U):
        self.V = np.ascontiguousarray(V)
        self.U = np.ascontiguousarray(U)
        self.utu = self.U.T @ self.U

    def matmat(self, X):
        return self.V @ (self.U.T @ X)

    def rmatmat(self, X):
        return self.U @ (self.V.T @ X)

    def dense(self):
        return self.V @ self.U.T


def eff(off, sl, cat=None):
    """eff_rows (blocks.py:103-113): V[sl] (U^T U) for a low-rank block -- a GEMM the
    reference executes on every use (counted under `cat`)."""
    if isinstance(off, LR):
        out = off.V[sl] @ off.utu
        if cat is not None:
            _f(cat, 2.0 * out.shape[0] * off.V.shape[1] ** 2)
        return out
    return off[sl]


def raw(off, sl):
    return off.V[sl] if isinstance(off, LR) else off[sl]


class Node:
    def __init__(self, j, c0, c1, rows):
        self.j, self.c0, self.c1, self.rows = j, c0, c1, rows
        self.diag = None
        self.off = None
        self.nib = None
        self.interior_id = -1

    @property
    def source_rows(self):
        return self.rows if self.nib is None else self.rows[: self.nib]


class Src:
    def __init__(self, kind, rows, order, node=None, blk=None):
        self.kind, self.rows, self.order, self.node, self.blk = kind, rows, order, node, blk


# ---------------------------------------------------------------------------
# interior blocks (interior.py)


class Interior:
    def __init__(self, bid, c0, c1, members, off_rows, coupling):
        self.id, self.c0, self.c1 = bid, c0, c1
        self.members, self.off_rows, self.coupling = members, off_rows, coupling

    def solve(self, G, transpose=False):
        X = np.array(G, dtype=np.float64, copy=True)
        vec = X.ndim == 1
        if vec:
            X = X.reshape(-1, 1)
        if not transpose:
            for m in self.members:
                a, b = m.c0 - self.c0, m.c1 - self.c0
                Y = trisolve(m.diag, X[a:b])
                X[a:b] = Y
                if m.nib:
                    X[m.rows[: m.nib] - self.c0] -= m.off @ Y
        else:
            for m in reversed(self.members):
                a, b = m.c0 - self.c0, m.c1 - self.c0
                Y = X[a:b]
                if m.nib:
                    Y = Y - m.off.T @ X[m.rows[: m.nib] - self.c0]
                X[a:b] = trisolve(m.diag, Y, transpose=True)
        return X[:, 0] if vec else X

    def factor_rows(self, full, rows):
        X = full[np.asarray(rows, dtype=np.int64), self.c0 : self.c1].toarray()
        return self.solve(X.T).T

    def multiply(self, full, R, C, G, transpose=False):
        if transpose:
            R, C = C, R
        if COUNT is not None:
            k = np.shape(G)[1] if np.ndim(G) == 2 else 1
            _f(_CAT[-1], 2.0 * k * (_nnz(full, C, self.c0, self.c1) + _nnz(full, R, self.c0, self.c1))
               + 4.0 * _nnzL(self) * k)
        T = full[np.asarray(C, dtype=np.int64), self.c0 : self.c1].T @ G
        T = self.solve(self.solve(T), transpose=True)
        return full[np.asarray(R, dtype=np.int64), self.c0 : self.c1] @ T

    def stored(self):
        return self.coupling.nnz + sum(
            (m.c1 - m.c0) * (m.c1 - m.c0 + 1) // 2 + (m.c1 - m.c0) * (m.nib or 0) for m in self.members)


def factor_interior(full, part, ids, bid):
    c0, c1 = int(part.starts[ids[0]]), int(part.starts[ids[-1] + 1])
    members, by_id, buckets = [], {}, {}
    for j in ids:
        j0, j1 = part.cols(j)
        rows = part.rows[j]
        nib = int(np.searchsorted(rows, c1))
        UD = full[j0:j1, j0:j1].toarray()
        UO = full[rows[:nib], j0:j1].toarray() if nib else np.zeros((0, j1 - j0))
        for k in sorted(buckets.get(j, ())):
            s = by_id[k]
            rk = s.rows[: s.nib]
            lo, hi = np.searchsorted(rk, (j0, j1))
            cpos = rk[lo:hi] - j0
            Bd = s.off[lo:hi]
            UD[np.ix_(cpos, cpos)] -= Bd @ Bd.T
            if hi < rk.shape[0] and nib:
                UO[np.ix_(np.searchsorted(rows, rk[hi:]), cpos)] -= s.off[hi:] @ Bd.T
            if hi < rk.shape[0]:
                buckets.setdefault(part.supernode_of(int(rk[hi])), []).append(k)
        if COUNT is not None:
            ncj = j1 - j0
            _f("potrf_trsm", ncj**3 / 3.0 + nib * ncj * ncj + nib * nib * ncj)
        nd = Node(j, j0, j1, rows)
        nd.diag = chol(UD)
        nd.off = trisolve(nd.diag, UO.T).T if nib else UO
        nd.nib = nib
        nd.interior_id = bid
        members.append(nd)
        by_id[j] = nd
        if nib:
            buckets.setdefault(part.supernode_of(int(rows[0])), []).append(j)
    tails = [m.rows[m.nib :] for m in members if m.rows[m.nib :].size]
    off_rows = np.unique(np.concatenate(tails)) if tails else np.empty(0, np.int64)
    coupling = full[off_rows, c0:c1].tocsr() if off_rows.size else full[:0, c0:c1].tocsr()
    return Interior(bid, c0, c1, members, off_rows, coupling)


# ---------------------------------------------------------------------------
# diagonal trees (diagblocks.py)


class TNode:
    __slots__ = ("s", "lo", "hi", "split", "left", "right", "parent")

    def __init__(self, s, lo, hi, split=None):
        self.s, self.lo, self.hi, self.split = s, lo, hi, split
        self.left = self.right = self.parent = None

    @property
    def leaf(self):
        return self.split is None


class Tree:
    def __init__(self, ncols, g0, split):
        self.ncols, self.g0 = ncols, g0
        self.nodes, self.blocks = {}, {}
        cnt = [0]

        def rec(piece, lo):
            if piece.is_leaf:
                cnt[0] += 1
                nd = TNode(cnt[0], lo, lo + piece.size)
                self.nodes[nd.s] = nd
                return nd
            l = rec(piece.left, lo)
            cnt[0] += 1
            nd = TNode(cnt[0], lo, lo + piece.size, lo + piece.left.size)
            self.nodes[nd.s] = nd
            r = rec(piece.right, lo + piece.left.size)
            nd.left, nd.right = l, r
            l.parent = r.parent = nd
            return nd

        self.root = rec(split, 0)

    def path_above(self, s):
        out, nd = [], self.nodes[s].parent
        while nd is not None:
            if nd.s < s:
                out.append(nd.s)
            nd = nd.parent
        return out

    def span(self, s):
        nd = self.nodes[s]
        if nd.leaf:
            return (nd.lo, nd.hi), (nd.lo, nd.hi)
        return (nd.split, nd.hi), (nd.lo, nd.split)

    def dense(self):
        L = np.zeros((self.ncols, self.ncols))
        for s, nd in self.nodes.items():
            (r0, r1), (c0, c1) = self.span(s)
            b = self.blocks[s]
            L[r0:r1, c0:c1] = np.tril(b) if nd.leaf else (b.dense() if isinstance(b, LR) else b)
        return L

    def stored(self):
        t = 0
        for s, nd in self.nodes.items():
            b = self.blocks.get(s)
            if b is None:
                continue
            if nd.leaf:
                k = nd.hi - nd.lo
                t += k * (k + 1) // 2
            elif isinstance(b, LR):
                t += b.V.size + b.U.size
            else:
                t += b.size
        return t


def _couple(b, X, transpose):
    if isinstance(b, LR):
        return b.rmatmat(X) if transpose else b.matmat(X)
    return b.T @ X if transpose else b @ X


def _tsolve(tree, G, transpose, nd):
    if nd.leaf:
        return trisolve(tree.blocks[nd.s], G, transpose=transpose)
    k = nd.split - nd.lo
    G1, G2 = G[:k], G[k:]
    b = tree.blocks[nd.s]
    if transpose:
        X2 = _tsolve(tree, G2, True, nd.right)
        X1 = _tsolve(tree, G1 - _couple(b, X2, True), True, nd.left)
    else:
        X1 = _tsolve(tree, G1, False, nd.left)
        X2 = _tsolve(tree, G2 - _couple(b, X1, False), False, nd.right)
    return np.concatenate([X1, X2], axis=0)


def diag_solve(node, G, transpose=False, s=None):
    G = np.asarray(G, dtype=np.float64)
    vec = G.ndim == 1
    X = G.reshape(-1, 1) if vec else G
    if isinstance(node.diag, Tree):
        root = node.diag.root if s is None else node.diag.nodes[s]
        out = _tsolve(node.diag, X, transpose, root)
    else:
        out = trisolve(node.diag, X, transpose=transpose)
    return out[:, 0] if vec else out


def _win_update(U, src, rw, cw, full):
    (r0, r1), (c0, c1) = rw, cw
    if src.kind == "interior":
        Yc = src.blk.factor_rows(full, np.arange(c0, c1))
        Yr = Yc if (r0, r1) == (c0, c1) else src.blk.factor_rows(full, np.arange(r0, r1))
        nl = _nnzL(src.blk) if COUNT is not None else 0
        _f("leaf_interior", 2.0 * nl * ((c1 - c0) + (0 if (r0, r1) == (c0, c1) else (r1 - r0)))
           + 2.0 * (r1 - r0) * (c1 - c0) * (src.blk.c1 - src.blk.c0))
        U -= Yr @ Yc.T
        return
    rows = src.rows
    clo, chi = np.searchsorted(rows, (c0, c1))
    rlo, rhi = np.searchsorted(rows, (r0, r1))
    if clo == chi or rlo == rhi:
        return
    off = src.node.off
    w = off.V.shape[1] if isinstance(off, LR) else off.shape[1]
    _f("leaf_syrk", 2.0 * (rhi - rlo) * (chi - clo) * w)
    U[np.ix_(rows[rlo:rhi] - r0, rows[clo:chi] - c0)] -= eff(off, slice(rlo, rhi), "leaf_syrk") @ raw(off, slice(clo, chi)).T


def _win_multiply(W, src, rw, cw, G, transpose, full):
    (r0, r1), (c0, c1) = rw, cw
    if src.kind == "interior":
        if transpose:
            W -= src.blk.multiply(full, np.arange(c0, c1), np.arange(r0, r1), G)
        else:
            W -= src.blk.multiply(full, np.arange(r0, r1), np.arange(c0, c1), G)
        return
    rows = src.rows
    clo, chi = np.searchsorted(rows, (c0, c1))
    rlo, rhi = np.searchsorted(rows, (r0, r1))
    if clo == chi or rlo == rhi:
        return
    off = src.node.off
    w = off.V.shape[1] if isinstance(off, LR) else off.shape[1]
    _f(_CAT[-1], 2.0 * ((rhi - rlo) + (chi - clo)) * w * G.shape[1])
    if transpose:
        T = eff(off, slice(rlo, rhi), _CAT[-1]).T @ G[rows[rlo:rhi] - r0]
        W[rows[clo:chi] - c0] -= raw(off, slice(clo, chi)) @ T
    else:
        T = raw(off, slice(clo, chi)).T @ G[rows[clo:chi] - c0]
        W[rows[rlo:rhi] - r0] -= eff(off, slice(rlo, rhi), _CAT[-1]) @ T


def _path_pair(tree, p, rspan, cspan, cat=None):
    base = tree.nodes[p].split
    b = tree.blocks[p]
    return eff(b, slice(rspan[0] - base, rspan[1] - base), cat), raw(b, slice(cspan[0] - base, cspan[1] - base))


def factor_leaf(full, node, s, srcs):
    tree = node.diag
    lf = tree.nodes[s]
    g0, g1 = tree.g0 + lf.lo, tree.g0 + lf.hi
    U = full[g0:g1, g0:g1].toarray()
    for src in srcs:
        _win_update(U, src, (g0, g1), (g0, g1), full)
    for p in tree.path_above(s):
        P, Q = _path_pair(tree, p, (lf.lo, lf.hi), (lf.lo, lf.hi), "leaf_path")
        _f("leaf_path", 2.0 * P.shape[0] * Q.shape[0] * P.shape[1])
        U -= P @ Q.T
    _f("potrf_trsm", (g1 - g0) ** 3 / 3.0)
    return chol(U)


def diag_multiply(full, node, s, G, transpose, srcs):
    tree = node.diag
    blk = tree.nodes[s]
    (r0, r1), (c0, c1) = tree.span(s)
    gr, gc = (tree.g0 + r0, tree.g0 + r1), (tree.g0 + c0, tree.g0 + c1)
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    _f("sketch_diag_solve", (c1 - c0) ** 2 * G.shape[1])
    _f(_CAT[-1], 2.0 * full[gr[0]:gr[1], gc[0]:gc[1]].nnz * G.shape[1])
    if not transpose:
        G1 = diag_solve(node, G, transpose=True, s=blk.left.s)
        W = full[gr[0] : gr[1], gc[0] : gc[1]] @ G1
        for src in srcs:
            _win_multiply(W, src, gr, gc, G1, False, full)
        for p in tree.path_above(s):
            P, Q = _path_pair(tree, p, (r0, r1), (c0, c1), _CAT[-1])
            _f(_CAT[-1], 2.0 * (P.shape[0] + Q.shape[0]) * P.shape[1] * G1.shape[1])
            W -= P @ (Q.T @ G1)
        return W
    W = full[gr[0] : gr[1], gc[0] : gc[1]].T @ G
    for src in srcs:
        _win_multiply(W, src, gr, gc, G, True, full)
    for p in tree.path_above(s):
        P, Q = _path_pair(tree, p, (r0, r1), (c0, c1), _CAT[-1])
        _f(_CAT[-1], 2.0 * (P.shape[0] + Q.shape[0]) * P.shape[1] * G.shape[1])
        W -= Q @ (P.T @ G)
    return diag_solve(node, W, transpose=False, s=blk.left.s)


def approx_diag_block(full, node, s, rank, q, seed, srcs):
    (r0, r1), (c0, c1) = node.diag.span(s)
    rank = min(rank, r1 - r0, c1 - c0)
    _CAT.append("diag_sketch")
    try:
        G = diag_multiply(full, node, s, gauss(r1 - r0, rank, seed), True, srcs)
        for _ in range(q):
            G = diag_multiply(full, node, s, diag_multiply(full, node, s, G, False, srcs), True, srcs)
        _f("qrcp", 4.0 * G.shape[0] * G.shape[1] ** 2)
        U = orth(G)
        return LR(diag_multiply(full, node, s, U, False, srcs), U)
    finally:
        _CAT.pop()


# ---------------------------------------------------------------------------
# supernode assembly and implicit products (factor.py)


def assemble_schur(full, node, R, srcs, want_off=True):
    c0, c1 = node.c0, node.c1
    want_off = want_off and R.size > 0
    UD = full[c0:c1, c0:c1].toarray()
    UO = full[R, c0:c1].toarray() if want_off else np.zeros((0, c1 - c0))
    for src in srcs:
        if src.kind == "interior":
            Yc = src.blk.factor_rows(full, np.arange(c0, c1))
            if COUNT is not None:
                nl, nb, nc = _nnzL(src.blk), src.blk.c1 - src.blk.c0, c1 - c0
                _f("interior_solve", 2.0 * nl * (nc + (R.size if want_off else 0)))
                _f("interior_gemm", 2.0 * nc * nc * nb + (2.0 * R.size * nc * nb if want_off else 0.0))
            UD -= Yc @ Yc.T
            if want_off:
                UO -= src.blk.factor_rows(full, R) @ Yc.T
            continue
        rows = src.rows
        lo, hi = np.searchsorted(rows, (c0, c1))
        if lo == hi:
            continue
        cpos = rows[lo:hi] - c0
        off = src.node.off
        Q = raw(off, slice(lo, hi))
        _f("node_syrk_gemm", 2.0 * (hi - lo) ** 2 * Q.shape[1]
           + (2.0 * (rows.shape[0] - hi) * (hi - lo) * Q.shape[1] if (hi < rows.shape[0] and want_off) else 0.0))
        UD[np.ix_(cpos, cpos)] -= eff(off, slice(lo, hi), "node_syrk_gemm") @ Q.T
        if hi < rows.shape[0] and want_off:
            UO[np.ix_(np.searchsorted(R, rows[hi:]), cpos)] -= eff(off, slice(hi, None), "node_syrk_gemm") @ Q.T
    return UD, UO


def off_mul(full, node, G, srcs):
    c0, c1, R = node.c0, node.c1, node.rows
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    if R.size == 0 or G.shape[1] == 0:
        return np.zeros((R.size, G.shape[1]))
    _f("sketch_diag_solve", (c1 - c0) ** 2 * G.shape[1])
    G1 = diag_solve(node, G, transpose=True)
    W = full[R, c0:c1] @ G1
    _f(_CAT[-1], 2.0 * W.shape[1] * full[R, c0:c1].nnz if COUNT is not None else 0.0)
    for src in srcs:
        if src.kind == "interior":
            W -= src.blk.multiply(full, R, np.arange(c0, c1), G1)
            continue
        rows = src.rows
        lo, hi = np.searchsorted(rows, (c0, c1))
        if lo == hi or hi == rows.shape[0]:
            continue
        off = src.node.off
        _f(_CAT[-1], 2.0 * (rows.shape[0] - lo) * raw(off, slice(lo, hi)).shape[1] * G1.shape[1])
        T = raw(off, slice(lo, hi)).T @ G1[rows[lo:hi] - c0]
        W[np.searchsorted(R, rows[hi:])] -= eff(off, slice(hi, None), _CAT[-1]) @ T
    return W


def off_mul_t(full, node, G, srcs):
    c0, c1, R = node.c0, node.c1, node.rows
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    if G.shape[1] == 0:
        return np.zeros((c1 - c0, 0))
    W = full[R, c0:c1].T @ G
    _f(_CAT[-1], 2.0 * G.shape[1] * full[R, c0:c1].nnz if COUNT is not None else 0.0)
    _f("sketch_diag_solve", (c1 - c0) ** 2 * G.shape[1])
    for src in srcs:
        if src.kind == "interior":
            W -= src.blk.multiply(full, np.arange(c0, c1), R, G)
            continue
        rows = src.rows
        lo, hi = np.searchsorted(rows, (c0, c1))
        if lo == hi or hi == rows.shape[0]:
            continue
        off = src.node.off
        _f(_CAT[-1], 2.0 * (rows.shape[0] - lo) * raw(off, slice(lo, hi)).shape[1] * G.shape[1])
        T = eff(off, slice(hi, None), _CAT[-1]).T @ G[np.searchsorted(R, rows[hi:])]
        W[rows[lo:hi] - c0] -= raw(off, slice(lo, hi)) @ T
    return diag_solve(node, W, transpose=False)


def approx_off(full, node, rank, q, seed, srcs):
    R = node.rows
    rank = min(rank, R.size, node.c1 - node.c0)
    G = off_mul_t(full, node, gauss(R.size, rank, seed), srcs)
    for _ in range(q):
        G = off_mul_t(full, node, off_mul(full, node, G, srcs), srcs)
    _f("qrcp", 4.0 * G.shape[0] * G.shape[1] ** 2)
    U = orth(G)
    return LR(off_mul(full, node, U, srcs), U)


# ---------------------------------------------------------------------------
# factor container + apply


class Factor:
    def __init__(self, n, plan, cfg):
        self.n, self.plan, self.cfg = n, plan, cfg
        self.perm = plan.perm
        self.nodes, self.interior, self.units = [], [], []
        self.stats = {}
        self.ranks = {}  # ("off", j) / ("diag", j, s) -> kept rank

    def apply(self, r):
        y = np.asarray(r, dtype=np.float64)[self.perm.inverse].copy()
        for kind, o in self.units:
            if kind == "interior":
                w = o.solve(y[o.c0 : o.c1])
                y[o.c0 : o.c1] = w
                if o.off_rows.size:
                    y[o.off_rows] -= o.coupling @ o.solve(w, transpose=True)
            else:
                w = diag_solve(o, y[o.c0 : o.c1])
                y[o.c0 : o.c1] = w
                if o.rows.size and o.off is not None:
                    y[o.rows] -= o.off.matmat(w) if isinstance(o.off, LR) else o.off @ w
        for kind, o in reversed(self.units):
            if kind == "interior":
                rhs = y[o.c0 : o.c1]
                if o.off_rows.size:
                    rhs = rhs - o.solve(o.coupling.T @ y[o.off_rows])
                y[o.c0 : o.c1] = o.solve(rhs, transpose=True)
            else:
                rhs = y[o.c0 : o.c1]
                if o.rows.size and o.off is not None:
                    rhs = rhs - (o.off.rmatmat(y[o.rows]) if isinstance(o.off, LR) else o.off.T @ y[o.rows])
                y[o.c0 : o.c1] = diag_solve(o, rhs, transpose=True)
        return y[self.perm.forward]

    __call__ = apply

    def stored_scalars(self):
        t = 0
        for kind, o in self.units:
            if kind == "interior":
                t += o.stored()
            else:
                nc = o.c1 - o.c0
                t += o.diag.stored() if isinstance(o.diag, Tree) else nc * (nc + 1) // 2
                if isinstance(o.off, LR):
                    t += o.off.V.size + o.off.U.size
                elif o.off is not None:
                    t += o.off.size
        return t

    def dense_lower(self):
        L = np.zeros((self.n, self.n))
        for kind, o in self.units:
            if kind == "interior":
                for m in o.members:
                    L[m.c0 : m.c1, m.c0 : m.c1] = np.tril(m.diag)
                    if m.nib:
                        L[m.rows[: m.nib], m.c0 : m.c1] = m.off
                if o.off_rows.size:
                    L[o.off_rows, o.c0 : o.c1] = o.solve(o.coupling.T.toarray()).T
            else:
                L[o.c0 : o.c1, o.c0 : o.c1] = o.diag.dense() if isinstance(o.diag, Tree) else np.tril(o.diag)
                if o.rows.size and o.off is not None:
                    L[o.rows, o.c0 : o.c1] = o.off.dense() if isinstance(o.off, LR) else o.off
        return L


def numeric_pass(full, F, cfg, alpha_d, counters, on_unit=None):
    plan = F.plan
    part = plan.partition
    M = part.count
    nodes = [None] * M
    F.nodes, F.interior, F.units, F.ranks = nodes, [], [], {}
    buckets = [[] for _ in range(M)]

    def file(src):
        if src.rows.size:
            buckets[part.supernode_of(int(src.rows[0]))].append(src)

    for u, (kind, payload) in enumerate(plan.units):
        if on_unit is not None:  # bench hook: per-unit timestamps / BLAS thread policy
            on_unit(u, kind, payload)
        if kind == "interior":
            blk = factor_interior(full, part, payload, len(F.interior))
            F.interior.append(blk)
            for m in blk.members:
                nodes[m.j] = m
            F.units.append(("interior", blk))
            if blk.off_rows.size:
                file(Src("interior", blk.off_rows, blk.c0, blk=blk))
            continue
        j = payload
        c0, c1 = part.cols(j)
        nc = c1 - c0
        R = part.rows[j]
        srcs = sorted(buckets[j], key=lambda s: s.order)
        buckets[j] = ()
        compress = bool(part.is_separator[j])
        node = Node(j, c0, c1, R)
        nodes[j] = node
        tree_diag = compress and j in plan.sep_splits
        r_off = block_rank(R.size, nc, cfg.alpha_o, cfg.oversample)
        compress_off = bool(compress and R.size and r_off < DENSE_FALLBACK * min(R.size, nc))
        UO = None
        if tree_diag:
            counters["diag_trees"] += 1
            tree = Tree(nc, c0, plan.sep_splits[j])
            node.diag = tree
            for s in sorted(tree.nodes):
                tn = tree.nodes[s]
                if tn.leaf:
                    tree.blocks[s] = factor_leaf(full, node, s, srcs)
                    continue
                nr, ncl = tn.hi - tn.split, tn.split - tn.lo
                r = block_rank(nr, ncl, alpha_d, cfg.oversample)
                if r >= DENSE_FALLBACK * min(nr, ncl):
                    _CAT.append("diag_sketch")
                    tree.blocks[s] = diag_multiply(full, node, s, np.eye(ncl), False, srcs)
                    _CAT.pop()
                    counters["dense_fallback"] += 1
                else:
                    tree.blocks[s] = approx_diag_block(full, node, s, r, cfg.power_iters,
                                                       block_seed(cfg.seed, 1, j, s), srcs)
                    F.ranks[("diag", j, s)] = tree.blocks[s].U.shape[1]
                    counters["compressed_diag"] += 1
        else:
            UD, UO = assemble_schur(full, node, R, srcs, want_off=not compress_off)
            _f("potrf_trsm", nc**3 / 3.0)
            node.diag = chol(UD)
        if R.size == 0:
            node.off = None
        elif compress_off:
            node.off = approx_off(full, node, r_off, cfg.power_iters, block_seed(cfg.seed, 0, j), srcs)
            F.ranks[("off", j)] = node.off.U.shape[1]
            counters["compressed_off"] += 1
        else:
            if compress:
                counters["dense_fallback"] += 1
            if tree_diag:
                _, UO2 = assemble_schur(full, node, R, srcs)
                node.off = diag_solve(node, UO2.T).T if UO2.shape[0] else UO2
            else:
                node.off = trisolve(node.diag, UO.T).T
            _f("potrf_trsm", R.size * nc * nc)
        F.units.append(("node", node))
        for src in srcs:
            hi = np.searchsorted(src.rows, c1)
            if hi < src.rows.shape[0]:
                buckets[part.supernode_of(int(src.rows[hi]))].append(src)
        if R.size:
            file(Src("node", R, c0, node=node))


def factorize(A, cfg=None, coords=None, plan=None, on_unit=None):
    """Oracle factorization (factor.py:642-740) on the product's symbolic plan."""
    from paper_1507_05593_b200.symbolic import analyze

    cfg = cfg or Config()
    t0 = time.perf_counter()
    if plan is None:
        plan = analyze(A, cfg.tau_o, cfg.tau_d, cfg.interior_blocks, coords=coords)
    t1 = time.perf_counter()
    full = plan.B.to_csr_full()
    F = Factor(A.n, plan, cfg)
    alpha_d = cfg.alpha_d
    hist = [alpha_d]
    restarts = 0
    while True:
        counters = {"diag_trees": 0, "compressed_off": 0, "compressed_diag": 0, "dense_fallback": 0}
        try:
            numeric_pass(full, F, cfg, alpha_d, counters, on_unit)
            break
        except OracleIndefinite:
            if counters["diag_trees"] == 0:
                raise
            restarts += 1
            if restarts > cfg.max_restarts:
                raise TooManyRestarts(f"alpha_d reached {alpha_d:g}") from None
            alpha_d *= cfg.alpha_d_growth
            hist.append(alpha_d)
    t2 = time.perf_counter()
    F.stats = dict(counters, restarts=restarts, alpha_d_history=hist, alpha_d_final=alpha_d,
                   t_plan=t1 - t0, t_numeric=t2 - t1, stored_scalars=F.stored_scalars())
    return F


@dataclass
class Report:
    iterations: int = 0
    converged: bool = False
    relative_residual: float = np.inf
    relative_residual_history: list = field(default_factory=list)


def pcg(A, b, M=None, tol=1e-5, max_iter=None, x0=None):
    """pcg.py:64-135."""
    b = np.asarray(b, dtype=np.float64)
    n = A.n
    max_iter = 10 * n if max_iter is None else max_iter
    op = A.to_csr_full()
    apply_m = (lambda r: r.copy()) if M is None else (M.apply if hasattr(M, "apply") else M)
    nb = float(np.linalg.norm(b))
    rep = Report()
    if nb == 0.0:
        rep.converged, rep.relative_residual, rep.relative_residual_history = True, 0.0, [0.0]
        return np.zeros(n), rep
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    r = b - op @ x if x0 is not None else b.copy()
    hist = [float(np.linalg.norm(r)) / nb]
    z = apply_m(r)
    p = z.copy()
    rz = float(r @ z)
    it, conv, relres = 0, False, hist[0]
    while it < max_iter:
        Ap = op @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise RuntimeError(f"breakdown pAp={pAp}")
        a = rz / pAp
        x += a * p
        r -= a * Ap
        it += 1
        relres = float(np.linalg.norm(r)) / nb
        hist.append(relres)
        if relres <= tol:
            tr = b - op @ x
            trel = float(np.linalg.norm(tr)) / nb
            if trel <= tol:
                conv, relres = True, trel
                break
            r, relres, hist[-1] = tr, trel, trel
        z = apply_m(r)
        rzn = float(r @ z)
        p = z + (rzn / rz) * p
        rz = rzn
    rep.iterations, rep.converged, rep.relative_residual, rep.relative_residual_history = it, conv, relres, hist
    return x, rep
