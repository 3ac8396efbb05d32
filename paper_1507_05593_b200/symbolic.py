"""Host symbolic phase: ordering, supernodes, row structures and the unit plan.

This is the input side of the hot path: it must reproduce the
reference's symbolic objects bit-for-bit, because kept ranks, seeds and every
index map downstream depend on them.  Pinned against the reference by
tests/test_symbolic.py (golden fixtures from tests/golden/make_golden.py).

  nested_dissection      ordering.py:277-368  (geometric / level bisection)
  partition_separator    ordering.py:525-554
  etree / postorder / column counts   symbolic.py:44-151 (C++: csrc/symbolic.cpp)
  form_supernodes        symbolic.py:189-277  (fundamental + CHOLMOD-tier amalgamation)
  compute_row_structures symbolic.py:280-306
  build_units            factor.py:512-535
  analyze                factor.py:657-695    (the symbolic half of factorize)
"""

import math
from collections import deque

import numpy as np
import scipy.sparse as sp

from . import _lib
from .errors import MissingCoordinates
from .problems import Coordinates
from .sparse import Permutation, SparseSpdMatrix, _permuted_lower

DEFAULT_LEAF_SIZE = 64
DIAG_TREE_FACTOR = 1
AMALG_TIERS = ((4, 1.0), (16, 0.8), (48, 0.1), (None, 0.05))


# ---------------------------------------------------------------------------
# separator tree


class SeparatorNode:
    """Dissection tree node in permuted indices: separator [lo, hi), whole subtree
    [subtree_lo, hi) (ordering.py:48-77)."""

    __slots__ = ("lo", "hi", "subtree_lo", "level", "left", "right")

    def __init__(self, lo, hi, subtree_lo, level, left=None, right=None):
        self.lo, self.hi, self.subtree_lo, self.level = lo, hi, subtree_lo, level
        self.left, self.right = left, right

    @property
    def is_separator(self):
        return self.left is not None

    @property
    def size(self):
        return self.hi - self.lo


class SeparatorTree:
    def __init__(self, n, root):
        self.n, self.root = n, root

    def separators(self, min_size=0):
        """Pre-order (left before right) separator nodes with >= min_size vertices."""
        stack = [self.root] if self.root is not None else []
        while stack:
            nd = stack.pop()
            if nd.is_separator:
                if nd.size >= min_size:
                    yield nd
                stack.append(nd.right)
                stack.append(nd.left)


class SplitTree:
    """Sizes-only recursive halving of a separator (ordering.py:497-522)."""

    __slots__ = ("size", "left", "right")

    def __init__(self, size, left=None, right=None):
        self.size, self.left, self.right = size, left, right

    @property
    def is_leaf(self):
        return self.left is None

    def leaf_sizes(self):
        return [self.size] if self.is_leaf else self.left.leaf_sizes() + self.right.leaf_sizes()

    @classmethod
    def natural(cls, size, tau_d):
        if size <= tau_d:
            return cls(size)
        half = (size + 1) // 2
        return cls(size, cls.natural(half, tau_d), cls.natural(size - half, tau_d))


def _adjacency(A):
    """Graph of A without the diagonal and stored zeros (C++ rsc_sym_full_csr)."""
    from .sparse import full_csr

    return full_csr(A, adjacency=True)


def _coords_xyz(coords, n):
    xyz = coords.xyz if hasattr(coords, "xyz") else np.asarray(coords, dtype=np.float64)
    if xyz.shape[0] != n:
        raise MissingCoordinates("need one coordinate row per matrix index")
    return xyz


class _Dissector:
    def __init__(self, A, leaf_size, xyz, method):
        self.n = A.n
        adj = _adjacency(A)
        self.indptr = adj.indptr.astype(np.int64)
        self.indices = adj.indices.astype(np.int64)
        self.deg = np.diff(self.indptr)
        self.xyz = xyz
        self._nd = None
        if method == "geometric" and xyz.ndim == 2 and xyz.shape[1] >= 1 and np.isfinite(xyz).all():
            from . import _lib

            self.xyz = np.ascontiguousarray(xyz, dtype=np.float64)
            self._nd = _lib.load().rsc_nd_split_geometric
        self.method = method
        self.leaf = leaf_size
        self.order = np.empty(self.n, dtype=np.int64)
        self.counter = 0
        self.mark = np.zeros(self.n, dtype=bool)   # side-1 membership scratch
        self.local = np.full(self.n, -1, dtype=np.int64)

    def emit(self, verts):
        k = len(verts)
        lo = self.counter
        self.order[lo:lo + k] = np.sort(verts)
        self.counter += k
        return lo, lo + k

    def _neighbors(self, vs):
        """Flattened neighbour lists of vs (CSR rows gathered in order)."""
        starts, cnt = self.indptr[vs], self.deg[vs]
        tot = int(cnt.sum())
        if tot == 0:
            return np.empty(0, np.int64), cnt
        first = np.cumsum(cnt) - cnt
        return self.indices[np.repeat(starts - first, cnt) + np.arange(tot)], cnt

    def boundary(self, side1, cand):
        """Members of `cand` (in order) with a neighbour in side1 (ordering.py:182-192)."""
        self.mark[side1] = True
        nb, cnt = self._neighbors(cand)
        hit = np.zeros(len(cand), dtype=bool)
        if nb.size:
            # per-candidate count of marked neighbours: segment sums over the CSR rows
            c = np.concatenate(([0], np.cumsum(self.mark[nb], dtype=np.int64)))
            ends = np.cumsum(cnt)
            hit = c[ends] > c[ends - cnt]
        self.mark[side1] = False
        return hit

    def split_by_order(self, verts, order):
        nv = len(verts)
        half = (nv + 1) // 2
        s1 = np.sort(order[:half])
        rest = np.sort(order[half:])
        hit = self.boundary(verts[s1], verts[rest])
        sep, s2 = rest[hit], rest[~hit]
        if s1.size == 0 or s2.size == 0:
            return None
        return verts[s1], verts[sep], verts[s2]

    def bisect_geometric(self, verts):
        if self._nd is not None:  # C++ split (csrc/nd.cpp), same result as below
            verts = np.ascontiguousarray(verts, dtype=np.int64)
            out = np.empty(len(verts), dtype=np.int64)
            cnt = np.empty(3, dtype=np.int64)
            rc = self._nd(len(verts), verts.ctypes.data, self.xyz.shape[1], self.xyz.ctypes.data,
                          self.indptr.ctypes.data, self.indices.ctypes.data, self.mark.ctypes.data,
                          out.ctypes.data, cnt.ctypes.data)
            if rc < 0:
                raise RuntimeError(f"rsc_nd_split_geometric failed ({rc})")
            if rc == 1:
                return None
            a, b = int(cnt[0]), int(cnt[0] + cnt[1])
            return out[:a], out[a:b], out[b:]
        pts = self.xyz[verts]
        axis = int(np.argmax(pts.max(axis=0) - pts.min(axis=0)))
        return self.split_by_order(verts, np.lexsort((verts, pts[:, axis])))

    # level-structure bisection (ordering.py:150-225), sequential BFS like the reference
    def _bfs(self, verts, start):
        level = np.full(len(verts), -1, dtype=np.int64)
        level[start] = 0
        dq = deque([start])
        ip, ix, loc = self.indptr, self.indices, self.local
        while dq:
            u = dq.popleft()
            g = verts[u]
            for w in ix[ip[g]:ip[g + 1]]:
                lw = loc[w]
                if lw >= 0 and level[lw] < 0:
                    level[lw] = level[u] + 1
                    dq.append(lw)
        return level

    def bisect_level(self, verts):
        r, ecc = 0, -1
        for _ in range(8):  # pseudo-peripheral start (ordering.py:167-179)
            level = self._bfs(verts, r)
            far = int(level.max())
            if far <= ecc:
                break
            ecc = far
            r = int(np.nonzero(level == far)[0][0])
        nlev = int(level.max()) + 1
        if nlev < 2:
            return None
        sizes = np.bincount(level, minlength=nlev)
        cum = np.concatenate(([0], np.cumsum(sizes)))
        total = len(verts)
        best_l, best_bal = 1, None
        for l in range(1, nlev):
            bal = abs(cum[l] - (total - cum[l] - sizes[l]))
            if best_bal is None or bal < best_bal:
                best_l, best_bal = l, bal
        s1 = np.nonzero(level < best_l)[0]
        rest = np.nonzero(level >= best_l)[0]
        cand = np.nonzero(level == best_l)[0]
        hit = self.boundary(verts[s1], verts[cand])
        sep = cand[hit]
        in_sep = np.zeros(len(verts), dtype=bool)
        in_sep[sep] = True
        s2 = rest[~in_sep[rest]]
        if s1.size == 0 or s2.size == 0:
            return None
        return verts[s1], verts[sep], verts[s2]

    def components(self, verts):
        loc = self.local
        loc[verts] = np.arange(len(verts))
        seen = np.zeros(len(verts), dtype=bool)
        comps = []
        ip, ix = self.indptr, self.indices
        for s in range(len(verts)):
            if seen[s]:
                continue
            comp = [s]
            seen[s] = True
            dq = deque([s])
            while dq:
                u = dq.popleft()
                g = verts[u]
                for w in ix[ip[g]:ip[g + 1]]:
                    lw = loc[w]
                    if lw >= 0 and not seen[lw]:
                        seen[lw] = True
                        comp.append(lw)
                        dq.append(lw)
            comps.append(verts[np.sort(np.asarray(comp))])
        loc[verts] = -1
        return comps

    def bisect(self, verts):
        if self.method == "geometric":
            return self.bisect_geometric(verts)
        if self.method == "level":
            self.local[verts] = np.arange(len(verts))
            try:
                return self.bisect_level(verts)
            finally:
                self.local[verts] = -1
        raise NotImplementedError(f"dissection method {self.method!r}")

    def dissect(self, verts, level, connected):
        sub_lo = self.counter
        if len(verts) <= self.leaf:
            lo, hi = self.emit(verts)
            return SeparatorNode(lo, hi, sub_lo, level)
        if not connected and self.method != "geometric":
            comps = self.components(verts)
            if len(comps) > 1:
                comps.sort(key=lambda c: (-len(c), c[0]))
                g1, g2, s1, s2 = [], [], 0, 0
                for c in comps:
                    if s1 <= s2:
                        g1.append(c)
                        s1 += len(c)
                    else:
                        g2.append(c)
                        s2 += len(c)
                left = self.dissect(np.sort(np.concatenate(g1)), level + 1, len(g1) == 1)
                right = self.dissect(np.sort(np.concatenate(g2)), level + 1, len(g2) == 1)
                lo = self.counter
                return SeparatorNode(lo, lo, sub_lo, level, left, right)
        split = self.bisect(verts)
        if split is None:
            lo, hi = self.emit(verts)
            return SeparatorNode(lo, hi, sub_lo, level)
        side1, sep, side2 = split
        left = self.dissect(side1, level + 1, False)
        right = self.dissect(side2, level + 1, False)
        lo, hi = self.emit(sep)
        return SeparatorNode(lo, hi, sub_lo, level, left, right)


def nested_dissection(A, leaf_size=DEFAULT_LEAF_SIZE, coords=None, method="auto"):
    """(Permutation, SeparatorTree): separators numbered after both subdomains,
    left before right (ordering.py:277-368)."""
    if leaf_size < 1:
        raise ValueError("leaf_size must be >= 1")
    if method == "auto":
        method = "geometric" if coords is not None else "level"
    xyz = None
    if method == "geometric":
        if coords is None:
            raise MissingCoordinates("geometric dissection needs coordinates")
        xyz = _coords_xyz(coords, A.n)
    if A.n == 0:
        return Permutation.identity(0), SeparatorTree(0, None)
    d = _Dissector(A, leaf_size, xyz, method)
    if d._nd is not None:
        return _nd_geometric_native(d)
    import sys

    sys.setrecursionlimit(max(sys.getrecursionlimit(), 10000))
    root = d.dissect(np.arange(A.n, dtype=np.int64), 0, False)
    fwd = np.empty(A.n, dtype=np.int64)
    fwd[d.order] = np.arange(A.n, dtype=np.int64)
    return Permutation(fwd), SeparatorTree(A.n, root)


def _nd_geometric_native(d):
    """The geometric recursion in one C++ call (rsc_nd_geometric, subtrees on host
    threads); the same order and tree as _Dissector.dissect."""
    n = d.n
    order = np.empty(n, dtype=np.int64)
    root = np.zeros(1, dtype=np.int64)
    # node capacity: a generous estimate first (the tree has ~4n/leaf nodes), the
    # worst case 2n+1 only if that overflows (-3)
    for cap in (min(2 * n + 1, 8 * (n // max(d.leaf, 1)) + 4096), 2 * n + 1):
        nodes = np.empty((6, cap), dtype=np.int64)
        cnt = _lib.load().rsc_nd_geometric(n, d.xyz.shape[1], d.xyz.ctypes.data, d.indptr.ctypes.data,
                                           d.indices.ctypes.data, d.leaf, order.ctypes.data, cap,
                                           *[nodes[i].ctypes.data for i in range(6)], root.ctypes.data)
        if cnt != -3:
            break
    if cnt < 0:
        raise RuntimeError(f"rsc_nd_geometric failed ({cnt})")
    lo, hi, sub, lev, left, right = (nodes[i, :cnt].tolist() for i in range(6))
    objs = [None] * cnt
    # children are created before their parent (post-order ids within a subtree) is
    # not guaranteed across threads: build by explicit stack from the root
    stack = [(int(root[0]), False)]
    while stack:
        i, done = stack.pop()
        if left[i] < 0:
            objs[i] = SeparatorNode(lo[i], hi[i], sub[i], lev[i])
        elif done:
            objs[i] = SeparatorNode(lo[i], hi[i], sub[i], lev[i], objs[left[i]], objs[right[i]])
        else:
            stack.append((i, True))
            stack.append((right[i], False))
            stack.append((left[i], False))
    fwd = np.empty(n, dtype=np.int64)
    fwd[order] = np.arange(n, dtype=np.int64)
    return Permutation(fwd), SeparatorTree(n, objs[int(root[0])])


def partition_separator(coords, C, tau_d):
    """Recursive longest-axis halving of separator indices C (ordering.py:525-554).
    Returns (reordered indices, SplitTree)."""
    C = np.asarray(C, dtype=np.int64)
    if coords is None:
        raise MissingCoordinates("partition_separator needs coordinates")
    xyz = coords.xyz if hasattr(coords, "xyz") else np.asarray(coords)
    if C.size and C.max() >= xyz.shape[0]:
        raise MissingCoordinates("coordinates missing for some separator indices")

    def rec(idx):
        if len(idx) <= tau_d:
            return idx, SplitTree(len(idx))
        pts = xyz[idx]
        axis = int(np.argmax(pts.max(axis=0) - pts.min(axis=0)))
        idx = idx[np.lexsort((idx, pts[:, axis]))]
        half = (len(idx) + 1) // 2
        li, lt = rec(idx[:half])
        ri, rt = rec(idx[half:])
        return np.concatenate([li, ri]), SplitTree(len(idx), lt, rt)

    return rec(C)


# ---------------------------------------------------------------------------
# elimination tree, supernodes, structures


def etree_postorder_counts(B, septree=None):
    """(parent, post, counts) of the permuted lower-CSC matrix (C++ host kernels; the
    etree's rows of disjoint ND subtrees on host threads when the tree is given)."""
    lib = _lib.load()
    n = B.n
    cp = np.ascontiguousarray(B.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(B.row_idx, dtype=np.int64)
    parent = np.empty(n, dtype=np.int64)
    post = np.empty(n, dtype=np.int64)
    counts = np.empty(n, dtype=np.int64)
    rc = 1
    if septree is not None and septree.root is not None:
        rg = _subtree_col_ranges(septree)
        if rg.size:
            rc = lib.rsc_sym_etree_par(n, cp.ctypes.data, ri.ctypes.data, rg.size // 2, rg.ctypes.data,
                                       parent.ctypes.data)
            if rc < 0:
                raise RuntimeError(f"rsc_sym_etree_par failed ({rc})")
    if rc != 0:
        _lib.check(lib.rsc_sym_etree(n, cp.ctypes.data, ri.ctypes.data, parent.ctypes.data), "rsc_sym_etree")
    _lib.check(lib.rsc_sym_postorder(n, parent.ctypes.data, post.ctypes.data), "rsc_sym_postorder")
    _lib.check(lib.rsc_sym_colcounts(n, cp.ctypes.data, ri.ctypes.data, parent.ctypes.data, post.ctypes.data,
                                     counts.ctypes.data), "rsc_sym_colcounts")
    return parent, post, counts


class SupernodePartition:
    """starts[M+1], is_separator[M], rows[j] (sorted int64), interior_id[M]
    (symbolic.py:154-186)."""

    def __init__(self, n, starts, is_separator):
        self.n = n
        self.starts = np.asarray(starts, dtype=np.int64)
        self.is_separator = np.asarray(is_separator, dtype=bool)
        self.rows = []
        self.interior_id = np.full(self.count, -1, dtype=np.int64)

    @property
    def count(self):
        return self.starts.shape[0] - 1

    def cols(self, j):
        return int(self.starts[j]), int(self.starts[j + 1])

    def ncols(self, j):
        return int(self.starts[j + 1] - self.starts[j])

    def supernode_of(self, col):
        return int(np.searchsorted(self.starts, col, side="right") - 1)


def _fundamental(lo, hi, parent, counts):
    if hi <= lo:
        return [lo, hi]
    j = np.arange(lo + 1, hi)
    brk = (parent[j - 1] != j) | (counts[j - 1] != counts[j] + 1)
    return [lo] + j[brk].tolist() + [hi]


def _amalgamate(bounds, parent, counts):
    """Relaxed amalgamation of one gap of fundamental supernodes (C++:
    rsc_sym_amalgamate; the same merge rule and IEEE fraction as the reference
    loop, symbolic.py:244-277)."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    nb = len(b) - 1
    if nb <= 0:
        return []
    par = np.ascontiguousarray(parent, dtype=np.int64)
    cnt = np.ascontiguousarray(counts, dtype=np.int64)
    tw = np.array([-1 if w is None else w for w, _ in AMALG_TIERS], dtype=np.int64)
    tb = np.array([bd for _, bd in AMALG_TIERS], dtype=np.float64)
    out = np.empty(nb, dtype=np.int64)
    k = _lib.load().rsc_sym_amalgamate(nb, b.ctypes.data, par.ctypes.data, cnt.ctypes.data, len(tw),
                                       tw.ctypes.data, tb.ctypes.data, out.ctypes.data)
    if k < 0:
        raise RuntimeError(f"rsc_sym_amalgamate failed ({k})")
    return out[:k].tolist()


def form_supernodes(n, parent, counts, septree, tau_o, relax=True):
    """Separators with >= tau_o vertices become one supernode each; the gaps are
    fundamental supernodes relaxed by amalgamation (symbolic.py:244-277)."""
    seps = sorted((nd.lo, nd.hi) for nd in septree.separators(min_size=max(tau_o, 1)))
    starts, flags, pos = [], [], 0
    for lo, hi in seps + [(n, n)]:
        if pos < lo:
            b = _fundamental(pos, lo, parent, counts)
            gap = _amalgamate(b, parent, counts) if relax else b[:-1]
            starts.extend(gap)
            flags.extend([False] * len(gap))
        if hi > lo:
            starts.append(lo)
            flags.append(True)
        pos = hi
    starts.append(n)
    return SupernodePartition(n, starts, flags)


def _subtree_front(septree, target=64):
    """~target disjoint ND subtrees: the largest subtree split first."""
    front = [septree.root]
    while len(front) < target:
        big = max((nd for nd in front if nd.is_separator), key=lambda nd: nd.hi - nd.subtree_lo, default=None)
        if big is None:
            break
        front.remove(big)
        front += [big.left, big.right]
    return front


def _subtree_col_ranges(septree, target=64):
    """Column ranges [subtree_lo, hi) of disjoint ND subtrees (flattened pairs)."""
    out = []
    for nd in _subtree_front(septree, target):
        if nd.hi - nd.subtree_lo >= 2:
            out += [nd.subtree_lo, nd.hi]
    return np.asarray(sorted(out), dtype=np.int64).reshape(-1)


def _subtree_ranges(part, septree, target=64):
    """Supernode ranges of disjoint ND subtrees (about `target` of them, largest
    first split) for the threaded row-structure sweep: a subtree's pieces only go to
    its own supernodes or to ancestor separators after it."""
    if septree.root is None:
        return np.zeros(0, dtype=np.int64)
    front = [septree.root]
    while len(front) < target:
        big = max((nd for nd in front if nd.is_separator), key=lambda nd: nd.hi - nd.subtree_lo, default=None)
        if big is None:
            break
        front.remove(big)
        front += [big.left, big.right]
    st = part.starts
    out = []
    for nd in front:
        lo, hi = nd.subtree_lo, nd.hi
        if hi - lo < 2:
            continue
        j0 = int(np.searchsorted(st, lo, side="left"))
        j1 = int(np.searchsorted(st, hi, side="left"))
        if j0 < j1 and st[j0] == lo and j1 < st.size and st[j1] == hi:
            out += [j0, j1]
    return np.asarray(sorted(out), dtype=np.int64)


def compute_row_structures(B, part, septree=None):
    """R_j = A's below-block rows of C_j  U  children's rows beyond their parent's
    columns (symbolic.py:280-306); the merge sweep runs in C++
    (rsc_sym_rows_compute / rsc_sym_rows_fetch), R_j are views of one array."""
    import ctypes

    M = part.count
    lib = _lib.load()
    st = np.ascontiguousarray(part.starts, dtype=np.int64)
    cp = np.ascontiguousarray(B.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(B.row_idx, dtype=np.int64)
    total = ctypes.c_longlong(0)
    rg = _subtree_ranges(part, septree) if septree is not None else np.zeros(0, dtype=np.int64)
    h = lib.rsc_sym_rows_compute_par(M, st.ctypes.data, cp.ctypes.data, ri.ctypes.data, rg.size // 2,
                                     rg.ctypes.data, ctypes.byref(total))
    ptr = np.empty(M + 1, dtype=np.int64)
    allrows = np.empty(max(total.value, 1), dtype=np.int64)
    _lib.check(lib.rsc_sym_rows_fetch(h, ptr.ctypes.data, allrows.ctypes.data), "rsc_sym_rows_fetch")
    rows = [allrows[ptr[j]:ptr[j + 1]] for j in range(M)]
    part.rows = rows
    part.rows_flat = (ptr, allrows)
    return rows


def build_units(septree, part, tau_o, interior_enabled):
    """Processing order (factor.py:512-535): compressed separators as ("node", j)
    in post-order, every maximal subtree below them as ("interior", [members])."""
    if not interior_enabled:
        return [("node", j) for j in range(part.count)]
    units = []

    def walk(nd):
        if nd is None:
            return
        if nd.is_separator and nd.size >= tau_o:
            walk(nd.left)
            walk(nd.right)
            units.append(("node", part.supernode_of(nd.lo)))
        elif nd.hi > nd.subtree_lo:
            j0 = part.supernode_of(nd.subtree_lo)
            j1 = part.supernode_of(nd.hi - 1)
            units.append(("interior", list(range(j0, j1 + 1))))

    walk(septree.root)
    return units


class SymbolicPlan:
    """Everything the numeric phase consumes (the output of factorize's host half)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def analyze(A, tau_o, tau_d, interior_blocks=True, coords=None):
    """Ordering + symbolic analysis exactly as factorize does it (factor.py:657-695).

    Returns a SymbolicPlan with perm, B (permuted matrix), septree, partition,
    sep_splits {supernode: SplitTree}, units, and the ordering/symbolic times."""
    import time
    import warnings

    if coords is not None and not hasattr(coords, "xyz"):
        coords = Coordinates(np.asarray(coords, dtype=np.float64))
    t0 = time.perf_counter()
    perm1, septree = nested_dissection(A, DEFAULT_LEAF_SIZE, coords=coords)
    sep_nodes = [nd for nd in septree.separators() if nd.size >= tau_o]
    tree_nodes = [nd for nd in sep_nodes if nd.size > DIAG_TREE_FACTOR * tau_d]
    fwd = perm1.forward.copy()
    splits_by_range = {}
    if tree_nodes:
        if coords is None:
            raise NotImplementedError(
                "diagonal trees without coordinates need spectral coordinates (ordering.py:466-490); "
                "pass coords")
        for nd in tree_nodes:
            orig = perm1.inverse[nd.lo:nd.hi]
            try:
                reordered, split = partition_separator(coords, orig, tau_d)
            except MissingCoordinates:
                reordered, split = orig, SplitTree.natural(nd.size, tau_d)
                warnings.warn("separator ordered naturally (no usable coordinates)")
            fwd[reordered] = np.arange(nd.lo, nd.hi, dtype=np.int64)
            splits_by_range[(nd.lo, nd.hi)] = split
    perm = Permutation(fwd)
    r, c, b_from_a = _permuted_lower(A, perm.forward)
    col_ptr = np.zeros(A.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(c, minlength=A.n), out=col_ptr[1:])
    B = SparseSpdMatrix(A.n, col_ptr, r, A.values[b_from_a], validate=False)
    t1 = time.perf_counter()
    parent, post, counts = etree_postorder_counts(B, septree)
    part = form_supernodes(B.n, parent, counts, septree, tau_o)
    compute_row_structures(B, part, septree)
    sep_splits = {part.supernode_of(lo): s for (lo, hi), s in splits_by_range.items()}
    units = build_units(septree, part, tau_o, interior_blocks)
    t2 = time.perf_counter()
    return SymbolicPlan(perm=perm, B=B, septree=septree, partition=part, sep_splits=sep_splits, units=units,
                        b_from_a=b_from_a, parent=parent, counts=counts, t_ordering=t1 - t0, t_symbolic=t2 - t1)


def block_rank(m, n, alpha, p):
    """min(ceil(alpha sqrt(k) log2 k) + p, k), k = min(m, n) (factor.py:313-321)."""
    k = min(int(m), int(n))
    if k <= 0:
        return 0
    return min(int(math.ceil(alpha * math.sqrt(k) * math.log2(k))) + int(p), k)
