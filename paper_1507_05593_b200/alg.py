"""The reference's algorithm-level API (rschol/__init__.py:34-58) on the device factor.

rschol exposes every step of the numeric sweep as a public function acting on a
(partial) factor: Alg. 1 (factor_supernode), Alg. 2 and its mirror
(off_diagonal_multiply[_trans]), Alg. 3 (approximate_off_diagonal), Alg. 4-6 on
diagonal trees (diagonal_solve, diagonal_multiply, factor_diagonal,
approximate_diagonal_block), interior blocks (factor_interior_block) and source
discovery (collect_sources).  Here they act on a RankStructuredFactor produced by
`factorize`: node j's operands are its update sources in that factor (exactly the
descendants the reference passes as `sources`), and every product, solve, POTRF
and pivoted QR runs through the same device kernels as the sweep
(numeric.LevelPass, librsc_b200.so).  Host numpy arrays in and out, as in the
reference.  `A` is the permuted matrix the factor was built from (what the
reference's numeric pass passes, factor.py:686-702); `sources`, when given, must
be the node's reference update sources (they are checked, not re-derived).
"""

import numpy as np

from . import engine as E
from .errors import IndefiniteError, ShapeMismatch
from .factor import DeviceTree, DevLR, _Indefinite, _raw_eff
from .numeric import LevelPass, diag_solve_many
from .views import DiagBlockTree, InteriorBlock, LowRankBlock, UpdateSource

__all__ = ["collect_sources", "factor_supernode", "off_diagonal_multiply", "off_diagonal_multiply_trans",
           "approximate_off_diagonal", "diagonal_solve", "diagonal_multiply", "factor_diagonal",
           "approximate_diagonal_block", "factor_interior_block", "build_diag_tree", "block_rank"]


class _Engine(LevelPass):
    """A LevelPass bound to a finished factor: the sweep's batched primitives with
    the factor's panels registered as update sources (no pass-wide sketches)."""

    def __init__(self, F):
        plan = F.plan
        # NumericPass.__init__ without the pass's device sketches
        self.np, self.sym, self.cfg, self.alpha_d = plan, plan.sym, F.config, F.stats.alpha_d_final or \
            F.config.alpha_d
        self.counters = {"diag_trees": 0, "compressed_off": 0, "compressed_diag": 0, "dense_fallback": 0}
        self.units, self.src_panel, self.ranks, self.flops = [], {}, {}, 0.0
        self.P, self.S = E.Arena(1 << 22), E.Arena(1 << 22)
        self.ibuf = E.zeros(64, dtype=E.I32)
        self.ipos = 0
        self.pending = []
        self.sketches = None
        ns = len(plan.sources)
        self.s_raw = np.zeros(ns, dtype=np.uint64)
        self.s_eff = np.zeros(ns, dtype=np.uint64)
        self.s_ld = np.ones(ns, dtype=np.int64)
        self.s_w = np.zeros(ns, dtype=np.int64)
        self.idx_base = np.uint64(plan.idx.dev.data_ptr())
        self._uslot, self._deferred, self._final, self._wterms, self._price = {}, [], None, [], {}
        self.split = None
        self.F = F
        self.by_j = {}
        for un in F.dunits:
            sid = plan.unit_source.get(un.u)
            if un.kind == "node":
                self.by_j[un.j] = un
                if sid is not None and un.off is not None:
                    self._set_source(sid, *_raw_eff(un.off))
            elif sid is not None:
                self._set_source(sid, un.off, un.off)

    def _ints(self, n):
        if self.ipos + n > self.ibuf.numel():  # calls are independent: grow and restart
            self.ibuf, self.ipos = E.zeros(max(64, 2 * n), dtype=E.I32), 0
        t = self.ibuf[self.ipos:self.ipos + n]
        self.ipos += n
        return t

    def node(self, j):
        un = self.by_j.get(int(j))
        if un is None:
            raise ShapeMismatch(f"supernode {j} is not a separator node of this factor")
        return un

    def check(self):
        """Raise IndefiniteError for a failed POTRF of this call (kernels.py:35-36)."""
        if not self.pending:
            return
        info = self.ibuf[: self.ipos].cpu().numpy()
        for off, cnt, *_ in self.pending:
            v = info[off:off + cnt]
            bad = np.nonzero(v)[0]
            if bad.size:
                self.pending = []
                raise IndefiniteError(int(v[bad[0]]) - 1)
        self.pending = []


def _engine(L):
    eng = getattr(L, "_alg_engine", None)
    if eng is None:
        eng = L._alg_engine = _Engine(L)
    # every call copies its results to the host before returning: the engine's
    # scratch, output arena and info words start over
    eng.S.reset()
    eng.P.reset()
    eng.ipos, eng.pending, eng._uslot, eng._price = 0, [], {}, {}
    return eng


def _dev2(G, rows):
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    if G.shape[0] != rows:
        raise ShapeMismatch(f"G must have {rows} rows, got {G.shape[0]}")
    return E.to_dev(np.ascontiguousarray(G))


def _check_sources(eng, j, sources):
    if sources is None:
        return
    want = {int(eng.np.sources[p.s].order) for p in eng.np.targets[j]}
    got = {int(s.order) for s in sources}
    if want != got:
        raise ValueError("sources do not match the node's update sources in this factor")


def block_rank(m, n, alpha, oversample):
    """factor.py:313-321."""
    from .symbolic import block_rank as br

    return br(m, n, alpha, oversample)


def collect_sources(L, j):
    """Update sources of supernode j, ascending by first column (factor.py:333-365):
    the factored supernodes and interior blocks whose rows reach into C_j."""
    plan = L.plan
    nodes = L.nodes
    out = []
    pairs = plan.targets.get(int(j))
    if pairs is None:  # an interior member: its in-block descendants
        blk = L.interior[int(L.partition.interior_id[j])] if L.partition.interior_id[j] >= 0 else None
        c0, c1 = L.partition.cols(j)
        if blk is not None:
            for m in blk.members:
                if m.j >= j:
                    break
                lo, hi = np.searchsorted(m.source_rows, (c0, c1))
                if lo < hi:
                    out.append(UpdateSource("node", m.source_rows, m.c0, node=m))
        return out
    interiors = {b.c0: b for b in L.interior}
    for p in pairs:
        src = plan.sources[p.s]
        if src.kind == "interior":
            out.append(UpdateSource("interior", src.rows, src.c0, block=interiors.get(src.c0)))
        else:
            k = int(L.partition.supernode_of(src.c0))
            out.append(UpdateSource("node", src.rows, src.c0, node=nodes[k]))
    out.sort(key=lambda s: s.order)
    return out


def factor_supernode(A, j, L, sources=None):
    """Alg. 1 for supernode j against the factor's sources (factor.py:402-415):
    (L_D, L_O) = (chol(U_D), U_O L_D^{-T}) with the dense Schur blocks of
    _assemble_schur (factor.py:372-399).  IndefiniteError propagates."""
    eng = _engine(L)
    node = eng.node(j)
    _check_sources(eng, j, sources)
    (UD, UO), = eng.assemble_many([(node, True, True)])
    tri, = eng._potrf_many([(UD, node.u)])
    eng.check()
    LD = np.tril(UD.cpu().numpy())
    if UO is None or UO.numel() == 0:
        return LD, np.zeros((node.rows.size, node.ncols))
    E.trsm_batched("right", 1, [tri.L.data_ptr()], [node.ncols], [E.ld(tri.L)], [tri.Dinv.data_ptr()],
                   [UO.data_ptr()], [UO.shape[0]], [E.ld(UO)])
    return LD, UO.cpu().numpy()


def off_diagonal_multiply(A, j, L, G, sources=None):
    """Alg. 2: L_O(j) G without forming L_O(j) (factor.py:427-456)."""
    eng = _engine(L)
    node = eng.node(j)
    _check_sources(eng, j, sources)
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    if node.rows.size == 0 or G.shape[1] == 0:
        if G.shape[0] != node.ncols:
            raise ShapeMismatch(f"G must have {node.ncols} rows, got {G.shape[0]}")
        return np.zeros((node.rows.size, G.shape[1]))
    W, = eng.off_mul_many([node], [_dev2(G, node.ncols)])
    return W.cpu().numpy()


def off_diagonal_multiply_trans(A, j, L, G, sources=None):
    """The mirror L_O(j)^T G (factor.py:459-483)."""
    eng = _engine(L)
    node = eng.node(j)
    _check_sources(eng, j, sources)
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    if G.shape[1] == 0:
        return np.zeros((node.ncols, 0))
    W, = eng.off_mul_t_many([node], [_dev2(G, node.rows.size)])
    return W.cpu().numpy()


def approximate_off_diagonal(A, j, L, rank, power_iters=1, seed=0, sources=None):
    """Alg. 3: randomized compression of L_O(j) (factor.py:486-505): reference PCG64
    sketch from `seed`, (1 + 2q) implicit products, pivoted QR with the reference
    cutoff, V = L_O U."""
    from .kernels import gaussian_matrix

    eng = _engine(L)
    node = eng.node(j)
    _check_sources(eng, j, sources)
    R = node.rows
    rank = min(rank, R.size, node.ncols)
    G, = eng.off_mul_t_many([node], [E.to_dev(gaussian_matrix(R.size, rank, seed))])
    for _ in range(power_iters):
        G, = eng.off_mul_t_many([node], eng.off_mul_many([node], [G]))
    U, = eng._orth_many([G])
    rk = int(eng.ibuf[eng._uslot.pop(id(U))].item())
    U = U[:, :rk].contiguous()
    if rk == 0:
        return LowRankBlock(np.zeros((R.size, 0)), np.zeros((node.ncols, 0)))
    V, = eng.off_mul_many([node], [U])
    return LowRankBlock(V.cpu().numpy(), U.cpu().numpy())


def _tree(eng, j):
    node = eng.node(j)
    if not isinstance(node.diag, DeviceTree):
        return node, None
    return node, node.diag


def diagonal_solve(L, j, G, transpose=False, s=None):
    """Alg. 4: apply the inverse (transpose) of node j's diagonal factor, or of the
    sub-triangle rooted at tree block s (diagblocks.py:176-213)."""
    eng = _engine(L)
    node, tree = _tree(eng, j)
    G = np.asarray(G, dtype=np.float64)
    vec = G.ndim == 1
    X = G.reshape(-1, 1) if vec else G
    if tree is None:
        if s is not None and s != 1:
            raise ShapeMismatch("dense diagonal has a single block")
        n = node.ncols
    else:
        nd = tree.shape.root if s is None else tree.shape.nodes[s]
        n = nd.hi - nd.lo
    Xd = _dev2(X, n)
    diag_solve_many([(node, Xd, bool(transpose)) + ((s,) if (tree is not None and s is not None) else ())],
                    eng.S.empty)
    out = Xd.cpu().numpy()
    return out[:, 0] if vec else out


def diagonal_multiply(A, L, j, s, G, transpose=False, sources=None):
    """Alg. 5: D_s G (or D_s^T G) for internal tree block s (diagblocks.py:303-346)."""
    eng = _engine(L)
    node, tree = _tree(eng, j)
    if tree is None or tree.shape.nodes[s].is_leaf:
        raise ShapeMismatch("diagonal_multiply needs an internal block of a diagonal tree")
    _check_sources(eng, j, sources)
    (r0, r1), (c0, c1) = tree.shape.span(s)
    G = np.atleast_2d(np.asarray(G, dtype=np.float64))
    W, = eng.diag_mul_many([(node, s)], [_dev2(G, (r1 - r0) if transpose else (c1 - c0))], bool(transpose))
    return W.cpu().numpy()


def factor_diagonal(A, L, j, s, sources=None):
    """Alg. 6: leaf s of node j's diagonal tree -- window of A minus every windowed
    source product and root-path product, then POTRF (diagblocks.py:276-300)."""
    eng = _engine(L)
    node, tree = _tree(eng, j)
    if tree is None or not tree.shape.nodes[s].is_leaf:
        raise ShapeMismatch("factor_diagonal needs a leaf of a diagonal tree")
    _check_sources(eng, j, sources)
    tri, = eng.leaves_many([(node, s)])
    eng.check()
    return np.tril(tri.L.cpu().numpy())


def approximate_diagonal_block(A, L, j, s, rank, power_iters=1, seed=0, sources=None):
    """Alg. 3 on internal tree block s (diagblocks.py:349-370)."""
    from .kernels import gaussian_matrix

    eng = _engine(L)
    node, tree = _tree(eng, j)
    if tree is None or tree.shape.nodes[s].is_leaf:
        raise ShapeMismatch("approximate_diagonal_block needs an internal block of a diagonal tree")
    _check_sources(eng, j, sources)
    (r0, r1), (c0, c1) = tree.shape.span(s)
    rank = min(rank, r1 - r0, c1 - c0)
    it = [(node, s)]
    G, = eng.diag_mul_many(it, [E.to_dev(gaussian_matrix(r1 - r0, rank, seed))], True)
    for _ in range(power_iters):
        G, = eng.diag_mul_many(it, eng.diag_mul_many(it, [G], False), True)
    U, = eng._orth_many([G])
    rk = int(eng.ibuf[eng._uslot.pop(id(U))].item())
    U = U[:, :rk].contiguous()
    if rk == 0:
        return LowRankBlock(np.zeros((r1 - r0, 0)), np.zeros((c1 - c0, 0)))
    V, = eng.diag_mul_many(it, [U], False)
    return LowRankBlock(V.cpu().numpy(), U.cpu().numpy())


def factor_interior_block(A, partition, member_ids, block_id=0):
    """Exact factor of one interior block (interior.py:105-156): A(C_B, C_B) on the
    device -> batched POTRF; the coupling rows stay implicit (A(off_rows, C_B) kept
    sparse) exactly as in the reference.  `A` is the permuted matrix."""
    from .factor import DenseTri, InteriorUnit

    ids = list(member_ids)
    c0, c1 = int(partition.starts[ids[0]]), int(partition.starts[ids[-1] + 1])
    nb = c1 - c0
    full = A.to_csr_full()
    M = E.to_dev(full[c0:c1, c0:c1].toarray())
    Dinv = E.empty(max(nb, 1), 64)
    info = E.zeros(1, dtype=E.I32)
    E.potrf_batched([M.data_ptr()], [nb], [nb], [Dinv.data_ptr()], info)
    bad = int(info.item())
    if bad:
        raise IndefiniteError(bad - 1)
    tails, stored = [], 0
    for jj in ids:
        rj = partition.rows[jj]
        nib = int(np.searchsorted(rj, c1))
        ncj = partition.ncols(jj)
        stored += ncj * (ncj + 1) // 2 + ncj * nib
        if rj.size > nib:
            tails.append(rj[nib:])
    off_rows = np.unique(np.concatenate(tails)) if tails else np.empty(0, np.int64)
    stored += full[off_rows, c0:c1].nnz if off_rows.size else 0
    unit = InteriorUnit(-1, ids, c0, c1, off_rows, DenseTri(M, Dinv), None, stored)
    return InteriorBlock(block_id, unit, partition, A)


def build_diag_tree(ncols, tau_d, split=None, g0=0):
    """Block-tree shape of a large separator diagonal (diagblocks.py:132-163)."""
    from .diagtree import TreeShape

    if split is None:
        from .symbolic import SplitTree  # noqa: F401

        raise ValueError("build_diag_tree needs the separator's SplitTree (ordering.partition_separator)")
    return DiagBlockTree(TreeShape(ncols, g0, split))
