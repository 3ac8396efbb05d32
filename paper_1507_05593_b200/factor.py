"""GPU numeric rank-structured factorization (drop-in for rschol.factorize).

Host Python walks the unit plan (factor.py:556-639 order) and issues grouped
sm_100a kernels through the C ABI; all numeric data stays in HBM:

  interior blocks    all factored up front in ONE batched POTRF + ONE batched TRSM
                     (they depend on nothing), coupling rows materialized as
                     Y_B = A(off_rows, C_B) L_B^{-T}  (interior.py:29-156)
  Schur assembly     gather -> DMMA -> scatter-subtract, one grouped launch over all
                     sources of the target (factor.py:372-399, diagblocks.py:220-238)
  implicit products  two grouped launches per product: T_s = X_s^T G[map] for all
                     sources, then W[map] -= Y_s T_s summed over sources in
                     reference order by an ordered (deterministic) reduction
                     (factor.py:427-483, diagblocks.py:241-346)
  compression        host PCG64 sketch -> products -> pivoted QR (rank cutoff) ->
                     projection V = L_O U  (factor.py:486-505, diagblocks.py:349-370)
  diagonal trees     leaf Schur + POTRF, internal blocks compressed or dense
                     (diagblocks.py:276-346), Alg. 4 tree solves on device
  restart            IndefiniteError restarts the pass with alpha_d *= growth when a
                     diagonal tree was started before the failing pivot
                     (factor.py:702-718)
"""

import math
import os
import time
import weakref
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import engine as E
from ._lib import GEMM_DTYPE
from .errors import DimensionMismatch, IndefiniteError, TooManyRestarts
from .plan import NumericPlan
from .sparse import as_spd
from .symbolic import analyze, block_rank

__all__ = ["SolverConfig", "FactorStats", "RankStructuredFactor", "block_rank", "factorize"]

DENSE_FALLBACK_FRACTION = 0.75


@dataclass
class SolverConfig:
    """Tuning knobs (factor.py:65-111), same names, defaults and validation."""

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

    def __post_init__(self):
        if self.tau_o < 1 or self.tau_d < 1:
            raise ValueError("tau_o and tau_d must be positive")
        if self.alpha_o <= 0 or self.alpha_d <= 0 or self.oversample <= 0:
            raise ValueError("alpha_o, alpha_d and oversample must be positive")
        if self.power_iters < 0 or self.max_restarts < 0:
            raise ValueError("power_iters and max_restarts must be nonnegative")
        if self.alpha_d_growth <= 1.0:
            raise ValueError("alpha_d_growth must exceed 1")

    def to_dict(self):
        d = dict(self.__dict__)
        if not math.isfinite(self.tau_o):
            d["tau_o"] = "inf"
        return d


@dataclass
class FactorStats:
    n: int = 0
    nnz_lower: int = 0
    supernodes: int = 0
    separator_supernodes: int = 0
    interior_block_count: int = 0
    compressed_offdiag: int = 0
    compressed_diag: int = 0
    dense_fallback: int = 0
    stored_scalars: int = 0
    restarts: int = 0
    alpha_d_final: float = 0.0
    alpha_d_history: list = field(default_factory=list)
    phase_times: dict = field(default_factory=dict)
    seed: int = 0
    gpu_launches: int = 0
    model_gflop: float = 0.0

    @property
    def compressed_blocks(self):
        return self.compressed_offdiag + self.compressed_diag

    def to_dict(self):
        return {
            "n": self.n, "nnz": self.nnz_lower, "supernodes": self.supernodes,
            "separator_supernodes": self.separator_supernodes, "interior_blocks": self.interior_block_count,
            "compressed_blocks": self.compressed_blocks, "compressed_offdiag": self.compressed_offdiag,
            "compressed_diag": self.compressed_diag, "dense_fallback": self.dense_fallback,
            "stored_scalars": self.stored_scalars, "restarts": self.restarts,
            "alpha_D_final": self.alpha_d_final, "alpha_D_history": self.alpha_d_history,
            "phase_times": self.phase_times, "seed": self.seed,
        }


def _block_seed(master, *tags):
    """factor.py:324-326."""
    ss = np.random.SeedSequence((int(master),) + tuple(int(t) for t in tags))
    return int(ss.generate_state(1, np.uint64)[0])


def _gaussian(m, n, seed):
    """Reference PCG64 stream (kernels.py:85-92), generated on the host."""
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((m, n))


# ---------------------------------------------------------------------------
# device factor blocks


class DenseTri:
    """Dense lower triangle + inverse 64x64 diagonal blocks."""

    __slots__ = ("L", "Dinv", "n", "Linv", "LinvT", "inv_mem")

    def __init__(self, L, Dinv):
        self.L, self.Dinv, self.n = L, Dinv, L.shape[0]
        self.Linv = self.LinvT = None  # explicit inverse (and its transpose), built for the apply
        self.inv_mem = None  # the arena Linv/LinvT were carved from (kept alive with them)

    def solve(self, X, transpose=False):
        """X <- L^{-1} X (or L^{-T} X) in place; X is an n x r row-major view."""
        if self.n == 0 or X.shape[1] == 0:
            return
        E.trsm_batched("left", 1 if transpose else 0, [self.L.data_ptr()], [self.n], [E.ld(self.L)],
                       [self.Dinv.data_ptr()], [X.data_ptr()], [X.shape[1]], [E.ld(X)])


class DevLR:
    """Low-rank block V U^T (U orthonormal), with E = V (U^T U) kept for the
    eff_rows role of blocks.py:103-113."""

    __slots__ = ("V", "U", "E", "k", "kslot")

    def __init__(self, V, U, Eff):
        self.V, self.U, self.E, self.k = V, U, Eff, U.shape[1]
        self.kslot = None  # device rank word while the columns are still sketch-padded


class DeviceTree:
    """Numeric content of a hierarchical diagonal (DenseTri leaves, dense or
    DevLR couplings) and its Alg. 4 solve (diagblocks.py:176-213)."""

    def __init__(self, shape):
        self.shape = shape
        self.blocks = {}

    def solve(self, X, transpose=False, s=None):
        nd = self.shape.root if s is None else self.shape.nodes[s]
        self._solve(nd, X, transpose)

    def _solve(self, nd, X, transpose):
        if nd.is_leaf:
            self.blocks[nd.s].solve(X, transpose)
            return
        k = nd.split - nd.lo
        X1, X2 = X[:k], X[k:]
        b = self.blocks[nd.s]
        if transpose:
            self._solve(nd.right, X2, True)
            _couple_sub(b, X2, X1, transpose=True)
            self._solve(nd.left, X1, True)
        else:
            self._solve(nd.left, X1, False)
            _couple_sub(b, X1, X2, transpose=False)
            self._solve(nd.right, X2, False)


def _gemm1(A, B, C, transA=False, transB=False, alpha=1.0, beta=0.0):
    if C.shape[0] == 0 or C.shape[1] == 0:
        return
    E.gemm(A, B, C, transA=transA, transB=transB, alpha=alpha, beta=beta)


def _couple_sub(b, X, Y, transpose):
    """Y -= block @ X (or block^T @ X) for a dense or low-rank coupling block."""
    r = X.shape[1]
    if isinstance(b, DevLR):
        if b.k == 0:
            return
        t = E.scratch(b.k, r)
        if transpose:  # U (V^T X)
            _gemm1(b.V, X, t, transA=True)
            _gemm1(b.U, t, Y, alpha=-1.0, beta=1.0)
        else:  # V (U^T X)
            _gemm1(b.U, X, t, transA=True)
            _gemm1(b.V, t, Y, alpha=-1.0, beta=1.0)
    else:
        _gemm1(b, X, Y, transA=transpose, alpha=-1.0, beta=1.0)


def _raw_eff(obj):
    """(raw, eff) panels of a dense or low-rank block (blocks.py:103-119)."""
    if isinstance(obj, DevLR):
        return obj.V, obj.E
    return obj, obj


class Grouped:
    """Accumulates problems of one grouped GEMM launch (vectorized descriptor build)."""

    def __init__(self, transA, transB):
        self.tA, self.tB = transA, transB
        self.rows = []

    def add(self, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, b_rows=0, c_rows=0, c_cols=0, atomic=0):
        if M > 0 and N > 0:
            self.rows.append((A, B, C, 0, 0, 0, b_rows, c_rows, c_cols, M, N, K, max(lda, 1), max(ldb, 1),
                              max(ldc, 1), 1, atomic, alpha, beta, 0, 0))

    def launch(self):
        if self.rows:
            E.gemm_balanced(np.array(self.rows, dtype=GEMM_DTYPE), self.tA, self.tB)
            self.rows = []


# ---------------------------------------------------------------------------
# unit records


class InteriorUnit:
    """Exact subdomain factor L_B (dense triangle) + materialized coupling Y_B."""

    kind = "interior"

    def __init__(self, u, members, c0, c1, off_rows, tri, Y, stored):
        self.u, self.members, self.c0, self.c1 = u, members, c0, c1
        self.rows = off_rows
        self.off_rows = off_rows
        self.diag = tri
        self.off = Y
        self._stored = stored

    @property
    def ncols(self):
        return self.c1 - self.c0


class NodeUnit:
    kind = "node"

    def __init__(self, u, j, c0, c1, rows):
        self.u, self.j, self.c0, self.c1, self.rows = u, j, c0, c1, rows
        self.diag = None
        self.off = None

    @property
    def ncols(self):
        return self.c1 - self.c0


# ---------------------------------------------------------------------------
# the numeric pass


class _Indefinite(Exception):
    def __init__(self, unit, pivot, trees=0):
        self.unit, self.pivot, self.trees = unit, pivot, trees


class NumericPass:
    """State shared by the numeric sweep (factor.py:538-639): arenas, the device
    info/rank words, pending pivot checks, the sketches, interior blocks.  The sweep
    itself is numeric.LevelPass (level-batched; it is the only driver)."""

    def __init__(self, plan, cfg, alpha_d):
        self.np = plan
        self.sym = plan.sym
        self.cfg = cfg
        self.alpha_d = alpha_d
        self.counters = {"diag_trees": 0, "compressed_off": 0, "compressed_diag": 0, "dense_fallback": 0}
        self.units = []
        self.src_panel = {}  # source id -> (raw tensor, eff tensor)
        self.ranks = {}
        self.flops = 0.0
        self.P = E.Arena()            # factor blocks (persist with the factor)
        self.S = E.Arena(1 << 24)     # per-unit transients, reset at every unit
        nints = 4 * (len(self.sym.units) + sum(len(t.nodes) for t in plan.tree_shapes.values())) + 64
        self.ibuf = E.zeros(nints, dtype=E.I32)  # POTRF info words + QR ranks
        self.ipos = 0
        self.pending = []             # (info offset, count, unit, diag trees started so far)
        self.sketches = plan.sketches_for(cfg, alpha_d)

    def _ints(self, n):
        t = self.ibuf[self.ipos:self.ipos + n]
        self.ipos += n
        return t

    def factor_interiors(self, defer=False, keep=None):
        """All interior blocks at once: dense A(C_B,C_B) -> batched POTRF, then
        Y_B = A(off_rows, C_B) L_B^{-T} by one batched TRSM.  defer=True records the
        POTRF info words as pending pivot checks instead of reading them back;
        keep(u) restricts the batch (multi-GPU: the rank's own subtrees)."""
        ints = self.np.interior
        if keep is not None:
            ints = [x for x in ints if keep(x[0])]
        self.first_interior_failure = None
        if not ints:
            return {}
        Ls, Ys = self._interior_mats(ints)
        Ds = [self.P.empty(max(c1 - c0, 1), 64) for (u, ids, c0, c1, off_rows, A_off, A_BB) in ints]
        info_off = self.ipos
        info = self._ints(len(ints))
        E.potrf_batched([L.data_ptr() for L in Ls], [L.shape[0] for L in Ls], [E.ld(L) for L in Ls],
                        [D.data_ptr() for D in Ds], info)
        E.trsm_batched("right", 1, [L.data_ptr() for L in Ls], [L.shape[0] for L in Ls], [E.ld(L) for L in Ls],
                       [D.data_ptr() for D in Ds], [Y.data_ptr() for Y in Ys], [Y.shape[0] for Y in Ys],
                       [E.ld(Y) for Y in Ys])
        iv = None if defer else info.cpu().numpy()
        out = {}
        self.first_interior_failure = None
        for i, (u, ids, c0, c1, off_rows, A_off, A_BB) in enumerate(ints):
            if defer:
                self.pending.append((info_off + i, 1, u, self._trees_before(u)))
            elif iv[i] and self.first_interior_failure is None:
                self.first_interior_failure = (u, int(iv[i]) - 1, self._trees_before(u))
            nb = c1 - c0
            stored = (A_off.nnz if A_off is not None else 0)
            part = self.sym.partition
            for j in ids:
                j0, j1 = part.cols(j)
                ncj = j1 - j0
                nib = int(np.searchsorted(part.rows[j], c1))
                stored += ncj * (ncj + 1) // 2 + ncj * nib
            out[u] = InteriorUnit(u, ids, c0, c1, off_rows, DenseTri(Ls[i], Ds[i]), Ys[i], stored)
            self.flops += nb**3 / 3.0 + off_rows.size * nb * nb
        return out

    def _path_terms(self, tree, s, rspan, cspan):
        out = []
        for p in tree.shape.path_above(s):
            base = tree.shape.nodes[p].split
            raw, eff = _raw_eff(tree.blocks[p])
            out.append((raw, eff, rspan[0] - base, rspan[1] - base, cspan[0] - base, cspan[1] - base))
        return out

    def _trees_before(self, u):
        """Diagonal trees started before unit u (the restart test of factor.py:709)."""
        # the tree counter is bumped before a tree node's own leaf POTRFs (factor.py:587-588)
        return int(np.searchsorted(self.np.tree_units, u, side="right"))

    def run(self):
        prev = E.SCRATCH
        E.SCRATCH = self.S
        try:
            self._run()
            self.check_pivots()
        finally:
            E.SCRATCH = prev


# ---------------------------------------------------------------------------
# factor container


class RankStructuredFactor:
    """Approximate Cholesky factor resident on the B200, applied as an SPD
    preconditioner (factor.py:155-310)."""

    def __init__(self, n, sym, plan, config):
        self.n = n
        self.sym = sym
        self.plan = plan
        self.perm = sym.perm
        self.partition = sym.partition
        self.config = config
        self.dunits = []
        self.ranks = {}
        self.stats = FactorStats(n=n, seed=config.seed)
        self._apply = None

    # -- reference object model (factor.py:163-172): lazy host views ------------
    def _build_views(self):
        from .views import DiagBlockTree, InteriorBlock, LowRankBlock, SupernodeFactor

        part = self.partition
        nodes = [None] * part.count
        interior, units = [], []
        for un in self.dunits:
            if un.kind == "interior":
                blk = InteriorBlock(len(interior), un, part, self.sym.B)
                interior.append(blk)
                for m in blk.members:
                    nodes[m.j] = m
                units.append(("interior", blk))
                continue
            if isinstance(un.diag, DeviceTree):
                diag = DiagBlockTree(un.diag.shape, un.diag)
            else:
                diag = (lambda t=un.diag: np.tril(t.L.cpu().numpy()))
            if un.off is None:
                off = None
            elif isinstance(un.off, DevLR):
                off = LowRankBlock(un.off)
            else:
                off = (lambda t=un.off: t.cpu().numpy())
            nd = SupernodeFactor(un.j, un.c0, un.c1, un.rows, diag, off)
            nd._dev = un
            nodes[un.j] = nd
            units.append(("node", nd))
        self._views = (nodes, interior, units)

    @property
    def nodes(self):
        """One SupernodeFactor per supernode (reference factor.py:168)."""
        if getattr(self, "_views", None) is None:
            self._build_views()
        return self._views[0]

    @property
    def interior(self):
        """The interior blocks, in sweep order (reference factor.py:169)."""
        if getattr(self, "_views", None) is None:
            self._build_views()
        return self._views[1]

    @property
    def units(self):
        """("interior", InteriorBlock) / ("node", SupernodeFactor) in sweep order
        (reference factor.py:170, 559-639)."""
        if getattr(self, "_views", None) is None:
            self._build_views()
        return self._views[2]

    # -- application -----------------------------------------------------------
    def apply(self, r):
        """z = P^T (L L^T)^{-1} P r (host vector in, host vector out)."""
        r = np.asarray(r, dtype=np.float64)
        if r.shape != (self.n,):
            raise DimensionMismatch(f"expected vector of length {self.n}")
        y = E.to_dev(r)
        z = self.apply_device(y)
        if getattr(self, "dist", None):  # sharded factor: assemble z from every rank's rows
            from .pcg import _DistOps

            if getattr(self, "_dist_ops", None) is None:
                self._dist_ops = _DistOps(self.source_matrix, self)
            self._dist_ops.combine(z)
        return z.cpu().numpy()

    __call__ = apply

    def apply_device(self, r_dev, out=None):
        from .apply import DeviceApply

        if self._apply is None:
            self._apply = DeviceApply(self)
            entry = getattr(self, "_entry", None)
            if entry is not None:  # reusable by later replays with the same ranks
                entry.apply, entry.apply_key = self._apply, self._apply_key()
        return self._apply(r_dev, out)

    def _apply_key(self):
        return tuple(sorted(self.ranks.items(), key=repr))

    # -- inspection ------------------------------------------------------------
    def stored_scalars(self):
        if getattr(self, "dist", None):  # a sharded factor: summed over the ranks at factorization
            return self.stats.stored_scalars
        total = 0
        for un in self.dunits:
            if un.kind == "interior":
                total += un._stored
                continue
            nc = un.ncols
            if isinstance(un.diag, DeviceTree):
                for s, nd in un.diag.shape.nodes.items():
                    b = un.diag.blocks[s]
                    if nd.is_leaf:
                        k = nd.hi - nd.lo
                        total += k * (k + 1) // 2
                    elif isinstance(b, DevLR):
                        total += b.V.numel() + b.U.numel()
                    else:
                        total += b.numel()
            else:
                total += nc * (nc + 1) // 2
            if isinstance(un.off, DevLR):
                total += un.off.V.numel() + un.off.U.numel()
            elif un.off is not None:
                total += un.off.numel()
        return total

    def _diag_dense(self, un):
        if isinstance(un.diag, DeviceTree):
            shape = un.diag.shape
            Ld = np.zeros((un.ncols, un.ncols))
            for s, nd in shape.nodes.items():
                (r0, r1), (c0, c1) = shape.span(s)
                b = un.diag.blocks[s]
                if nd.is_leaf:
                    Ld[r0:r1, c0:c1] = np.tril(b.L.cpu().numpy())
                elif isinstance(b, DevLR):
                    Ld[r0:r1, c0:c1] = b.V.cpu().numpy() @ b.U.cpu().numpy().T
                else:
                    Ld[r0:r1, c0:c1] = b.cpu().numpy()
            return Ld
        return np.tril(un.diag.L.cpu().numpy())

    def _off_dense(self, un):
        if isinstance(un.off, DevLR):
            return un.off.V.cpu().numpy() @ un.off.U.cpu().numpy().T
        return un.off.cpu().numpy()

    def dense_lower(self):
        """Explicit lower-triangular factor (small problems, testing)."""
        L = np.zeros((self.n, self.n))
        for un in self.dunits:
            L[un.c0:un.c1, un.c0:un.c1] = self._diag_dense(un)
            if un.rows.size and un.off is not None:
                L[un.rows, un.c0:un.c1] = self._off_dense(un)
        return L

    def to_scipy_lower(self):
        import scipy.sparse as sp

        rows, cols, vals = [], [], []
        for un in self.dunits:
            cr = np.arange(un.c0, un.c1)
            for blk, rr in ((self._diag_dense(un), cr),
                            (self._off_dense(un) if (un.rows.size and un.off is not None) else None, un.rows)):
                if blk is None:
                    continue
                a, b = np.nonzero(blk)
                rows.append(rr[a])
                cols.append(cr[b])
                vals.append(blk[a, b])
        if not rows:
            return sp.csc_matrix((self.n, self.n))
        return sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(self.n, self.n))


# Refactorization through CUDA graphs: with a reused plan (factorize(..., prepared=)),
# the sweep for a given alpha_d is captured once and replayed for every later matrix
# of the same pattern -- the same kernels on the new values, without the host
# re-issuing ~4k launches.  The replay rewrites the captured pass's memory, so it is
# used only while no earlier factor from that graph is alive (otherwise an ordinary
# pass runs on fresh memory).  RSC_GRAPH=0 disables it.
GRAPH_REFACTOR = os.environ.get("RSC_GRAPH", "1") != "0"


class _GraphEntry:
    __slots__ = ("ps", "owner", "apply", "apply_key")

    def __init__(self, ps):
        self.ps, self.owner, self.apply, self.apply_key = ps, None, None, None


def _numeric_pass(plan, config, alpha_d, use_graph):
    """One numeric pass at alpha_d -> (pass, graph entry or None); raises _Indefinite."""
    from .numeric import LevelPass

    if use_graph:
        graphs = plan.__dict__.setdefault("graphs", {})
        entry = graphs.get(alpha_d)
        if entry is None and alpha_d in plan.__dict__.setdefault("eager_seen", set()):
            # second pass at this alpha_d: every kernel has run eagerly once (function
            # attributes set, tables initialised), so the sweep can be recorded
            ps = LevelPass(plan, config, alpha_d)
            ps.capture()
            entry = graphs[alpha_d] = _GraphEntry(ps)
            ps.replay()
            return ps, entry
        if entry is not None and (entry.owner is None or entry.owner() is None):
            entry.ps.replay()
            return entry.ps, entry
        plan.eager_seen.add(alpha_d)
    ps = LevelPass(plan, config, alpha_d)
    ps.run()
    return ps, None


def _normalize(A):
    """Stored explicit zeros are dropped before ordering and symbolic analysis.  The
    reference orders on the zero-free graph (ordering.py:113-119) but builds the
    elimination tree and row structures from the stored pattern (symbolic.py:52,296),
    so interior-block update sources land in buckets no supernode drains
    (factor.py:547-554) and the factor silently loses Schur terms (SURVEY Appendix
    A.1).  Dropping them makes both agree; the operator is unchanged."""
    if getattr(A, "_zero_free", False):
        return A
    nz = int(np.count_nonzero(A.values == 0.0))
    if not nz:
        try:
            A._zero_free = True  # immutable matrix (sparse.py:47-48): checked once
        except AttributeError:
            pass
    if nz:
        from .sparse import strip_explicit_zeros

        warnings.warn(f"factorize: dropped {nz} stored zeros before the symbolic analysis "
                      "(SURVEY Appendix A.1)", RuntimeWarning, stacklevel=3)
        A = strip_explicit_zeros(A)
    return A


def prepare(A, config=None, coords=None):
    """Host half of factorize: ordering + symbolic + device plan upload.  The
    result can be reused by factorize(..., prepared=...) for repeated numeric
    factorizations of matrices with the same pattern (quasi-static load steps)."""
    E.require_cuda()
    A = _normalize(as_spd(A))
    config = config if config is not None else SolverConfig()
    t0 = time.perf_counter()
    sym = analyze(A, config.tau_o, config.tau_d, config.interior_blocks, coords=coords)
    t1 = time.perf_counter()
    plan = NumericPlan(sym, config.interior_blocks, A)
    t2 = time.perf_counter()
    return (sym, plan, config, t0, t1, t2)


def factorize(A, config=None, coords=None, prepared=None):
    """Order, analyze and factor A on the B200 (factor.py:642-740).

    Same contract as rschol.factorize: ordering/symbolic on the host, the numeric
    sweep on the device, restart with alpha_d *= alpha_d_growth on an indefinite
    pivot once a diagonal tree is in play, TooManyRestarts after max_restarts.
    """
    with E.gc_paused():
        return _factorize(A, config, coords, prepared)


def _factorize(A, config, coords, prepared):
    A = _normalize(as_spd(A))
    reuse = prepared is not None
    if prepared is None:
        prepared = prepare(A, config, coords)
        sym, plan, config, t0, t_plan0, t2 = prepared
    else:
        sym, plan, config, _, _, _ = prepared
        t0 = t_plan0 = time.perf_counter()
        sym.t_ordering = sym.t_symbolic = 0.0
        plan.load_values(A)  # same pattern, possibly new values (refactorization)
        t2 = time.perf_counter()
    from . import _lib

    lib = _lib.load()
    launches0 = int(lib.rsc_launch_counter(0))
    alpha_d = config.alpha_d
    history = [alpha_d]
    restarts = 0
    use_graph = reuse and GRAPH_REFACTOR
    while True:
        try:
            ps, entry = _numeric_pass(plan, config, alpha_d, use_graph)
            torch.cuda.current_stream().synchronize()
            break
        except _Indefinite as e:
            torch.cuda.current_stream().synchronize()
            if e.trees == 0:
                raise IndefiniteError(e.pivot) from None
            restarts += 1
            if restarts > config.max_restarts:
                raise TooManyRestarts(
                    f"still indefinite after {config.max_restarts} restarts (alpha_d reached {alpha_d:g})"
                ) from None
            alpha_d *= config.alpha_d_growth
            history.append(alpha_d)
    t3 = time.perf_counter()
    F = RankStructuredFactor(A.n, sym, plan, config)
    F.dunits = ps.units
    F._mem = ps.P  # the factor owns its arena: chunks return to the pool only when F dies
    F.ranks = ps.ranks
    if entry is not None:
        entry.owner = weakref.ref(F)  # the graph may rewrite this memory once F is gone
        F._entry = entry
        if entry.apply is not None:
            key = F._apply_key()
            # same memory, same ranks: the apply program still holds once its explicit
            # inverses are re-derived; other ranks: patch its rank dimensions first
            if entry.apply_key == key or entry.apply.rekey(F):
                F._apply = entry.apply
                F._apply.refresh_inverses()
                entry.apply_key = key
    part = sym.partition
    st = F.stats
    st.n, st.nnz_lower = A.n, A.nnz_lower
    st.supernodes = part.count
    st.separator_supernodes = int(part.is_separator.sum())
    st.interior_block_count = len(plan.interior)
    st.compressed_offdiag = ps.counters["compressed_off"]
    st.compressed_diag = ps.counters["compressed_diag"]
    st.dense_fallback = ps.counters["dense_fallback"]
    st.stored_scalars = F.stored_scalars()
    st.restarts = restarts
    st.alpha_d_final = alpha_d
    st.alpha_d_history = history
    st.gpu_launches = int(lib.rsc_launch_counter(0)) - launches0
    if entry is not None:
        st.gpu_launches = ps.launches  # kernel nodes of the replayed graph
    from . import numeric as _nm

    st.model_gflop = ps.flops / 1e9 if _nm.FLOP_MODEL else float("nan")  # RSC_FLOP_MODEL=1
    st.phase_times = {"ordering": sym.t_ordering, "symbolic": sym.t_symbolic + (t2 - t_plan0),
                      "numeric": t3 - t2, "total": t3 - t0}
    return F
