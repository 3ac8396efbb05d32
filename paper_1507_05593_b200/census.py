"""Algorithmic work census of one factorization: the flops of the
operations the REFERENCE algorithm executes, per category, counted analytically from
the symbolic plan and the kept ranks -- not the GPU's executed (padded, materialized)
work.  This is the numerator of "factor GFLOP/s".

Conventions: POTRF n^3/3; right TRSM m n^2; dense triangular solve
n^2 k; GEMM 2mnk (SYRK counted full, 2 m^2 k, like the reference's dense `@`);
QRCP 4 m r^2; sparse x dense 2 nnz k; block-triangular solve with L_B and k
right-hand sides 2 nnz(L_B) k per pass; interior-block internals = member
POTRF + TRSM + a nib^2 nc update bound.  Operation by operation this follows
  _numeric_pass / _assemble_schur / off_diagonal_multiply[_trans] /
  approximate_off_diagonal                     factor.py:372-505, 538-639
  factor_diagonal / diagonal_multiply /
  approximate_diagonal_block                   diagblocks.py:220-370
  InteriorBlock.factor_rows / multiply         interior.py:77-95
and matches the counters of the oracle restatement operation for operation
(tests/test_census.py)."""

import math

import numpy as np

from .diagtree import TreeShape

CATEGORIES = ("off_sketch", "diag_sketch", "leaf_interior", "leaf_syrk", "leaf_path", "interior_gemm",
              "interior_solve", "sketch_diag_solve", "node_syrk_gemm", "qrcp", "potrf_trsm")
LABELS = {
    "off_sketch": "off-diagonal sketch products",
    "diag_sketch": "diagonal-tree sketch products",
    "leaf_interior": "diagonal-tree leaf interior-block terms",
    "leaf_syrk": "diagonal-tree leaf SYRK windows",
    "leaf_path": "diagonal-tree leaf path products",
    "interior_gemm": "interior-block update GEMM",
    "interior_solve": "interior-block solves",
    "sketch_diag_solve": "sketch diagonal solves",
    "node_syrk_gemm": "SYRK + GEMM in non-tree nodes",
    "qrcp": "QRCP",
    "potrf_trsm": "POTRF/TRSM of all kinds",
}
DENSE_FALLBACK = 0.75


def _block_rank(m, n, alpha, p):
    k = min(int(m), int(n))
    if k <= 0:
        return 0
    return min(int(math.ceil(alpha * math.sqrt(k) * math.log2(k))) + int(p), k)


class _Nnz:
    """nnz of row-set x column-range blocks of the full symmetric CSR, vectorized
    through one sorted key array (row * (n+1) + col)."""

    def __init__(self, full):
        n = full.shape[0]
        self.n1 = n + 1
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(full.indptr))
        self.keys = rows * self.n1 + full.indices.astype(np.int64)
        self.ptr = full.indptr.astype(np.int64)

    def rows(self, R, c0, c1):
        R = np.asarray(R, dtype=np.int64)
        if R.size == 0 or c1 <= c0:
            return 0
        b = R * self.n1
        return int(np.sum(np.searchsorted(self.keys, b + c1) - np.searchsorted(self.keys, b + c0)))

    def range(self, r0, r1, c0, c1):
        return self.rows(np.arange(r0, r1), c0, c1)


class _Src:
    __slots__ = ("kind", "rows", "order", "w", "nb", "nnzL", "c0", "c1", "lr")


def census(sym, cfg, ranks, alpha_d=None, per_unit=None):
    """{category: flops} of one factorization.  `ranks` maps ("off", j) and
    ("diag", j, s) to the kept rank of that compressed block (None: every block
    priced at its sketch width, an upper bound); `alpha_d` is the
    final (post-restart) alpha_D.  If `per_unit` is a list, the cumulative total
    after every unit (sweep order) is appended to it."""
    part = sym.partition
    full = sym.B.to_csr_full()
    nz = _Nnz(full)
    alpha_d = cfg.alpha_d if alpha_d is None else alpha_d
    q, p = cfg.power_iters, cfg.oversample
    C = dict.fromkeys(CATEGORIES, 0.0)
    M = part.count
    buckets = [[] for _ in range(M)]
    starts = part.starts

    def file(src, col):
        buckets[int(np.searchsorted(starts, col, side="right") - 1)].append(src)

    def src_terms(src, Rrows, c0, c1):
        """One implicit product's term of `src` (off_diagonal_multiply[_trans] /
        _source_window_multiply) with rows Rrows (global rows, or a (r0, r1) window)
        against cols [c0, c1): (flops per right-hand side, width-independent flops)."""
        if src.kind == "interior":
            rr = np.arange(*Rrows) if isinstance(Rrows, tuple) else Rrows
            return 2.0 * (nz.rows(np.arange(c0, c1), src.c0, src.c1) + nz.rows(rr, src.c0, src.c1)) \
                + 4.0 * src.nnzL, 0.0
        rows = src.rows
        clo, chi = np.searchsorted(rows, (c0, c1))
        if isinstance(Rrows, tuple):  # window rows [r0, r1)
            rlo, rhi = np.searchsorted(rows, Rrows)
            if clo == chi or rlo == rhi:
                return 0.0, 0.0
            # + eff_rows: V[sel] (U^T U) of a low-rank source, on every use
            return 2.0 * ((rhi - rlo) + (chi - clo)) * src.w, (2.0 * (rhi - rlo) * src.w**2 if src.lr else 0.0)
        if clo == chi or chi == rows.shape[0]:  # off-diagonal: rows[hi:] against R
            return 0.0, 0.0
        return 2.0 * (rows.shape[0] - clo) * src.w, (2.0 * (rows.shape[0] - chi) * src.w**2 if src.lr else 0.0)

    for u, (kind, payload) in enumerate(sym.units):
        if per_unit is not None and u:
            per_unit.append(sum(C.values()))
        if kind == "interior":
            ids = payload
            b0, b1 = part.cols(ids[0])[0], part.cols(ids[-1])[1]
            nnzL = 0
            tails = []
            for j in ids:
                j0, j1 = part.cols(j)
                ncj = j1 - j0
                rj = part.rows[j]
                nib = int(np.searchsorted(rj, b1))
                C["potrf_trsm"] += ncj**3 / 3.0 + nib * ncj * ncj + nib * nib * ncj
                nnzL += ncj * (ncj + 1) // 2 + ncj * nib
                if rj.size > nib:
                    tails.append(rj[nib:])
            off_rows = np.unique(np.concatenate(tails)) if tails else np.empty(0, np.int64)
            if off_rows.size:
                s = _Src()
                s.kind, s.rows, s.order, s.w, s.nb, s.nnzL, s.c0, s.c1 = \
                    "interior", off_rows, b0, 0, b1 - b0, nnzL, b0, b1
                s.lr = False
                file(s, off_rows[0])
            continue
        j = payload
        c0, c1 = part.cols(j)
        nc = c1 - c0
        R = part.rows[j]
        srcs = sorted(buckets[j], key=lambda s: s.order)
        buckets[j] = ()
        compress = bool(part.is_separator[j])
        tree_diag = compress and j in sym.sep_splits
        r_off = _block_rank(R.size, nc, cfg.alpha_o, p)
        compress_off = bool(compress and R.size and r_off < DENSE_FALLBACK * min(R.size, nc))
        nnzRC = nz.rows(R, c0, c1) if (R.size and compress_off) else 0
        tree_w = {}
        tree_lr = {}

        def assemble(want_off):
            want_off = want_off and R.size > 0
            for s in srcs:
                if s.kind == "interior":
                    C["interior_solve"] += 2.0 * s.nnzL * (nc + (R.size if want_off else 0))
                    C["interior_gemm"] += 2.0 * nc * nc * s.nb + (2.0 * R.size * nc * s.nb if want_off else 0.0)
                    continue
                lo, hi = np.searchsorted(s.rows, (c0, c1))
                if lo == hi:
                    continue
                C["node_syrk_gemm"] += 2.0 * (hi - lo) ** 2 * s.w + (2.0 * (hi - lo) * s.w * s.w if s.lr else 0.0)
                if hi < s.rows.shape[0] and want_off:
                    C["node_syrk_gemm"] += 2.0 * (s.rows.shape[0] - hi) * (hi - lo) * s.w \
                        + (2.0 * (s.rows.shape[0] - hi) * s.w * s.w if s.lr else 0.0)

        if tree_diag:
            shape = TreeShape(nc, c0, sym.sep_splits[j])
            for s in shape.order:
                tn = shape.nodes[s]
                if tn.is_leaf:
                    k = tn.hi - tn.lo
                    g0, g1 = c0 + tn.lo, c0 + tn.hi
                    for sr in srcs:
                        if sr.kind == "interior":
                            C["leaf_interior"] += 2.0 * sr.nnzL * k + 2.0 * k * k * sr.nb
                            continue
                        lo, hi = np.searchsorted(sr.rows, (g0, g1))
                        if lo < hi:
                            C["leaf_syrk"] += 2.0 * (hi - lo) ** 2 * sr.w + (2.0 * (hi - lo) * sr.w**2 if sr.lr else 0.0)
                    for pa in shape.path_above(s):
                        C["leaf_path"] += 2.0 * k * k * tree_w[pa] + (2.0 * k * tree_w[pa] ** 2 if tree_lr[pa] else 0.0)
                    C["potrf_trsm"] += k**3 / 3.0
                    continue
                (r0, r1), (k0, k1) = shape.span(s)
                nrows, ncols = r1 - r0, k1 - k0
                gr, gc = (c0 + r0, c0 + r1), (c0 + k0, c0 + k1)
                nnzw = nz.range(gr[0], gr[1], gc[0], gc[1])
                path = shape.path_above(s)

                per_k, const = 2.0 * nnzw, 0.0
                for sr in srcs:
                    a, b = src_terms(sr, gr, gc[0], gc[1])
                    per_k += a
                    const += b
                for pa in path:
                    per_k += 2.0 * (nrows + ncols) * tree_w[pa]
                    const += 2.0 * nrows * tree_w[pa] ** 2 if tree_lr[pa] else 0.0

                def dmul(k, cat, per_k=per_k, const=const, ncols=ncols):
                    C["sketch_diag_solve"] += ncols * ncols * k
                    C[cat] += per_k * k + const

                r = _block_rank(nrows, ncols, alpha_d, p)
                if r >= DENSE_FALLBACK * min(nrows, ncols):
                    dmul(ncols, "diag_sketch")
                    tree_w[s], tree_lr[s] = ncols, False
                else:
                    rr = min(r, nrows, ncols)
                    kept = rr if ranks is None else int(ranks[("diag", j, s)])
                    for _ in range(1 + 2 * q):
                        dmul(rr, "diag_sketch")
                    C["qrcp"] += 4.0 * ncols * rr * rr
                    dmul(kept, "diag_sketch")
                    tree_w[s], tree_lr[s] = kept, True
        else:
            assemble(not compress_off)
            C["potrf_trsm"] += nc**3 / 3.0

        if R.size and compress_off:
            rr = min(r_off, R.size, nc)
            kept = rr if ranks is None else int(ranks[("off", j)])

            per_k, const = 2.0 * nnzRC, 0.0
            for sr in srcs:
                a, b = src_terms(sr, R, c0, c1)
                per_k += a
                const += b

            def omul(k):
                if k == 0:
                    return
                C["sketch_diag_solve"] += nc * nc * k
                C["off_sketch"] += per_k * k + const

            for _ in range(1 + 2 * q):
                omul(rr)
            C["qrcp"] += 4.0 * nc * rr * rr
            omul(kept)
            w, lr = kept, True
        elif R.size:
            if tree_diag:
                assemble(True)
            C["potrf_trsm"] += R.size * nc * nc
            w, lr = nc, False
        # advance this node's sources, then file the node itself (factor.py:636-639)
        for sr in srcs:
            hi = np.searchsorted(sr.rows, c1)
            if hi < sr.rows.shape[0]:
                file(sr, sr.rows[hi])
        if R.size:
            s = _Src()
            s.kind, s.rows, s.order, s.w, s.nb, s.nnzL, s.c0, s.c1 = "node", R, c0, w, 0, 0, c0, c1
            s.lr = lr
            file(s, R[0])
    if per_unit is not None and sym.units:
        per_unit.append(sum(C.values()))
    return C


def census_table(C):
    tot = sum(C.values())
    return [(LABELS[k], C[k] / 1e9, C[k] / tot if tot else 0.0) for k in sorted(C, key=lambda k: -C[k])]
