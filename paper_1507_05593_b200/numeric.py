"""Level-batched numeric sweep (the production driver of factorize).

The reference sweeps its units one at a time (factor.py:556-639).  A compressed
separator only reads its update sources -- interior blocks and separators lower in
the nested-dissection tree -- so all separators of one ND level are independent
and their work is issued together: every step below is ONE grouped launch (or one
batched call) over all nodes of the level.  Compressed blocks stay at sketch width
(the QR zeroes the columns past the rank), so the whole pass is issued without a
host<->device synchronisation; one readback at the end trims the blocks to their
ranks and resolves pivot failures.  Results are identical to the unit-by-unit order
because each node's arithmetic is unchanged (the padded columns add exact zeros);
only its interleaving with independent nodes differs.

Per level:
  dense diagonals   A-block scatter + Schur update of all (node, source) pairs,
                    batched POTRF, batched TRSM for dense off-diagonals
  diagonal trees    advanced in lock-step over in-order block positions; leaves
                    by batched window assembly + POTRF, internal blocks by batched
                    implicit products (Alg. 5) whose Alg. 4 sub-solves run as
                    lock-step waves across trees
  compression       sketch products of all compressed off-diagonals of the level
                    (Alg. 2 and its transpose), one batched pivoted QR, V = L_O U

Pivot failures are collected and resolved at the end of the pass in sweep order
(the earliest failing unit decides restart vs. re-raise, factor.py:705-710).
"""

import os

import numpy as np

from . import engine as E
from ._lib import GEMM_DTYPE
from .factor import (
    DENSE_FALLBACK_FRACTION,
    DenseTri,
    DeviceTree,
    DevLR,
    Grouped,
    InteriorUnit,
    NodeUnit,
    NumericPass,
    _Indefinite,
    _raw_eff,
)
from .symbolic import block_rank

FLOP_MODEL = os.environ.get("RSC_FLOP_MODEL", "0") == "1"



# ---------------------------------------------------------------------------
# lock-step batched Alg. 4


def tree_ops(tree, s, X, transpose):
    """Flatten the block substitution of subtree s of `tree` acting on X."""
    ops = []
    nd0 = tree.shape.root if s is None else tree.shape.nodes[s]

    def rec(nd, Xv):
        if nd.is_leaf:
            ops.append(("leaf", tree.blocks[nd.s], Xv, transpose))
            return
        k = nd.split - nd.lo
        X1, X2 = Xv[:k], Xv[k:]
        b = tree.blocks[nd.s]
        if transpose:
            rec(nd.right, X2)
            ops.append(("couple", b, X2, X1, True))
            rec(nd.left, X1)
        else:
            rec(nd.left, X1)
            ops.append(("couple", b, X1, X2, False))
            rec(nd.right, X2)

    rec(nd0, X)
    return ops


def run_waves(seqs, scratch):
    """Execute op sequences in lock-step: wave w runs op w of every sequence.

    The ops of one wave belong to different trees, so they are independent: per wave
    the leaf solves are one batched TRSM per direction, every transposed-A product
    (dense couplings in the transposed sweep and the first factor t = P1^T X of every
    low-rank coupling) is one grouped launch, and every plain product (dense
    couplings of the forward sweep and the second factor Y -= P2 t) is one more."""
    seqs = [s for s in seqs if s]
    if not seqs:
        return
    for w in range(max(len(s) for s in seqs)):
        keep = []  # temporaries must outlive the launches below (torch may recycle freed blocks)
        leaves = {0: [], 1: []}
        g_t = Grouped(True, False)    # transposed-A products (independent of each other)
        g_n = Grouped(False, False)   # plain products (the low-rank ones need g_t's t)
        lr = []
        for seq in seqs:
            if w >= len(seq):
                continue
            op = seq[w]
            if op[0] == "leaf":
                _, tri, Xv, tr = op
                if tri.n and Xv.shape[1]:
                    leaves[int(tr)].append((tri, Xv))
                continue
            _, b, Xs, Yd, tr = op
            r = Xs.shape[1]
            if r == 0:
                continue
            if isinstance(b, DevLR):
                if b.k == 0:
                    continue
                lr.append((b, Xs, Yd, tr, r))
            elif tr:
                g_t.add(b.data_ptr(), E.ld(b), Xs.data_ptr(), E.ld(Xs), Yd.data_ptr(), E.ld(Yd), b.shape[1], r,
                        b.shape[0], -1.0, 1.0)
            else:
                g_n.add(b.data_ptr(), E.ld(b), Xs.data_ptr(), E.ld(Xs), Yd.data_ptr(), E.ld(Yd), b.shape[0], r,
                        b.shape[1], -1.0, 1.0)
        if lr:
            ts = scratch(sum(b.k * r for b, _, _, _, r in lr))
            ts.zero_()  # t = P1^T X accumulates (ordered): balance_k may split its tall K
            keep.append(ts)
            off = 0
            for b, Xs, Yd, tr, r in lr:
                tp = ts.data_ptr() + 8 * off
                off += b.k * r
                # t = U^T X (forward) or V^T X (transposed); then Y -= V t or U t
                P1 = b.V if tr else b.U
                P2 = b.U if tr else b.V
                g_t.add(P1.data_ptr(), E.ld(P1), Xs.data_ptr(), E.ld(Xs), tp, r, b.k, r, Xs.shape[0], 1.0, 0.0,
                        atomic=1)
                g_n.add(P2.data_ptr(), E.ld(P2), tp, r, Yd.data_ptr(), E.ld(Yd), Yd.shape[0], r, b.k, -1.0, 1.0)
        for tr, lst in leaves.items():
            if lst:
                E.trsm_batched("left", tr, [t.L.data_ptr() for t, _ in lst], [t.n for t, _ in lst],
                               [E.ld(t.L) for t, _ in lst], [t.Dinv.data_ptr() for t, _ in lst],
                               [X.data_ptr() for _, X in lst], [X.shape[1] for _, X in lst],
                               [E.ld(X) for _, X in lst])
        g_t.launch()
        g_n.launch()


def diag_solve_many(items, scratch):
    """items: (node, X, transpose[, subtree s]) -> X <- D^{-1} X / D^{-T} X in place."""
    dense = {0: [], 1: []}
    seqs = []
    for it in items:
        node, X, tr = it[0], it[1], it[2]
        s = it[3] if len(it) > 3 else None
        if X.shape[1] == 0 or X.shape[0] == 0:
            continue
        if isinstance(node.diag, DeviceTree):
            seqs.append(tree_ops(node.diag, s, X, tr))
        else:
            dense[int(tr)].append((node.diag, X))
    for tr, lst in dense.items():
        if lst:
            E.trsm_batched("left", tr, [t.L.data_ptr() for t, _ in lst], [t.n for t, _ in lst],
                           [E.ld(t.L) for t, _ in lst], [t.Dinv.data_ptr() for t, _ in lst],
                           [X.data_ptr() for _, X in lst], [X.shape[1] for _, X in lst], [E.ld(X) for _, X in lst])
    run_waves(seqs, scratch)


# ---------------------------------------------------------------------------


class LevelPass(NumericPass):
    """Level-batched version of NumericPass (same results, far fewer launches)."""

    # fault injection for the restart tests: callable(pass, leaf
    # items) -> True to make the first leaf of that batch indefinite
    fault_hook = None

    def __init__(self, plan, cfg, alpha_d):
        super().__init__(plan, cfg, alpha_d)
        ns = len(plan.sources)
        self.s_raw = np.zeros(ns, dtype=np.uint64)   # device address of the raw panel
        self.s_eff = np.zeros(ns, dtype=np.uint64)   # ... of the eff panel (V U^T U or = raw)
        self.s_ld = np.ones(ns, dtype=np.int64)
        self.s_w = np.zeros(ns, dtype=np.int64)      # panel width (0 = contributes nothing)
        self.idx_base = np.uint64(plan.idx.dev.data_ptr())
        self._uslot = {}     # id(U) -> device rank word of a fresh QR factor
        self._deferred = []  # (ranks key, DevLR) trimmed at the end of the pass
        self._final = None   # frozen (key, DevLR, padded V, U, E) after the first trim
        self.graph = None
        self.launches = None
        self._wterms = []    # flop terms coef * w * r whose widths may be sketch-padded
        self._price = {}     # data_ptr of a final-product operand -> its U (re-priced at rank)
        # multi-GPU split of the shared top separators (distributed.factorize_distributed):
        # (rank, world, owner rank of every source id, process group) -- each rank
        # launches only the source terms of the sources it owns, rank 0 the A-matrix
        # and root-path terms, and every accumulated block is all-reduced before the
        # step that consumes it.  Flop accounting always covers the full sums.
        self.split = None

    def _mine(self, sids):
        """Mask of the source terms this rank launches (all of them when not split)."""
        if self.split is None:
            return np.ones(len(sids), dtype=bool)
        rank, _, owner, _ = self.split
        return owner[np.asarray(sids, dtype=np.int64)] == rank

    def _lead(self):
        """This rank launches the A-matrix and root-path terms."""
        return self.split is None or self.split[0] == 0

    def _reduce(self, tensors):
        """Sum the per-rank partial blocks (NCCL all-reduce; gloo stages via the host)."""
        if self.split is None:
            return
        import torch.distributed as dist

        group = self.split[3]
        for t in tensors:
            if t is None or t.numel() == 0:
                continue
            if t.is_cuda and dist.get_backend(group) == "gloo":
                h = t.cpu()
                dist.all_reduce(h, group=group)
                t.copy_(h)
            else:
                dist.all_reduce(t, group=group)

    def _wflops(self, coef, w=1, wbase=0, r=1, rbase=0):
        """Count flops coef * w * r where w is a source panel's width (panel base
        pointer wbase) and r the width of the block being formed (its U at rbase, for
        final products).  Compressed panels are sketch-padded during the pass;
        _finalize_ranks re-prices these terms at the kept ranks so model_gflop stays
        the reference's work model.  Off unless RSC_FLOP_MODEL=1 (census.py is the
        reference work model the bench reports; this per-launch bookkeeping costs
        host time on the one-shot path)."""
        if not FLOP_MODEL:
            return
        if np.ndim(coef) == 0 and np.ndim(w) == 0 and np.ndim(r) == 0:
            self.flops += float(coef) * float(w) * float(r)
            if wbase or rbase:
                self._wterms.append(tuple(np.array([v], dtype=t) for v, t in (
                    (coef, np.float64), (w, np.int64), (wbase, np.uint64), (r, np.int64), (rbase, np.uint64))))
            return
        coef, w, wbase, r, rbase = np.broadcast_arrays(
            np.asarray(coef, dtype=np.float64), np.asarray(w, dtype=np.int64), np.asarray(wbase, dtype=np.uint64),
            np.asarray(r, dtype=np.int64), np.asarray(rbase, dtype=np.uint64))
        self.flops += float(np.sum(coef * w * r))
        self._wterms.append((coef.copy(), w.copy(), wbase.copy(), r.copy(), rbase.copy()))

    def _set_source(self, sid, raw, eff):
        self.src_panel[sid] = (raw, eff)
        self.s_raw[sid] = raw.data_ptr()
        self.s_eff[sid] = eff.data_ptr()
        self.s_ld[sid] = E.ld(raw)
        self.s_w[sid] = raw.shape[1]

    def _pairs(self, j, need_rd=True, need_ro=False):
        """Flat descriptor arrays of target j's source pairs (widths > 0)."""
        t = self.np.tarr[j]
        s = t["s"]
        keep = self.s_w[s] > 0
        if need_rd:
            keep &= t["nrd"] > 0
        if need_ro:
            keep &= t["nro"] > 0
        return {k: v[keep] for k, v in t.items()}

    # -- batched primitives ----------------------------------------------------
    def _interior_mats(self, ints):
        blocks = []
        for (u, ids, c0, c1, off_rows, A_off, A_BB) in ints:
            blocks.append((A_BB, c1 - c0, c1 - c0))
            blocks.append((A_off, off_rows.size, c1 - c0))
        D = self._dense_many(blocks)
        return D[0::2], D[1::2]

    def _dense_many(self, blocks):
        """[(csr block or None, nrows, ncols)] -> persistent dense tensors (one launch)."""
        outs, rp, ci, va, nr, dp, ld = [], [], [], [], [], [], []
        mats = self.P.zeros_many([(m, n) for _, m, n in blocks])
        for (blk, m, n), D in zip(blocks, mats):
            outs.append(D)
            if blk is not None and blk.nnz and m and n:
                rp.append(blk.indptr_ptr)
                ci.append(blk.indices_ptr)
                va.append(blk.data_ptr)
                nr.append(blk.nrows)
                dp.append(D.data_ptr())
                ld.append(E.ld(D))
        if nr and self._lead():
            E.csr_to_dense_batched(rp, ci, va, nr, dp, ld)
        return outs

    def _potrf_many(self, mats_units):
        mats_units = [(M, u) for M, u in mats_units]
        tris = []
        live = []
        for M, u in mats_units:
            n = M.shape[0]
            tris.append(DenseTri(M, self.P.empty(max(n, 1), 64)))
            if n:
                live.append((M, u, tris[-1]))
            self.flops += n**3 / 3.0
        if live:
            info = self._ints(len(live))
            E.potrf_batched([M.data_ptr() for M, _, _ in live], [M.shape[0] for M, _, _ in live],
                            [E.ld(M) for M, _, _ in live], [t.Dinv.data_ptr() for _, _, t in live], info)
            base = self.ipos - len(live)
            for i, (_, u, _) in enumerate(live):
                self.pending.append((base + i, 1, u, self._trees_before(u)))
        return tris

    def _spmm_many(self, items, alpha=1.0, beta=0.0):
        """items: (csr block or None, X, Y) -> Y = alpha S X + beta Y."""
        rp, ci, va, nr, rr, xp, lx, yp, ly = [], [], [], [], [], [], [], [], []
        for blk, X, Y in items:
            if Y.numel() == 0:
                continue
            if blk is None or blk.nrows == 0 or X.shape[1] == 0:
                if beta == 0.0:
                    Y.zero_()
                continue
            rp.append(blk.indptr_ptr)
            ci.append(blk.indices_ptr)
            va.append(blk.data_ptr)
            nr.append(blk.nrows)
            rr.append(int(X.shape[1]))
            xp.append(X.data_ptr())
            lx.append(E.ld(X))
            yp.append(Y.data_ptr())
            ly.append(E.ld(Y))
            self._wflops(2.0 * blk.nnz, r=X.shape[1], rbase=self._price.get(X.data_ptr(), 0))
        if nr and not self._lead():
            if beta == 0.0:
                for Y in [it[2] for it in items]:
                    if Y.numel():
                        Y.zero_()
            return
        if nr:
            lib = E.require_cuda()
            from ._lib import int_array, ptr_array

            a = [ptr_array(rp), ptr_array(ci), ptr_array(va), int_array(nr), int_array(rr), ptr_array(xp),
                 int_array(lx), ptr_array(yp), int_array(ly)]
            E.check(lib.rsc_spmm_csr_batched(len(nr), a[0].ctypes.data, a[1].ctypes.data, a[2].ctypes.data,
                                             a[3].ctypes.data, a[4].ctypes.data, a[5].ctypes.data,
                                             a[6].ctypes.data, float(alpha), float(beta), a[7].ctypes.data,
                                             a[8].ctypes.data, E.stream_handle()), "rsc_spmm_csr_batched")

    def _orth_many(self, Gs):
        """One batched pivoted QR over all sketches.  The orthonormal factors are kept
        at sketch width with exact zero columns past the rank (rsc_qrcp_batched zeroes
        them), so nothing downstream needs the ranks on the host: they are read back
        once, at the end of the pass, to trim the stored blocks (_finalize_ranks)."""
        Us = [None] * len(Gs)
        live = [(i, G) for i, G in enumerate(Gs) if G.shape[0] and G.shape[1]]
        for i, G in enumerate(Gs):
            if not (G.shape[0] and G.shape[1]):
                Us[i] = self.P.empty(G.shape[0], 0)
        if not live:
            return Us
        Qs = [self.P.empty(*G.shape) for _, G in live]
        base = self.ipos
        rank = self._ints(len(live))
        E.qrcp_batched([G.data_ptr() for _, G in live], [G.shape[0] for _, G in live],
                       [G.shape[1] for _, G in live], [E.ld(G) for _, G in live], [Q.data_ptr() for Q in Qs],
                       [E.ld(Q) for Q in Qs], rank, alloc=self.S.empty)
        for j, ((i, G), Q) in enumerate(zip(live, Qs)):
            Us[i] = Q
            self._uslot[id(Q)] = base + j
            self.flops += 4.0 * G.shape[0] * G.shape[1] ** 2
        return Us

    def _lowrank_many(self, VUs):
        out = []
        g1, g2 = Grouped(True, False), Grouped(False, False)
        # U^T U has a tall K (the rows of U) and few tiles: accumulate it into zeroed
        # buffers so balance_k can split that K across CTAs
        utus = self.S.zeros_many([(max(U.shape[1], 1), max(U.shape[1], 1)) for _, U in VUs])
        for (V, U), utu in zip(VUs, utus):
            k = U.shape[1]
            Eff = self.P.empty(V.shape[0], k)
            if k:
                g1.add(U.data_ptr(), E.ld(U), U.data_ptr(), E.ld(U), utu.data_ptr(), k, k, k, U.shape[0], 1.0, 0.0,
                       atomic=1)
                g2.add(V.data_ptr(), E.ld(V), utu.data_ptr(), k, Eff.data_ptr(), E.ld(Eff), V.shape[0], k, k,
                       1.0, 0.0)
            lr = DevLR(V, U, Eff)
            lr.kslot = self._uslot.pop(id(U), None)
            out.append(lr)
        g1.launch()
        g2.launch()
        return out

    # -- dense-diagonal nodes ---------------------------------------------------
    def assemble_many(self, items):
        """items: (node, want_diag, want_off) -> [(UD or None, UO or None)] with all
        Schur updates of all nodes in one grouped launch (factor.py:372-399)."""
        blocks, layout = [], []
        for node, wd, wo in items:
            A_CC, A_RC, _ = self.np.node_blocks[node.j]
            nc, R = node.ncols, node.rows
            wo = wo and R.size > 0
            layout.append((len(blocks) if wd else None, len(blocks) + (1 if wd else 0) if wo else None))
            if wd:
                blocks.append((A_CC, nc, nc))
            if wo:
                blocks.append((A_RC, R.size, nc))
        dense = self._dense_many(blocks)
        out = []
        # every (node, source) pair of the batch in one set of flat arrays; problems
        # of different targets may interleave (the ordered reduction groups them by
        # target and keeps each target's sources in reference order)
        cols = {k: [] for k in ("s", "lo", "hi", "nrd", "nro", "cpos", "rpos")}
        per = {k: [] for k in ("ud", "uo", "nc", "nr", "cnt")}
        for (node, wd, wo), (iD, iO) in zip(items, layout):
            UD = dense[iD] if iD is not None else None
            UO = dense[iO] if iO is not None else None
            out.append((UD, UO))
            t = self.np.tarr[node.j]
            for k in cols:
                cols[k].append(t[k])
            per["ud"].append(UD.data_ptr() if UD is not None else 0)
            per["uo"].append(UO.data_ptr() if UO is not None else 0)
            per["nc"].append(node.ncols)
            per["nr"].append(UO.shape[0] if UO is not None else 0)
            per["cnt"].append(t["s"].size)
        if not items or sum(per["cnt"]) == 0:
            self._reduce([t for pair in out for t in pair])
            return out
        c = {k: np.concatenate(v) for k, v in cols.items()}
        cnt = np.asarray(per["cnt"], dtype=np.int64)
        ud = np.repeat(np.asarray(per["ud"], dtype=np.uint64), cnt)
        uo = np.repeat(np.asarray(per["uo"], dtype=np.uint64), cnt)
        nc = np.repeat(np.asarray(per["nc"], dtype=np.int64), cnt)
        nr = np.repeat(np.asarray(per["nr"], dtype=np.int64), cnt)
        s_ = c["s"]
        w, ld = self.s_w[s_], self.s_ld[s_]
        base = (w > 0) & (c["nrd"] > 0) & self._mine(s_)
        cpos = self.idx_base + (4 * c["cpos"]).astype(np.uint64)
        Qp = self.s_raw[s_] + (8 * c["lo"] * ld).astype(np.uint64)
        probs = []
        for which in ("ud", "uo"):
            tgt = ud if which == "ud" else uo
            sel = base & (tgt != 0)
            if which == "uo":
                sel &= c["nro"] > 0
            n = int(sel.sum())
            if n == 0:
                continue
            p = np.zeros(n, dtype=GEMM_DTYPE)
            row0 = c["lo"] if which == "ud" else c["hi"]
            ldk = ld[sel]
            p["A"] = self.s_eff[s_[sel]] + (8 * row0[sel] * ldk).astype(np.uint64)
            p["lda"], p["ldb"] = ldk, ldk
            p["B"], p["C"], p["ldc"] = Qp[sel], tgt[sel], nc[sel]
            p["M"] = c["nrd"][sel] if which == "ud" else c["nro"][sel]
            p["N"], p["K"] = c["nrd"][sel], w[sel]
            p["c_rows"] = cpos[sel] if which == "ud" else self.idx_base + (4 * c["rpos"][sel]).astype(np.uint64)
            p["c_cols"] = cpos[sel]
            p["batch"], p["atomic"], p["alpha"], p["beta"] = 1, 1, -1.0, 1.0
            p["ext_r"] = nc[sel] if which == "ud" else nr[sel]
            p["ext_c"] = nc[sel]
            self._wflops(2.0 * p["M"] * p["N"], w=p["K"], wbase=self.s_raw[s_[sel]])
            probs.append(p)
        if probs:
            P = E.gcat(probs)
            if P.size:
                E.gemm_balanced(P, False, True)
        self._reduce([t for pair in out for t in pair])
        return out

    # -- implicit products, batched over nodes -----------------------------------
    def off_mul_many(self, nodes, Gs, final=False):
        Ws, G1s, sol = [], [], []
        for node, G in zip(nodes, Gs):
            R = node.rows
            r = G.shape[1]
            W = (self.P if final else self.S).empty(R.size, r)
            Ws.append(W)
            G1 = self.S.empty(*G.shape)
            if G.numel():
                G1.copy_(G)
            G1s.append(G1)
            sol.append((node, G1, True))
            rb = G.data_ptr() if final else 0
            if final:
                self._price[G1.data_ptr()] = rb
            self._wflops(node.ncols**2, r=r, rbase=rb)
        diag_solve_many(sol, self.S.empty)
        self._spmm_many([(self.np.node_blocks[n.j][1], G1, W) for n, G1, W in zip(nodes, G1s, Ws)])
        self._products_many(nodes, G1s, Ws, trans=False)
        self._reduce(Ws)
        self._price.clear()
        return Ws

    def off_mul_t_many(self, nodes, Gs):
        Ws = [self.S.empty(n.ncols, G.shape[1]) for n, G in zip(nodes, Gs)]
        self._spmm_many([(self.np.node_blocks[n.j][2], G, W) for n, G, W in zip(nodes, Gs, Ws)])
        self._products_many(nodes, Gs, Ws, trans=True)
        self._reduce(Ws)
        diag_solve_many([(n, W, False) for n, W in zip(nodes, Ws)], self.S.empty)
        for n, W in zip(nodes, Ws):
            self.flops += n.ncols**2 * W.shape[1]
        return Ws

    def _products_many(self, nodes, Gs, Ws, trans):
        """Source terms of Alg. 2 (trans=False: W[rpos] -= E[hi:] (V[lo:hi]^T G[cpos]))
        or its mirror for all nodes: two grouped launches, descriptors built with
        numpy over every (node, source) pair at once."""
        parts = []
        for node, G, W in zip(nodes, Gs, Ws):
            r = G.shape[1]
            if r == 0 or W.numel() == 0:
                continue
            t = self._pairs(node.j, need_rd=True, need_ro=True)
            if t["s"].size == 0:
                continue
            parts.append((t, r, G.data_ptr(), E.ld(G), W.data_ptr(), E.ld(W), self._price.get(G.data_ptr(), 0),
                          W.shape[0], W.shape[1]))
        if not parts:
            return
        cat = lambda key: np.concatenate([p[0][key] for p in parts])
        s, lo, hi, nrd, nro = cat("s"), cat("lo"), cat("hi"), cat("nrd"), cat("nro")
        cpos = self.idx_base + (4 * cat("cpos")).astype(np.uint64)
        rpos = self.idx_base + (4 * cat("rpos")).astype(np.uint64)
        cnt = [p[0]["s"].size for p in parts]
        rep = lambda i: np.repeat(np.array([p[i] for p in parts]), cnt)
        r, gp, ldg, wp, ldw = rep(1), rep(2).astype(np.uint64), rep(3), rep(4).astype(np.uint64), rep(5)
        w, ld = self.s_w[s], self.s_ld[s]
        tsz = w * r
        toff = np.concatenate([[0], np.cumsum(tsz)[:-1]])
        T = self.S.zeros(int(tsz.sum()))  # p1 accumulates into it (K may be split)
        tp = np.uint64(T.data_ptr()) + (8 * toff).astype(np.uint64)
        raw_lo = self.s_raw[s] + (8 * lo * ld).astype(np.uint64)
        eff_hi = self.s_eff[s] + (8 * hi * ld).astype(np.uint64)
        n = s.size
        p1 = np.zeros(n, dtype=GEMM_DTYPE)
        p2 = np.zeros(n, dtype=GEMM_DTYPE)
        p1["B"], p1["ldb"], p1["C"], p1["ldc"], p1["M"], p1["N"] = gp, ldg, tp, r, w, r
        p1["lda"], p1["batch"], p1["alpha"] = ld, 1, 1.0
        p2["B"], p2["ldb"], p2["C"], p2["ldc"], p2["N"], p2["K"] = tp, r, wp, ldw, r, w
        p2["lda"], p2["batch"], p2["alpha"], p2["beta"], p2["atomic"] = ld, 1, -1.0, 1.0, 1
        p2["ext_r"], p2["ext_c"] = rep(7), rep(8)
        if not trans:  # T = V[lo:hi]^T G1[cpos] ; W[rpos] -= E[hi:] T
            p1["A"], p1["K"], p1["b_rows"] = raw_lo, nrd, cpos
            p2["A"], p2["M"], p2["c_rows"] = eff_hi, nro, rpos
        else:  # T = E[hi:]^T G[rpos] ; W[cpos] -= V[lo:hi] T
            p1["A"], p1["K"], p1["b_rows"] = eff_hi, nro, rpos
            p2["A"], p2["M"], p2["c_rows"] = raw_lo, nrd, cpos
        p1["atomic"] = 1  # T is zeroed: p1 accumulates, so its tall K may be split
        self._wflops(2.0 * (nrd + nro), w=w, wbase=self.s_raw[s], r=r, rbase=rep(6).astype(np.uint64))
        keep = self._mine(s)
        p1, p2 = p1[keep], p2[keep]
        if p1.size:
            E.gemm_balanced(p1, True, False)
            E.gemm_balanced(p2, False, False)

    def approx_off_many(self, nodes, ranks):
        """Alg. 3 for every compressed off-diagonal of the level (factor.py:486-505)."""
        if not nodes:
            return []
        Gs = []
        for node, rk in zip(nodes, ranks):
            R = node.rows
            rk = min(rk, R.size, node.ncols)
            Gs.append(self.sketches.device(("off", node.j), R.size, rk, self.S))
        Gs = self.off_mul_t_many(nodes, Gs)
        for _ in range(self.cfg.power_iters):
            Gs = self.off_mul_t_many(nodes, self.off_mul_many(nodes, Gs))
        Us = self._orth_many(Gs)
        Vs = self.off_mul_many(nodes, Us, final=True)
        return self._lowrank_many(list(zip(Vs, Us)))

    # -- diagonal trees, batched over trees ---------------------------------------
    def _path_probs(self, tree, s, rspan, cspan):
        """Earlier root-path blocks p < s of the tree: (raw, eff, ld, w, row lo/hi, col lo/hi)
        in block-local coordinates (diagblocks.py:265-273)."""
        out = []
        for raw, eff, a, b, c, d in self._path_terms(tree, s, rspan, cspan):
            w = raw.shape[1]
            if w:
                out.append((raw.data_ptr(), eff.data_ptr(), E.ld(raw), w, a, b, c, d))
        return out

    def _tmaps(self, j, s):
        t = self.np.tmap[(j, s)]
        keep = self.s_w[t["s"]] > 0
        return {k: v[keep] for k, v in t.items()}

    def leaves_many(self, items):
        """items: (node, s) leaf blocks -> DenseTri (Alg. 6, diagblocks.py:276-300):
        window of A, minus all windowed source products, minus root-path products,
        as one grouped launch; then one batched POTRF."""
        blocks = []
        for node, s in items:
            _, blk, _ = self.np.tree_maps[(node.j, s)]
            lf = node.diag.shape.nodes[s]
            k = lf.hi - lf.lo
            blocks.append((blk, k, k))
        Us = self._dense_many(blocks)
        parts, bases, keeps = [], [], []
        for (node, s), U in zip(items, Us):
            tree = node.diag
            lf = tree.shape.nodes[s]
            k = lf.hi - lf.lo
            t = self._tmaps(node.j, s)
            src = t["s"]
            if src.size:
                ld, w = self.s_ld[src], self.s_w[src]
                p = np.zeros(src.size, dtype=GEMM_DTYPE)
                p["A"] = self.s_eff[src] + (8 * t["rlo"] * ld).astype(np.uint64)
                p["B"] = self.s_raw[src] + (8 * t["clo"] * ld).astype(np.uint64)
                p["lda"], p["ldb"], p["K"] = ld, ld, w
                p["M"], p["N"] = t["rhi"] - t["rlo"], t["chi"] - t["clo"]
                p["c_rows"] = self.idx_base + (4 * t["ridx"]).astype(np.uint64)
                p["c_cols"] = self.idx_base + (4 * t["cidx"]).astype(np.uint64)
                p["C"], p["ldc"] = U.data_ptr(), k
                p["ext_r"], p["ext_c"] = k, k
                parts.append(p)
                bases.append(self.s_raw[src])
                keeps.append(self._mine(src))
            path = self._path_probs(tree, s, (lf.lo, lf.hi), (lf.lo, lf.hi))
            if path:
                p = np.zeros(len(path), dtype=GEMM_DTYPE)
                for i, (rawp, effp, ld, w, a0, a1, c0, c1) in enumerate(path):
                    p[i]["A"], p[i]["B"] = effp + 8 * a0 * ld, rawp + 8 * c0 * ld
                    p[i]["lda"], p[i]["ldb"], p[i]["K"], p[i]["M"], p[i]["N"] = ld, ld, w, a1 - a0, c1 - c0
                p["C"], p["ldc"] = U.data_ptr(), k
                p["ext_r"], p["ext_c"] = k, k
                parts.append(p)
                bases.append(np.array([pt[0] for pt in path], dtype=np.uint64))
                keeps.append(np.full(len(path), self._lead()))
        if parts:
            P = E.gcat(parts)
            P["batch"], P["atomic"], P["alpha"], P["beta"] = 1, 1, -1.0, 1.0
            self._wflops(2.0 * P["M"] * P["N"], w=P["K"], wbase=np.concatenate(bases))
            P = P[np.concatenate(keeps)]
            if P.size:
                E.gemm_balanced(P, False, True)
        self._reduce(Us)
        if LevelPass.fault_hook is not None and Us and LevelPass.fault_hook(self, items):
            Us[0][0, 0] = -1.0  # test hook: make the first leaf of this batch indefinite
        return self._potrf_many([(U, node.u) for (node, s), U in zip(items, Us)])

    def diag_mul_many(self, items, Gs, transpose, final=False):
        """Alg. 5 for several (node, s) internal blocks at once (diagblocks.py:303-346):
        batched left-subtree solves, grouped SpMM with the A windows, and all source and
        root-path terms of all blocks in two grouped launches."""
        mem = self.P if final else self.S
        Ws, srcs, sol, spm = [], [], [], []
        for (node, s), G in zip(items, Gs):
            shape = node.diag.shape
            (r0, r1), (c0, c1) = shape.span(s)
            _, blk, blkT = self.np.tree_maps[(node.j, s)]
            r = G.shape[1]
            if not transpose:
                G1 = self.S.empty(*G.shape)
                if G.numel():
                    G1.copy_(G)
                sol.append((node, G1, True, shape.nodes[s].left.s))
                rb = G.data_ptr() if final else 0
                if final:
                    self._price[G1.data_ptr()] = rb
                self._wflops((c1 - c0) ** 2, r=r, rbase=rb)
                W = mem.empty(r1 - r0, r)
                spm.append((blk, G1, W))
                srcs.append(G1)
            else:
                W = mem.empty(c1 - c0, r)
                spm.append((blkT, G, W))
                srcs.append(G)
            Ws.append(W)
        if sol:
            diag_solve_many(sol, self.S.empty)
        self._spmm_many(spm)
        # all source-window and root-path terms of all blocks as two flat problem sets
        # (per block: its pairs in reference order, then its path terms)
        acc = {k: [] for k in ("ld", "w", "base", "raw_c", "eff_r", "nc", "nr", "cidx", "ridx", "keep")}
        per = []  # (count, r, src ptr, ld src, W ptr, ld W, W rows, W cols, price)
        for (node, s), src, W in zip(items, srcs, Ws):
            tree = node.diag
            (r0, r1), (c0, c1) = tree.shape.span(s)
            r = src.shape[1]
            if r == 0 or W.numel() == 0:
                continue
            t = self._tmaps(node.j, s)
            sid = t["s"]
            ld = self.s_ld[sid]
            path = self._path_probs(tree, s, (r0, r1), (c0, c1))
            acc["ld"].append(ld)
            acc["w"].append(self.s_w[sid])
            acc["base"].append(self.s_raw[sid])
            acc["raw_c"].append(self.s_raw[sid] + (8 * t["clo"] * ld).astype(np.uint64))
            acc["eff_r"].append(self.s_eff[sid] + (8 * t["rlo"] * ld).astype(np.uint64))
            acc["nc"].append(t["chi"] - t["clo"])
            acc["nr"].append(t["rhi"] - t["rlo"])
            acc["cidx"].append(self.idx_base + (4 * t["cidx"]).astype(np.uint64))
            acc["ridx"].append(self.idx_base + (4 * t["ridx"]).astype(np.uint64))
            acc["keep"].append(self._mine(sid))
            if path:
                # (raw, eff, ld, w, row lo, row hi, col lo, col hi), window-aligned, no index maps
                pa = np.array(path, dtype=np.int64)
                acc["ld"].append(pa[:, 2])
                acc["w"].append(pa[:, 3])
                acc["base"].append(pa[:, 0].astype(np.uint64))
                acc["raw_c"].append((pa[:, 0] + 8 * pa[:, 6] * pa[:, 2]).astype(np.uint64))
                acc["eff_r"].append((pa[:, 1] + 8 * pa[:, 4] * pa[:, 2]).astype(np.uint64))
                acc["nc"].append(pa[:, 7] - pa[:, 6])
                acc["nr"].append(pa[:, 5] - pa[:, 4])
                acc["cidx"].append(np.zeros(len(path), np.uint64))
                acc["ridx"].append(np.zeros(len(path), np.uint64))
                acc["keep"].append(np.full(len(path), self._lead()))
            n = sid.size + len(path)
            if n:
                per.append((n, r, src.data_ptr(), E.ld(src), W.data_ptr(), E.ld(W), W.shape[0], W.shape[1],
                            self._price.get(src.data_ptr(), 0)))
        if per:
            c = {k: np.concatenate(v) for k, v in acc.items()}
            cnt = np.array([x[0] for x in per], dtype=np.int64)
            rep = lambda i, dt=np.int64: np.repeat(np.array([x[i] for x in per], dtype=dt), cnt)
            r_, sp, sld = rep(1), rep(2, np.uint64), rep(3)
            wp, wld, wr, wc = rep(4, np.uint64), rep(5), rep(6), rep(7)
            w, ld = c["w"], c["ld"]
            tsz = w * r_
            toff = np.cumsum(tsz) - tsz
            T = self.S.zeros(int(tsz.sum()))  # p1 accumulates into it (K may be split)
            tp = np.uint64(T.data_ptr()) + (8 * toff).astype(np.uint64)
            n = w.size
            p1 = np.zeros(n, dtype=GEMM_DTYPE)
            p2 = np.zeros(n, dtype=GEMM_DTYPE)
            p1["lda"], p1["M"], p1["N"], p1["C"], p1["ldc"] = ld, w, r_, tp, r_
            p1["B"], p1["ldb"] = sp, sld
            p2["lda"], p2["K"], p2["N"], p2["B"], p2["ldb"] = ld, w, r_, tp, r_
            p2["C"], p2["ldc"] = wp, wld
            p2["ext_r"], p2["ext_c"] = wr, wc
            if not transpose:  # T = V[cwin]^T G1[cidx] ; W[ridx] -= E[rwin] T
                p1["A"], p1["K"], p1["b_rows"] = c["raw_c"], c["nc"], c["cidx"]
                p2["A"], p2["M"], p2["c_rows"] = c["eff_r"], c["nr"], c["ridx"]
            else:  # T = E[rwin]^T G[ridx] ; W[cidx] -= V[cwin] T
                p1["A"], p1["K"], p1["b_rows"] = c["eff_r"], c["nr"], c["ridx"]
                p2["A"], p2["M"], p2["c_rows"] = c["raw_c"], c["nc"], c["cidx"]
            self._wflops(2.0 * (c["nc"] + c["nr"]), w=w, wbase=c["base"], r=r_, rbase=rep(8, np.uint64))
            keep = c["keep"]
            P1, P2 = p1[keep], p2[keep]
            P1["batch"], P1["alpha"] = 1, 1.0
            P2["batch"], P2["atomic"], P2["alpha"], P2["beta"] = 1, 1, -1.0, 1.0
            P1["atomic"] = 1  # T is zeroed: P1 accumulates, so its tall K may be split
            if P1.size:
                E.gemm_balanced(P1, True, False)
                E.gemm_balanced(P2, False, False)
        self._reduce(Ws)
        if transpose:
            sol2 = []
            for (node, s), W in zip(items, Ws):
                (r0, r1), (c0, c1) = node.diag.shape.span(s)
                sol2.append((node, W, False, node.diag.shape.nodes[s].left.s))
                self.flops += (c1 - c0) ** 2 * W.shape[1]
            diag_solve_many(sol2, self.S.empty)
        return Ws

    def approx_diag_many(self, items, ranks):
        Gs = []
        for (node, s), rk in zip(items, ranks):
            (r0, r1), (c0, c1) = node.diag.shape.span(s)
            rk = min(rk, r1 - r0, c1 - c0)
            Gs.append(self.sketches.device(("diag", node.j, s), r1 - r0, rk, self.S))
        Gs = self.diag_mul_many(items, Gs, True)
        for _ in range(self.cfg.power_iters):
            Gs = self.diag_mul_many(items, self.diag_mul_many(items, Gs, False), True)
        Us = self._orth_many(Gs)
        Vs = self.diag_mul_many(items, Us, False, final=True)
        return self._lowrank_many(list(zip(Vs, Us)))

    def trees_many(self, nodes):
        """Build every diagonal tree of the level, advancing all trees one in-order
        block position at a time (block s only needs blocks < s of its own tree)."""
        for node in nodes:
            node.diag = DeviceTree(self.np.tree_shapes[node.j])
            self.counters["diag_trees"] += 1
        maxlen = max((len(n.diag.shape.order) for n in nodes), default=0)
        for p in range(maxlen):
            self.S.reset()
            leaves, comp, comp_r, dense = [], [], [], []
            for node in nodes:
                order = node.diag.shape.order
                if p >= len(order):
                    continue
                s = order[p]
                tn = node.diag.shape.nodes[s]
                if tn.is_leaf:
                    leaves.append((node, s))
                    continue
                nrows, ncols = tn.hi - tn.split, tn.split - tn.lo
                r = block_rank(nrows, ncols, self.alpha_d, self.cfg.oversample)
                if r >= DENSE_FALLBACK_FRACTION * min(nrows, ncols):
                    dense.append((node, s))
                else:
                    comp.append((node, s))
                    comp_r.append(r)
            if leaves:
                for (node, s), tri in zip(leaves, self.leaves_many(leaves)):
                    node.diag.blocks[s] = tri
            if dense:
                eyes = []
                for node, s in dense:
                    tn = node.diag.shape.nodes[s]
                    ncols = tn.split - tn.lo
                    eye = self.S.zeros(ncols, ncols)
                    eye.fill_diagonal_(1.0)
                    eyes.append(eye)
                for (node, s), W in zip(dense, self.diag_mul_many(dense, eyes, False, final=True)):
                    node.diag.blocks[s] = W
                    self.counters["dense_fallback"] += 1
            if comp:
                for (node, s), lr in zip(comp, self.approx_diag_many(comp, comp_r)):
                    node.diag.blocks[s] = lr
                    self._deferred.append((("diag", node.j, s), lr))
                    self.counters["compressed_diag"] += 1

    # -- the sweep ------------------------------------------------------------------
    def _run(self):
        self._by_unit = {}
        self._run_units(None)
        self.units = [self._by_unit[u] for u in range(len(self.sym.units))]

    def _run_units(self, keep):
        """Sweep the units u with keep(u) (all when keep is None), in level order.
        The multi-GPU driver (distributed.factorize_distributed) runs the owned
        subtree units first and the shared top separators after the source exchange."""
        part = self.sym.partition
        cfg = self.cfg
        interiors = self.factor_interiors(defer=True, keep=keep)
        by_unit = self._by_unit
        for u, iu in interiors.items():
            by_unit[u] = iu
            sid = self.np.unit_source.get(u)
            if sid is not None:
                self._set_source(sid, iu.off, iu.off)
        for level in self.np.node_levels:
            if keep is not None:
                level = [u for u in level if keep(u)]
                if not level:
                    continue
            self.S.reset()
            nodes, trees, dense, off_dense, off_tree, comp, comp_r = [], [], [], [], [], [], []
            for u in level:
                j = self.sym.units[u][1]
                c0, c1 = part.cols(j)
                nc = c1 - c0
                R = part.rows[j]
                node = NodeUnit(u, j, c0, c1, R)
                nodes.append(node)
                by_unit[u] = node
                compress = bool(part.is_separator[j])
                tree_diag = compress and j in self.sym.sep_splits
                r_off = block_rank(R.size, nc, cfg.alpha_o, cfg.oversample)
                compress_off = bool(compress and R.size and r_off < DENSE_FALLBACK_FRACTION * min(R.size, nc))
                node._compress, node._compress_off = compress, compress_off
                (trees if tree_diag else dense).append(node)
                if R.size and compress_off:
                    comp.append(node)
                    comp_r.append(r_off)
                elif R.size:
                    (off_tree if tree_diag else off_dense).append(node)
            # dense diagonals (+ their dense off-diagonal blocks)
            if dense:
                asm = self.assemble_many([(n, True, not n._compress_off) for n in dense])
                tris = self._potrf_many([(UD, n.u) for n, (UD, UO) in zip(dense, asm)])
                for n, tri, (UD, UO) in zip(dense, tris, asm):
                    n.diag = tri
                    n._UO = UO
            # hierarchical diagonals
            if trees:
                self.trees_many(trees)
            self.S.reset()
            # dense off-diagonals
            if off_dense:
                lst = [n for n in off_dense]
                E.trsm_batched("right", 1, [n.diag.L.data_ptr() for n in lst], [n.ncols for n in lst],
                               [E.ld(n.diag.L) for n in lst], [n.diag.Dinv.data_ptr() for n in lst],
                               [n._UO.data_ptr() for n in lst], [n._UO.shape[0] for n in lst],
                               [E.ld(n._UO) for n in lst])
                for n in lst:
                    n.off = n._UO
                    self.flops += n.rows.size * n.ncols**2
            if off_tree:
                asm = self.assemble_many([(n, False, True) for n in off_tree])
                Xs = []
                for n, (_, UO) in zip(off_tree, asm):
                    X = self.S.empty(n.ncols, n.rows.size)
                    X.copy_(UO.t())
                    Xs.append(X)
                diag_solve_many([(n, X, False) for n, X in zip(off_tree, Xs)], self.S.empty)
                for n, X in zip(off_tree, Xs):
                    n.off = self.P.empty(n.rows.size, n.ncols)
                    n.off.copy_(X.t())
            for n in off_dense + off_tree:
                if n._compress:
                    self.counters["dense_fallback"] += 1
            # compressed off-diagonals
            if comp:
                for n, lr in zip(comp, self.approx_off_many(comp, comp_r)):
                    n.off = lr
                    self._deferred.append((("off", n.j), lr))
                    self.counters["compressed_off"] += 1
            for n in nodes:
                n._UO = None
                sid = self.np.unit_source.get(n.u)
                if sid is not None:
                    self._set_source(sid, *_raw_eff(n.off))

    def _finalize_ranks(self, info):
        """Trim every compressed block to its kept rank (views; the padded columns are
        exact zeros) and record the ranks -- the pass's single rank readback.  The
        padded tensors and the width-dependent flop terms are kept, so a CUDA-graph
        replay of the pass (new values, possibly new ranks) can trim again."""
        if self._final is None:
            self._final = [(key, lr, lr.V, lr.U, lr.E) for key, lr in self._deferred]
            self._deferred = []
            self._flops_padded = self.flops
            self._wt = tuple(np.concatenate([t[i] for t in self._wterms]) for i in range(5)) \
                if self._wterms else None
            self._wterms = []
        kept = {}
        self.ranks = {}
        for key, lr, V, U, Ef in self._final:
            k = int(info[lr.kslot]) if lr.kslot is not None else V.shape[1]
            kept[V.data_ptr()] = k
            kept[U.data_ptr()] = k
            lr.V, lr.U, lr.E, lr.k = V[:, :k], U[:, :k], Ef[:, :k], k
            self.ranks[key] = k
        self.flops = self._flops_padded
        kept.update(getattr(self, "extra_kept", {}))  # panels received from other ranks
        mark = getattr(self, "phase_mark", None)  # (padded flops, term count) after phase A
        if mark is not None:
            self.flops_phase_a = mark[0]
        if self._wt is not None and kept:
            coef, w, wb, r, rb = self._wt

            def look(bases, width):
                ub, inv = np.unique(bases, return_inverse=True)
                kk = np.array([kept.get(int(b), -1) for b in ub], dtype=np.int64)[inv]
                return np.where(kk >= 0, kk, width)

            wt, rt = look(wb, w), look(rb, r)
            d = coef * (w * r - wt * rt)
            self.flops -= float(np.sum(d))
            if mark is not None:
                self.flops_phase_a = mark[0] - float(np.sum(d[: mark[1]]))

    def mark_phase(self):
        """Record the flop-model position after the multi-GPU subtree phase."""
        self.phase_mark = (self.flops, int(sum(len(t[0]) for t in self._wterms)))

    def check_pivots(self):
        """One readback of the pass's device words (POTRF info + QR ranks): trim the
        compressed blocks, then resolve every recorded pivot failure (the earliest unit
        in sweep order wins)."""
        info = self.ibuf[: self.ipos].cpu().numpy()
        self._last_info = info
        self._finalize_ranks(info)
        worst = None
        for rec in self.pending:
            off, cnt, unit, trees = rec[:4]
            if off < 0:
                cand = (unit, rec[4], trees)
            else:
                v = info[off:off + cnt]
                bad = np.nonzero(v)[0]
                if not bad.size:
                    continue
                cand = (unit, int(v[bad[0]]) - 1, trees)
            if worst is None or cand[0] < worst[0]:
                worst = cand
        if worst is not None:
            raise _Indefinite(*worst)

    # -- CUDA-graph refactorization ---------------------------------------------------
    def capture(self):
        """Record the whole sweep (no host synchronisation inside) as one CUDA graph.
        Nothing executes until replay(); the Python structure of the factor (units,
        blocks, arenas) is built once here and stays valid for every replay, which
        rewrites the same device memory."""
        import torch

        from . import _lib

        lib = _lib.load()
        n0 = int(lib.rsc_launch_counter(0))
        self.graph = torch.cuda.CUDAGraph()
        prev = E.SCRATCH
        E.SCRATCH = self.S
        try:
            with torch.cuda.graph(self.graph):
                self._run()
        finally:
            E.SCRATCH = prev
        self.launches = int(lib.rsc_launch_counter(0)) - n0

    def replay(self):
        """Run the recorded sweep on the current values of the plan's A blocks, then
        the single readback (ranks + pivots)."""
        self.graph.replay()
        self.check_pivots()


# ---------------------------------------------------------------------------
# optional per-section device timing (active only under engine.PROFILE)


def _timed(name, fn):
    def wrap(*a, **k):
        with E.region(name):
            return fn(*a, **k)

    wrap.__name__ = fn.__name__
    wrap.__doc__ = fn.__doc__
    return wrap


for _name in ("_products_many", "_spmm_many", "_orth_many", "_lowrank_many", "assemble_many", "_potrf_many",
              "leaves_many", "factor_interiors", "diag_mul_many", "approx_off_many", "approx_diag_many",
              "trees_many"):
    setattr(LevelPass, _name, _timed(_name.strip("_"), getattr(LevelPass, _name)))
diag_solve_many = _timed("diag_solve", diag_solve_many)
