"""Preconditioner application z = P^T (L L^T)^{-1} P r on the device
(reference factor.py:175-218).

Forward sweep: per unit, a diagonal solve of its columns, then the coupling update
y[R] -= L_O w (dense panel, materialized interior coupling Y_B, or V (U^T w));
backward sweep mirrored.  With Y_B materialized the interior branch (two in-block
solves + sparse coupling, factor.py:189-194,206-210) is the same operator as the
dense branch, so every unit runs the same kernels.

Level scheduling: a unit depends only on the units whose rows reach into its
columns (its update sources), so units are grouped by height in that DAG.  Each
level is a handful of launches of the HBM-streaming kernels of csrc/apply.cu:
one batched TRSV over all dense diagonals of the level, one batched gather/scatter
GEMV for all dense couplings, two for all low-rank couplings, and the diagonal
trees of the level advanced in lock-step waves (Alg. 4 flattened).  All launch
descriptors are static after factorization and built once; after a few eager
applies the whole sweep is replayed from a CUDA graph.
"""

import numpy as np
import torch

from . import _lib
from . import engine as E
from ._lib import int_array, ptr_array
from .factor import DenseTri, DeviceTree, DevLR


class _Launch:
    """One pre-built batched launch (host descriptor arrays kept alive)."""

    def __init__(self, fn, arrays, scalars):
        self.fn = fn
        self.arrays = arrays
        self.args = [a.ctypes.data if isinstance(a, np.ndarray) else a for a in arrays] + scalars

    def __call__(self, stream):
        _lib.check(self.fn(*self.args, stream), "apply launch")


def _trsv(tris, xptrs, trans, y2p=None, yp=None):
    """Diagonal solves of a level.  With the explicit inverses built at apply setup,
    x = L^{-1} b is a row-parallel GEMV (warp per row, no dependency chain):
    forward reads Linv (lower), backward reads LinvT = Linv^T (upper), both from the
    snapshot y2 of y taken before the solves, writing y (assign)."""
    if not tris:
        return None
    if y2p is not None:
        M = [t.LinvT if trans else t.Linv for t in tris]
        items = [(m.data_ptr(), t.n, t.n, E.ld(m), y2p + (xp - yp), 0, xp, 0) for m, t, xp in zip(M, tris, xptrs)]
        return _gemv(items, 4 | (8 if trans else 2), 1.0)
    lib = _lib.load()
    arrs = [int(len(tris)), ptr_array([t.L.data_ptr() for t in tris]), int_array([t.n for t in tris]),
            int_array([E.ld(t.L) for t in tris]), ptr_array([t.Dinv.data_ptr() for t in tris]), ptr_array(xptrs)]
    return _Launch(lib.rsc_trsv_batched, arrs, [int(trans)])


def _gemv(items, trans, alpha):
    """items: (M ptr, rows, cols, ldm, x ptr, xidx ptr|0, y ptr, yidx ptr|0)."""
    if not items:
        return None
    lib = _lib.load()
    cols = list(zip(*items))
    arrs = [int(len(items)), ptr_array(cols[0]), int_array(cols[1]), int_array(cols[2]), int_array(cols[3]),
            ptr_array(cols[4]), ptr_array(cols[5]), ptr_array(cols[6]), ptr_array(cols[7])]
    return _Launch(lib.rsc_gemv_batched, arrs, [int(trans), float(alpha)])


class _Prog:
    """Ordered list of launches and zero-fills (a static program)."""

    def __init__(self):
        self.steps = []

    def launch(self, l):
        if l is not None:
            self.steps.append(l)

    def zero(self, t):
        if t is not None and t.numel():
            self.steps.append(("zero", t))

    def copy(self, dst, src):
        self.steps.append(("copy", dst, src))

    def run(self):
        s = E.stream_handle()
        for st in self.steps:
            if isinstance(st, tuple):
                if st[0] == "zero":
                    st[1].zero_()
                else:
                    st[1].copy_(st[2])
            else:
                st(s)


class DeviceApply:
    def __init__(self, F):
        # no strong reference back to the factor (it owns this program): a cycle would
        # keep the factor's device arena alive until the cyclic GC runs
        self.n = F.n
        plan = F.plan
        self.fwd = E.to_dev(np.asarray(F.perm.forward, dtype=np.int32))
        self.inv = E.to_dev(np.asarray(F.perm.inverse, dtype=np.int32))
        self.y = E.empty(self.n, 1)
        self.y2 = E.empty(self.n, 1)  # snapshot of y read by the inverse-based diagonal solves
        self.zbuf = E.empty(self.n)
        self.r_in = E.empty(self.n)
        self.keep = []
        units = F.units
        self._build_inverses(units)
        uidx = {un.u: i for i, un in enumerate(units)}
        level = [0] * len(units)
        for i, un in enumerate(units):
            if un.kind == "node":
                lv = 0
                for p in plan.targets[un.j]:
                    su = uidx[plan.sources[p.s].unit]
                    lv = max(lv, level[su] + 1)
                level[i] = lv
        nlev = max(level) + 1 if units else 0
        groups = [[units[i] for i in range(len(units)) if level[i] == lv] for lv in range(nlev)]
        self.prog = _Prog()
        for us in groups:
            self._forward_level(us, plan)
        for us in reversed(groups):
            self._backward_level(us, plan)
        self.graph = None
        self.calls = 0

    # -- program construction ------------------------------------------------------
    def _build_inverses(self, units):
        """Linv = L^{-1} (one batched TRSM against identities) and LinvT for every dense
        diagonal triangle and tree leaf: O(n^3/3) once per factor, after which every
        apply's diagonal solves are bandwidth-bound GEMVs.  The buffers hang on the
        triangles and are rewritten in place, so refresh_inverses() re-derives them
        after a graph replay has overwritten the factor with new values."""
        tris = []
        for u in units:
            if isinstance(u.diag, DenseTri):
                tris.append(u.diag)
            elif isinstance(u.diag, DeviceTree):
                tris.extend(b for s_, b in u.diag.blocks.items() if u.diag.shape.nodes[s_].is_leaf)
        self.tris = [t for t in tris if t.n]
        if any(t.Linv is None for t in self.tris):
            self.mem = E.Arena()
            for t in self.tris:
                if t.Linv is None:
                    t.Linv = self.mem.empty(t.n, t.n)
                    t.LinvT = self.mem.empty(t.n, t.n)
        self.refresh_inverses()

    def refresh_inverses(self):
        tris = self.tris
        if not tris:
            return
        for t in tris:
            t.Linv.zero_()
            t.Linv.fill_diagonal_(1.0)
        E.trsm_batched("left", 0, [t.L.data_ptr() for t in tris], [t.n for t in tris], [E.ld(t.L) for t in tris],
                       [t.Dinv.data_ptr() for t in tris], [t.Linv.data_ptr() for t in tris], [t.n for t in tris],
                       [t.n for t in tris])
        for t in tris:
            t.LinvT.copy_(t.Linv.t())

    def _rows_ptr(self, plan, un):
        key = ("int", un.u) if un.kind == "interior" else un.j
        return plan.idx.ptr(plan.rows_off[key])

    def _tbuf(self, sizes):
        """One zero-initialised buffer carved into per-problem t vectors."""
        tot = sum(sizes)
        if tot == 0:
            return None, []
        t = E.empty(tot)
        self.keep.append(t)
        offs = np.concatenate([[0], np.cumsum(sizes)[:-1]])
        return t, [t.data_ptr() + 8 * int(o) for o in offs]

    def _tree_waves(self, trees, trans):
        """Alg. 4 of every tree in `trees` on its slice of y, in lock-step waves."""
        from .numeric import tree_ops

        yp = self.y.data_ptr()
        seqs = [tree_ops(u.diag, None, self.y[u.c0:u.c1], trans) for u in trees]
        seqs = [s for s in seqs if s]
        if not seqs:
            return
        for w in range(max(len(s) for s in seqs)):
            leaves, dense, lr = [], [], []
            for s in seqs:
                if w >= len(s):
                    continue
                op = s[w]
                if op[0] == "leaf":
                    if op[1].n:
                        leaves.append((op[1], op[2].data_ptr()))
                    continue
                _, b, Xs, Yd, tr = op
                if isinstance(b, DevLR):
                    if b.k:
                        lr.append((b, Xs, Yd, tr))
                else:
                    dense.append((b, Xs, Yd, tr))
            if leaves:
                self.prog.copy(self.y2, self.y)
            self.prog.launch(_trsv([t for t, _ in leaves], [p for _, p in leaves], trans, self.y2.data_ptr(), yp))
            # dense coupling: Y -= B X (forward) or Y -= B^T X (transposed)
            self.prog.launch(_gemv([(b.data_ptr(), b.shape[0], b.shape[1], E.ld(b), Xs.data_ptr(), 0, Yd.data_ptr(), 0)
                                    for b, Xs, Yd, tr in dense], trans, -1.0))
            if lr:
                t, tp = self._tbuf([b.k for b, _, _, _ in lr])
                self.prog.zero(t)
                # t = U^T X (forward) or V^T X (transposed)
                first = [((b.V if tr else b.U), Xs, p) for (b, Xs, Yd, tr), p in zip(lr, tp)]
                self.prog.launch(_gemv([(P.data_ptr(), P.shape[0], P.shape[1], E.ld(P), Xs.data_ptr(), 0, p, 0)
                                        for P, Xs, p in first], 1, 1.0))
                # Y -= V t (forward) or U t (transposed)
                second = [((b.U if tr else b.V), Yd, p) for (b, Xs, Yd, tr), p in zip(lr, tp)]
                self.prog.launch(_gemv([(P.data_ptr(), P.shape[0], P.shape[1], E.ld(P), p, 0, Yd.data_ptr(), 0)
                                        for P, Yd, p in second], 0, -1.0))

    def _forward_level(self, us, plan):
        yp = self.y.data_ptr()
        dense = [u for u in us if isinstance(u.diag, DenseTri)]
        trees = [u for u in us if isinstance(u.diag, DeviceTree)]
        if dense:
            self.prog.copy(self.y2, self.y)
        self.prog.launch(_trsv([u.diag for u in dense], [yp + 8 * u.c0 for u in dense], 0, self.y2.data_ptr(), yp))
        if trees:
            self._tree_waves(trees, False)
        dn, lr = [], []
        for u in us:
            if not u.rows.size or u.off is None:
                continue
            if isinstance(u.off, DevLR):
                if u.off.k:
                    lr.append(u)
            else:
                dn.append(u)
        # y[R] -= L_O w
        self.prog.launch(_gemv([(u.off.data_ptr(), u.rows.size, u.ncols, E.ld(u.off), yp + 8 * u.c0, 0, yp,
                                 self._rows_ptr(plan, u)) for u in dn], 0, -1.0))
        if lr:
            t, tp = self._tbuf([u.off.k for u in lr])
            self.prog.zero(t)
            # t = U^T w ; y[R] -= V t
            self.prog.launch(_gemv([(u.off.U.data_ptr(), u.ncols, u.off.k, E.ld(u.off.U), yp + 8 * u.c0, 0, p, 0)
                                    for u, p in zip(lr, tp)], 1, 1.0))
            self.prog.launch(_gemv([(u.off.V.data_ptr(), u.rows.size, u.off.k, E.ld(u.off.V), p, 0, yp,
                                     self._rows_ptr(plan, u)) for u, p in zip(lr, tp)], 0, -1.0))

    def _backward_level(self, us, plan):
        yp = self.y.data_ptr()
        dn, lr = [], []
        for u in us:
            if not u.rows.size or u.off is None:
                continue
            if isinstance(u.off, DevLR):
                if u.off.k:
                    lr.append(u)
            else:
                dn.append(u)
        # w -= L_O^T y[R]
        self.prog.launch(_gemv([(u.off.data_ptr(), u.rows.size, u.ncols, E.ld(u.off), yp, self._rows_ptr(plan, u),
                                 yp + 8 * u.c0, 0) for u in dn], 1, -1.0))
        if lr:
            t, tp = self._tbuf([u.off.k for u in lr])
            self.prog.zero(t)
            # t = V^T y[R] ; w -= U t
            self.prog.launch(_gemv([(u.off.V.data_ptr(), u.rows.size, u.off.k, E.ld(u.off.V), yp,
                                     self._rows_ptr(plan, u), p, 0) for u, p in zip(lr, tp)], 1, 1.0))
            self.prog.launch(_gemv([(u.off.U.data_ptr(), u.ncols, u.off.k, E.ld(u.off.U), p, 0, yp + 8 * u.c0, 0)
                                    for u, p in zip(lr, tp)], 0, -1.0))
        trees = [u for u in us if isinstance(u.diag, DeviceTree)]
        if trees:
            self._tree_waves(trees, True)
        dense = [u for u in us if isinstance(u.diag, DenseTri)]
        if dense:
            self.prog.copy(self.y2, self.y)
        self.prog.launch(_trsv([u.diag for u in dense], [yp + 8 * u.c0 for u in dense], 1, self.y2.data_ptr(), yp))

    # -- execution ---------------------------------------------------------------
    def _body(self):
        n = self.n
        E.gather_rows(self.inv, self.r_in.reshape(n, 1), self.y)
        self.prog.run()
        E.gather_rows(self.fwd, self.y, self.zbuf.reshape(n, 1))

    # eager applies before the sweep is captured into a CUDA graph (capture costs
    # about two eager applies; PCG with 1-3 iterations never amortises it)
    GRAPH_AFTER = 3

    def __call__(self, r_dev, out=None):
        self.r_in.copy_(r_dev.reshape(-1))
        self.calls += 1
        if self.graph is None and self.calls > self.GRAPH_AFTER:
            try:
                s = torch.cuda.Stream()
                s.wait_stream(torch.cuda.current_stream())
                g = torch.cuda.CUDAGraph()
                with torch.cuda.stream(s):
                    with torch.cuda.graph(g, stream=s):
                        self._body()
                torch.cuda.current_stream().wait_stream(s)
                self.graph = g
            except Exception:
                self.graph = False
        if self.graph:
            self.graph.replay()
        else:
            self._body()
        z = out if out is not None else E.empty(self.n)
        z.copy_(self.zbuf)
        return z
