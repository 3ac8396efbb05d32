"""Preconditioner application z = P^T (L L^T)^{-1} P r on the device
(reference factor.py:175-218).

Forward sweep: per unit, a diagonal solve of its columns, then the coupling update
y[R] -= L_O w (dense panel, materialized interior coupling Y_B, or V (U^T w));
backward sweep mirrored.  With Y_B materialized the interior branch (two in-block
solves + sparse coupling, factor.py:189-194,206-210) is the same operator as the
dense branch, so every unit runs the same kernels.

Level scheduling: a unit depends only on the units whose rows reach into its
columns (its update sources), so units are grouped by height in that DAG and each
level runs as a handful of grouped launches -- batched TRSV over all dense
diagonals of the level, one grouped GEMV-scatter (FP64 atomics) for all dense
couplings, two for all low-rank couplings, and the diagonal trees of the level
advanced in lock-step waves (Alg. 4 flattened).  All problem descriptors are
static after factorization and are built once; the whole apply is then replayed
from a CUDA graph.
"""

import numpy as np
import torch

from . import engine as E
from ._lib import GEMM_DTYPE
from .factor import DenseTri, DeviceTree, DevLR


def _rows(probs):
    return np.array(probs, dtype=GEMM_DTYPE) if probs else None


def _p(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, b_rows=0, c_rows=0, atomic=0):
    return (A, B, C, 0, 0, 0, b_rows, c_rows, 0, M, N, K, max(lda, 1), max(ldb, 1), max(ldc, 1), 1, atomic,
            alpha, beta)


class _Trsv:
    """Batched triangular solves on vector slices (one rsc_trsm_batched call)."""

    def __init__(self, tris, ptrs, trans):
        self.trans = trans
        self.L = [t.L.data_ptr() for t in tris]
        self.n = [t.n for t in tris]
        self.ld = [E.ld(t.L) for t in tris]
        self.D = [t.Dinv.data_ptr() for t in tris]
        self.B = list(ptrs)

    def run(self):
        if self.L:
            E.trsm_batched("left", self.trans, self.L, self.n, self.ld, self.D, self.B, [1] * len(self.L),
                           [1] * len(self.L))


class DeviceApply:
    def __init__(self, F):
        self.F = F
        self.n = F.n
        plan = F.plan
        self.fwd = E.to_dev(np.asarray(F.perm.forward, dtype=np.int32))
        self.inv = E.to_dev(np.asarray(F.perm.inverse, dtype=np.int32))
        self.y = E.empty(self.n, 1)
        self.zbuf = E.empty(self.n)
        units = F.units
        # level of every unit = 1 + max level of its update sources
        uidx = {un.u: i for i, un in enumerate(units)}
        level = [0] * len(units)
        for i, un in enumerate(units):
            if un.kind == "node":
                lv = 0
                for p in plan.targets[un.j]:
                    su = uidx[plan.sources[p.s].unit]
                    lv = max(lv, level[su] + 1)
                level[i] = lv
        self.levels = []
        nlev = max(level) + 1 if units else 0
        yp = self.y.data_ptr()
        self.scratch = []
        for lv in range(nlev):
            idx = [i for i in range(len(units)) if level[i] == lv]
            self.levels.append(self._build_level([units[i] for i in idx], plan, yp))
        self.graph = None
        self.r_in = E.empty(self.n)

    def _rows_ptr(self, plan, un):
        key = ("int", un.u) if un.kind == "interior" else un.j
        return plan.idx.ptr(plan.rows_off[key])

    def _build_level(self, us, plan, yp):
        L = {}
        dense = [u for u in us if isinstance(u.diag, DenseTri)]
        trees = [u for u in us if isinstance(u.diag, DeviceTree)]
        L["fwd_diag"] = _Trsv([u.diag for u in dense], [yp + 8 * u.c0 for u in dense], 0)
        L["bwd_diag"] = _Trsv([u.diag for u in dense], [yp + 8 * u.c0 for u in dense], 1)
        L["trees"] = trees
        # coupling products
        fd, fl1, fl2, bd, bl1, bl2 = [], [], [], [], [], []
        lr = [u for u in us if isinstance(u.off, DevLR) and u.rows.size and u.off.k]
        tsz = sum(u.off.k for u in lr)
        t = E.empty(max(tsz, 1))
        self.scratch.append(t)
        toff = 0
        for u in us:
            m = u.rows.size
            if m == 0 or u.off is None:
                continue
            rp = self._rows_ptr(plan, u)
            w = yp + 8 * u.c0
            if isinstance(u.off, DevLR):
                k = u.off.k
                if k == 0:
                    continue
                tp = t.data_ptr() + 8 * toff
                toff += k
                V, U = u.off.V, u.off.U
                fl1.append(_p(U.data_ptr(), E.ld(U), w, 1, tp, 1, k, 1, u.ncols, 1.0, 0.0))
                fl2.append(_p(V.data_ptr(), E.ld(V), tp, 1, yp, 1, m, 1, k, -1.0, 1.0, c_rows=rp, atomic=1))
                bl1.append(_p(V.data_ptr(), E.ld(V), yp, 1, tp, 1, k, 1, m, 1.0, 0.0, b_rows=rp))
                bl2.append(_p(U.data_ptr(), E.ld(U), tp, 1, w, 1, u.ncols, 1, k, -1.0, 1.0))
            else:
                O = u.off
                fd.append(_p(O.data_ptr(), E.ld(O), w, 1, yp, 1, m, 1, u.ncols, -1.0, 1.0, c_rows=rp, atomic=1))
                bd.append(_p(O.data_ptr(), E.ld(O), yp, 1, w, 1, u.ncols, 1, m, -1.0, 1.0, b_rows=rp))
        L["fd"], L["fl1"], L["fl2"] = _rows(fd), _rows(fl1), _rows(fl2)
        L["bd"], L["bl1"], L["bl2"] = _rows(bd), _rows(bl1), _rows(bl2)
        return L

    @staticmethod
    def _g(probs, ta=False):
        if probs is not None:
            E.gemm_grouped(probs, ta, False)

    def _sweep(self):
        y = self.y
        from .numeric import run_waves, tree_ops

        for L in self.levels:
            L["fwd_diag"].run()
            if L["trees"]:  # Alg. 4 of every tree of the level in lock-step waves
                run_waves([tree_ops(u.diag, None, y[u.c0:u.c1], False) for u in L["trees"]], E.scratch)
            self._g(L["fd"])
            self._g(L["fl1"], True)
            self._g(L["fl2"])
        for L in reversed(self.levels):
            self._g(L["bd"], True)
            self._g(L["bl1"], True)
            self._g(L["bl2"])
            if L["trees"]:
                run_waves([tree_ops(u.diag, None, y[u.c0:u.c1], True) for u in L["trees"]], E.scratch)
            L["bwd_diag"].run()

    def _body(self):
        n = self.n
        E.gather_rows(self.inv, self.r_in.reshape(n, 1), self.y)
        self._sweep()
        E.gather_rows(self.fwd, self.y, self.zbuf.reshape(n, 1))

    # eager applies before the sweep is captured into a CUDA graph (capture costs
    # about two eager applies; PCG with 1-3 iterations never amortises it)
    GRAPH_AFTER = 3

    def __call__(self, r_dev, out=None):
        self.r_in.copy_(r_dev.reshape(-1))
        self.calls = getattr(self, "calls", 0) + 1
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
