"""Preconditioner application z = P^T (L L^T)^{-1} P r on the device
(reference factor.py:175-218).

Forward sweep over the units in factorization order: diagonal solve of the unit's
columns, then the coupling update y[R] -= L_O w (dense panel, materialized interior
coupling Y_B, or V (U^T w)); backward sweep mirrored.  With Y_B materialized the
interior branch (two in-block solves + sparse coupling, factor.py:189-194,206-210)
is the same operator as the dense branch, so every unit runs the same kernels.
"""

import numpy as np

from . import engine as E
from ._lib import GEMM_DTYPE
from .factor import DeviceTree, DevLR


class DeviceApply:
    def __init__(self, F):
        self.F = F
        self.n = F.n
        self.fwd = E.to_dev(np.asarray(F.perm.forward, dtype=np.int32))
        self.inv = E.to_dev(np.asarray(F.perm.inverse, dtype=np.int32))
        plan = F.plan
        self.rows_ptr = []
        for un in F.units:
            key = ("int", un.u) if un.kind == "interior" else un.j
            self.rows_ptr.append(plan.idx.ptr(plan.rows_off[key]))

    @staticmethod
    def _prob(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, b_rows=0, c_rows=0):
        p = np.zeros(1, dtype=GEMM_DTYPE)
        p["A"], p["B"], p["C"] = A, B, C
        p["lda"], p["ldb"], p["ldc"] = max(lda, 1), max(ldb, 1), max(ldc, 1)
        p["M"], p["N"], p["K"] = M, N, K
        p["alpha"], p["beta"], p["batch"] = alpha, beta, 1
        p["b_rows"], p["c_rows"] = b_rows, c_rows
        return p

    def __call__(self, r_dev, out=None):
        n = self.n
        r = r_dev.reshape(n, 1)
        y = E.empty(n, 1)
        E.gather_rows(self.inv, r, y)
        yp = y.data_ptr()
        units = self.F.units
        # forward
        for un, rp in zip(units, self.rows_ptr):
            w = y[un.c0:un.c1]
            self._diag_solve(un, w, False)
            m = un.rows.size
            if m == 0 or un.off is None:
                continue
            if isinstance(un.off, DevLR):
                k = un.off.k
                if k == 0:
                    continue
                t = E.empty(k, 1)
                E.gemm_grouped(self._prob(un.off.U.data_ptr(), E.ld(un.off.U), w.data_ptr(), 1, t.data_ptr(), 1,
                                          k, 1, un.ncols, 1.0, 0.0), True, False)
                E.gemm_grouped(self._prob(un.off.V.data_ptr(), E.ld(un.off.V), t.data_ptr(), 1, yp, 1, m, 1, k,
                                          -1.0, 1.0, c_rows=rp))
            else:
                E.gemm_grouped(self._prob(un.off.data_ptr(), E.ld(un.off), w.data_ptr(), 1, yp, 1, m, 1,
                                          un.ncols, -1.0, 1.0, c_rows=rp))
        # backward
        for un, rp in zip(reversed(units), reversed(self.rows_ptr)):
            w = y[un.c0:un.c1]
            m = un.rows.size
            if m and un.off is not None:
                if isinstance(un.off, DevLR):
                    k = un.off.k
                    if k:
                        t = E.empty(k, 1)
                        E.gemm_grouped(self._prob(un.off.V.data_ptr(), E.ld(un.off.V), yp, 1, t.data_ptr(), 1, k, 1,
                                                  m, 1.0, 0.0, b_rows=rp), True, False)
                        E.gemm_grouped(self._prob(un.off.U.data_ptr(), E.ld(un.off.U), t.data_ptr(), 1, w.data_ptr(),
                                                  1, un.ncols, 1, k, -1.0, 1.0))
                else:
                    E.gemm_grouped(self._prob(un.off.data_ptr(), E.ld(un.off), yp, 1, w.data_ptr(), 1, un.ncols, 1,
                                              m, -1.0, 1.0, b_rows=rp), True, False)
            self._diag_solve(un, w, True)
        z = out if out is not None else E.empty(n)
        E.gather_rows(self.fwd, y, z.reshape(n, 1))
        return z

    @staticmethod
    def _diag_solve(un, w, transpose):
        if isinstance(un.diag, DeviceTree):
            un.diag.solve(w, transpose)
        else:
            un.diag.solve(w, transpose)
