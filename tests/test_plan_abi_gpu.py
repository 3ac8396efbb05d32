"""Plan-level C-ABI entries (include/rsc_b200.h: rsc_schur_update,
rsc_offdiag_products, rsc_interior_factor_batched, rsc_tree_trsm, rsc_apply_sweep,
rsc_nccl_*) against numpy restatements of the reference steps and against the
package's own device factor."""
import ctypes

import numpy as np
import pytest

from conftest import relerr

pytestmark = pytest.mark.gpu


def _P(vals, ctype):
    return (ctype * len(vals))(*vals)


def _ptrs(ts):
    return _P([t.data_ptr() if t is not None else 0 for t in ts], ctypes.c_void_p)


def _ints(v):
    return _P([int(x) for x in v], ctypes.c_int)


def _sources(rng, nc, nr, nsrc):
    """Random update sources: panel pair (eff, raw) with a row run inside C_j
    (cpos) followed by rows beyond (rpos)."""
    src = []
    for _ in range(nsrc):
        nrd = int(rng.integers(1, nc))
        nro = int(rng.integers(1, nr))
        lo = int(rng.integers(0, 5))
        w = int(rng.integers(1, 40))
        rows = lo + nrd + nro + int(rng.integers(0, 3))
        raw, eff = rng.standard_normal((rows, w)), rng.standard_normal((rows, w))
        cpos = np.sort(rng.choice(nc, nrd, replace=False)).astype(np.int32)
        rpos = np.sort(rng.choice(nr, nro, replace=False)).astype(np.int32)
        src.append((eff, raw, w, lo, nrd, nro, cpos, rpos))
    return src


def _dev_sources(src):
    from paper_1507_05593_b200 import engine as E

    keep = []
    cols = {k: [] for k in ("eff", "raw", "ld", "w", "lo", "nrd", "nro", "cpos", "rpos")}
    for eff, raw, w, lo, nrd, nro, cpos, rpos in src:
        d = [E.to_dev(eff), E.to_dev(raw), E.to_dev(cpos), E.to_dev(rpos)]
        keep += d
        cols["eff"].append(d[0]); cols["raw"].append(d[1]); cols["cpos"].append(d[2]); cols["rpos"].append(d[3])
        cols["ld"].append(w); cols["w"].append(w); cols["lo"].append(lo); cols["nrd"].append(nrd)
        cols["nro"].append(nro)
    args = [_ptrs(cols["eff"]), _ptrs(cols["raw"]), _ints(cols["ld"]), _ints(cols["w"]), _ints(cols["lo"]),
            _ints(cols["nrd"]), _ints(cols["nro"]), _ptrs(cols["cpos"]), _ptrs(cols["rpos"])]
    return args, keep


def test_schur_update(cuda):
    """factor.py:383-398: UD[cpos,cpos] -= E V^T, UO[rpos,cpos] -= E_hi V^T, in source order."""
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(21)
    nc, nr = 70, 90
    src = _sources(rng, nc, nr, 7)
    UD0, UO0 = rng.standard_normal((nc, nc)), rng.standard_normal((nr, nc))
    UD, UO = UD0.copy(), UO0.copy()
    for eff, raw, w, lo, nrd, nro, cpos, rpos in src:
        V = raw[lo:lo + nrd]
        UD[np.ix_(cpos, cpos)] -= eff[lo:lo + nrd] @ V.T
        UO[np.ix_(rpos, cpos)] -= eff[lo + nrd:lo + nrd + nro] @ V.T
    E.ensure_gemm_workspace()
    dUD, dUO = E.to_dev(UD0), E.to_dev(UO0)
    args, keep = _dev_sources(src)
    lib = _lib.load()
    outs = []
    for _ in range(2):
        dUD.copy_(E.to_dev(UD0))
        dUO.copy_(E.to_dev(UO0))
        rc = lib.rsc_schur_update(dUD.data_ptr(), nc, nc, dUO.data_ptr(), nc, nr, len(src), *args,
                                  E.stream_handle())
        assert rc == 0
        outs.append((dUD.cpu().numpy(), dUO.cpu().numpy()))
    assert relerr(outs[0][0], UD) < 1e-13 and relerr(outs[0][1], UO) < 1e-13
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])  # ordered sums


@pytest.mark.parametrize("trans", [0, 1])
def test_offdiag_products(cuda, trans):
    """factor.py:444-455 / 471-482: the source terms of off_diagonal_multiply[_trans]."""
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(22 + trans)
    nc, nr, r = 60, 80, 11
    src = _sources(rng, nc, nr, 6)
    G = rng.standard_normal((nr if trans else nc, r))
    W0 = rng.standard_normal((nc if trans else nr, r))
    W = W0.copy()
    for eff, raw, w, lo, nrd, nro, cpos, rpos in src:
        V, Eh = raw[lo:lo + nrd], eff[lo + nrd:lo + nrd + nro]
        if not trans:
            W[rpos] -= Eh @ (V.T @ G[cpos])
        else:
            W[cpos] -= V @ (Eh.T @ G[rpos])
    E.ensure_gemm_workspace()
    dW, dG = E.to_dev(W0), E.to_dev(G)
    T = E.empty(sum(s[2] for s in src) * r)
    args, keep = _dev_sources(src)
    rc = _lib.load().rsc_offdiag_products(trans, dW.data_ptr(), r, W0.shape[0], r, dG.data_ptr(), r, r, len(src),
                                          *args, T.data_ptr(), E.stream_handle())
    assert rc == 0
    assert relerr(dW.cpu().numpy(), W) < 1e-13


def test_interior_factor_batched(cuda):
    """interior.py:105-156: L_B = chol(A_BB), Y_B = A(off_rows, C_B) L_B^{-T}."""
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(23)
    ns, ms = [17, 64, 150], [30, 0, 77]
    As, Ys = [], []
    for n, m in zip(ns, ms):
        G = rng.standard_normal((n, n))
        As.append(G @ G.T + n * np.eye(n))
        Ys.append(rng.standard_normal((m, n)))
    dA = [E.to_dev(a) for a in As]
    dY = [E.to_dev(y) if y.size else E.empty(1, n) for y, n in zip(Ys, ns)]
    dD = [E.empty(n, 64) for n in ns]
    info = E.zeros(len(ns), dtype=E.I32)
    rc = _lib.load().rsc_interior_factor_batched(len(ns), _ptrs(dA), _ints(ns), _ints(ns), _ptrs(dD), _ptrs(dY),
                                                 _ints(ms), _ints(ns), info.data_ptr(), E.stream_handle())
    assert rc == 0
    assert not info.cpu().numpy().any()
    for a, y, da, dy, n, m in zip(As, Ys, dA, dY, ns, ms):
        L = np.linalg.cholesky(a)
        assert relerr(np.tril(da.cpu().numpy()), L) < 1e-13
        if m:
            assert relerr(dy.cpu().numpy()[:m], np.linalg.solve(L, y.T).T) < 1e-12


def _factor_with_trees():
    from paper_1507_05593_b200 import factorize
    from paper_1507_05593_b200.factor import DeviceTree, SolverConfig
    from paper_1507_05593_b200.problems import laplacian_3d

    A, coords = laplacian_3d(14)
    F = factorize(A, SolverConfig(tau_o=32, oversample=10, tau_d=48), coords=coords)
    trees = [u.diag for u in F.dunits if isinstance(u.diag, DeviceTree)]
    assert trees
    return F, trees


@pytest.mark.parametrize("trans", [0, 1])
def test_tree_trsm_matches_device_tree(cuda, trans):
    """Alg. 4 (diagblocks.py:192-273) through the C-ABI vs DeviceTree.solve."""
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E
    from paper_1507_05593_b200.factor import DevLR

    F, trees = _factor_with_trees()
    lib = _lib.load()
    rng = np.random.default_rng(24 + trans)
    for tree in trees[:4]:
        sh = tree.shape
        ids = sorted(sh.nodes)
        pos = {s: i for i, s in enumerate(ids)}
        lo, hi, split, left, right = [], [], [], [], []
        L, ldl, Dinv, B, ldb, V, U, ldv, ldu, k = [], [], [], [], [], [], [], [], [], []
        kmax = 1
        for s in ids:
            nd, b = sh.nodes[s], tree.blocks[s]
            lo.append(nd.lo); hi.append(nd.hi)
            split.append(-1 if nd.is_leaf else nd.split)
            left.append(pos[nd.left.s] if not nd.is_leaf else -1)
            right.append(pos[nd.right.s] if not nd.is_leaf else -1)
            if nd.is_leaf:
                L.append(b.L); ldl.append(E.ld(b.L)); Dinv.append(b.Dinv)
                B.append(None); ldb.append(1); V.append(None); U.append(None); ldv.append(1); ldu.append(1); k.append(0)
            else:
                L.append(None); ldl.append(1); Dinv.append(None)
                if isinstance(b, DevLR):
                    B.append(None); ldb.append(1); V.append(b.V); U.append(b.U)
                    ldv.append(E.ld(b.V)); ldu.append(E.ld(b.U)); k.append(b.k); kmax = max(kmax, b.k)
                else:
                    B.append(b); ldb.append(E.ld(b)); V.append(None); U.append(None); ldv.append(1); ldu.append(1)
                    k.append(0)
        n, r = sh.ncols, 5
        X0 = rng.standard_normal((n, r))
        Xr = E.to_dev(X0)
        tree.solve(Xr, transpose=bool(trans))
        Xc = E.to_dev(X0)
        tws = E.empty(kmax * r)
        rc = lib.rsc_tree_trsm(trans, len(ids), pos[sh.root.s], _ints(lo), _ints(hi), _ints(split), _ints(left),
                               _ints(right), _ptrs(L), _ints(ldl), _ptrs(Dinv), _ptrs(B), _ints(ldb), _ptrs(V),
                               _ptrs(U), _ints(ldv), _ints(ldu), _ints(k), Xc.data_ptr(), r, r, tws.data_ptr(),
                               E.stream_handle())
        assert rc == 0
        assert relerr(Xc.cpu().numpy(), Xr.cpu().numpy()) < 1e-13


def test_apply_sweep_reproduces_device_apply(cuda, monkeypatch):
    """factor.py:175-218 through rsc_apply_sweep: the apply program's phases (forward
    then backward) replayed from flat C arrays give the package's apply."""
    import torch

    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E
    from paper_1507_05593_b200.apply import DeviceApply

    F, _ = _factor_with_trees()
    monkeypatch.setattr(DeviceApply, "TASK_BYTES", 0)  # phases only: the program is a flat sweep
    monkeypatch.setattr(DeviceApply, "TREE_CLUSTER", False)
    ap = DeviceApply(F)
    r = E.to_dev(np.random.default_rng(25).standard_normal(F.n))
    z_ref = E.empty(F.n)
    ap(r, z_ref)
    # the same program through the C-ABI: one flat array set over all phases
    cnt, cols = [], [[] for _ in range(10)]
    for n, arrs, _ in ap.launches:
        cnt.append(n)
        for i, a in enumerate(arrs):
            cols[i].extend(a.tolist())
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    flat = [_P(cols[0], P), _P(cols[1], I), _P(cols[2], I), _P(cols[3], I), _P(cols[4], P), _P(cols[5], P),
            _P(cols[6], P), _P(cols[7], P), _P(cols[8], I), _P(cols[9], D)]
    n = F.n
    ap.r_in.copy_(r)
    ap.tall.zero_()
    E.gather_rows(ap.inv, ap.r_in.reshape(n, 1), ap.y)
    rc = _lib.load().rsc_apply_sweep(len(cnt), _ints(cnt), *flat, E.stream_handle())
    assert rc == 0
    z = E.empty(n)
    E.gather_rows(ap.fwd, ap.y, z.reshape(n, 1))
    torch.cuda.synchronize()
    assert relerr(z.cpu().numpy(), z_ref.cpu().numpy()) < 1e-13


def test_nccl_single_rank(cuda):
    """NCCL wrappers on a one-rank communicator: all-reduce and broadcast are copies."""
    import torch

    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E

    lib = _lib.load()
    if not lib.rsc_nccl_available():
        pytest.skip("libnccl.so.2 not loadable")
    uid = ctypes.create_string_buffer(128)
    assert lib.rsc_nccl_unique_id(uid) == 0
    comm = ctypes.c_void_p()
    assert lib.rsc_nccl_comm_init(1, uid, 0, ctypes.byref(comm)) == 0
    x = E.to_dev(np.arange(1000, dtype=np.float64))
    y = E.empty(1000)
    assert lib.rsc_nccl_allreduce_sum_f64(comm, x.data_ptr(), y.data_ptr(), 1000, E.stream_handle()) == 0
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), np.arange(1000.0))
    y.zero_()
    assert lib.rsc_nccl_broadcast_f64(comm, x.data_ptr(), y.data_ptr(), 1000, 0, E.stream_handle()) == 0
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), np.arange(1000.0))
    assert lib.rsc_nccl_comm_destroy(comm) == 0
