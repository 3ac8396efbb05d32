"""GPU dense kernels vs the reference's golden vectors and KATs (through the C ABI)."""
import numpy as np
import pytest

from conftest import golden, relerr

pytestmark = pytest.mark.gpu


def test_gemm_grouped_all_transposes_and_maps(cuda):
    import torch
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(1)
    for ta in (False, True):
        for tb in (False, True):
            for (M, N, K) in [(1, 1, 1), (70, 33, 5), (129, 65, 200), (64, 64, 16), (3, 130, 0)]:
                A = rng.standard_normal((K, M) if ta else (M, K))
                B = rng.standard_normal((N, K) if tb else (K, N))
                C0 = rng.standard_normal((M, N))
                ref = 0.5 * ((A.T if ta else A) @ (B.T if tb else B)) - 2.0 * C0
                Cd = E.to_dev(C0)
                E.gemm(E.to_dev(A), E.to_dev(B), Cd, transA=ta, transB=tb, alpha=0.5, beta=-2.0)
                assert relerr(Cd.cpu().numpy(), ref) < 1e-14, (ta, tb, M, N, K)
    # gather on B rows + scatter into C rows/cols with atomics (two problems, same target)
    M, N, K = 40, 50, 30
    A = rng.standard_normal((M, K))
    Bbig = rng.standard_normal((100, N))
    brow = rng.choice(100, K, replace=False).astype(np.int32)
    crow = np.sort(rng.choice(90, M, replace=False)).astype(np.int32)
    ccol = np.sort(rng.choice(70, N, replace=False)).astype(np.int32)
    C = np.zeros((90, 70))
    Ad, Bd, Cd = E.to_dev(A), E.to_dev(Bbig), E.to_dev(C)
    idx = [E.to_dev(x) for x in (brow, crow, ccol)]
    p = E.gemm_problems(2)
    for i in range(2):
        p[i]["A"], p[i]["B"], p[i]["C"] = Ad.data_ptr(), Bd.data_ptr(), Cd.data_ptr()
        p[i]["b_rows"], p[i]["c_rows"], p[i]["c_cols"] = (t.data_ptr() for t in idx)
        p[i]["M"], p[i]["N"], p[i]["K"] = M, N, K
        p[i]["lda"], p[i]["ldb"], p[i]["ldc"] = K, N, 70
        p[i]["batch"], p[i]["atomic"], p[i]["alpha"] = 1, 1, -1.0
        p[i]["ext_r"], p[i]["ext_c"] = 90, 70
    E.gemm_grouped(p)
    ref = np.zeros((90, 70))
    ref[np.ix_(crow, ccol)] -= 2 * (A @ Bbig[brow])
    assert relerr(Cd.cpu().numpy(), ref) < 1e-14


def test_gemm_ordered_accumulation_deterministic(cuda):
    """Many accumulating problems scattered into shared targets (interleaved groups,
    split-K slabs, several chunks through a small workspace): the result equals the
    sequential sum C + P_1 + P_2 + ... in problem order, bit-identically on every
    launch (rsc_gemm_grouped's ordered reduction replaces FP64 atomics)."""
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(11)
    T = 3  # targets
    shapes = [(300, 120), (97, 64), (1000, 37)]
    C0 = [rng.standard_normal(s) for s in shapes]
    Cd = [E.to_dev(c) for c in C0]
    keep, probs, ref = [], [], [c.copy() for c in C0]
    for n in range(60):
        t = n % T
        er, ec = shapes[t]
        M, N, K = int(rng.integers(1, min(er, 130))), int(rng.integers(1, ec)), int(rng.integers(1, 300))
        rows = np.sort(rng.choice(er, M, replace=False)).astype(np.int32)
        cols = np.sort(rng.choice(ec, N, replace=False)).astype(np.int32)
        A, B = rng.standard_normal((M, K)), rng.standard_normal((K, N))
        dA, dB, dr, dc = E.to_dev(A), E.to_dev(B), E.to_dev(rows), E.to_dev(cols)
        keep += [dA, dB, dr, dc]
        q = E.gemm_problems(1)
        q["A"], q["B"], q["C"], q["c_rows"], q["c_cols"] = dA.data_ptr(), dB.data_ptr(), Cd[t].data_ptr(), \
            dr.data_ptr(), dc.data_ptr()
        q["M"], q["N"], q["K"], q["lda"], q["ldb"], q["ldc"] = M, N, K, K, N, ec
        q["batch"], q["atomic"], q["alpha"], q["beta"], q["ext_r"], q["ext_c"] = 1, 1, -0.5, 1.0, er, ec
        probs.append(q)
        ref[t][np.ix_(rows, cols)] += -0.5 * (A @ B)
    P = np.concatenate(probs)
    P = E.balance_k(P, False, False, ctas=8)  # force split-K slabs (kept in place)
    lib = _lib.load()
    outs = []
    for ws_mb in (512, 1):  # 1 MB: the launch is cut into several ordered chunks
        ws = E.empty((ws_mb << 20) // 8)
        E.check(lib.rsc_gemm_set_workspace(E.stream_handle(), ws.data_ptr(), ws_mb << 20, 0), "ws")
        for _ in range(3):
            for t in range(T):
                Cd[t].copy_(E.to_dev(C0[t]))
            E.gemm_grouped(P)
            outs.append([c.cpu().numpy() for c in Cd])
        E._GEMM_WS.pop(E.stream_handle(), None)
        E.ensure_gemm_workspace()
    E.check(lib.rsc_gemm_set_workspace(E.stream_handle(), E._GEMM_WS[E.stream_handle()].data_ptr(),
                                       E.GEMM_WS_BYTES, 0), "ws")
    for o in outs[1:]:
        for t in range(T):
            assert np.array_equal(o[t], outs[0][t])
    for t in range(T):
        assert relerr(outs[0][t], ref[t]) < 1e-14
    # the library-side K balancing (rsc_gemm_grouped_balanced) splits exactly like
    # engine.balance_k: bit-identical results
    P0 = np.concatenate(probs)
    for t in range(T):
        Cd[t].copy_(E.to_dev(C0[t]))
    E.gemm_balanced(P0, ctas=8)
    for t in range(T):
        assert np.array_equal(Cd[t].cpu().numpy(), outs[0][t])


def test_gemm_ordered_accumulation_row_mapped(cuda):
    """Accumulating problems scattered by row only, every partial as wide as its
    target (the sketch-product shape, ordered_reduce_kernel's row-sweep path),
    including repeated target rows whose extra products are exact zeros: equals the
    sequential sum in problem order, bit-identical on every launch."""
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(5)
    shapes = [(700, 64), (300, 130), (90, 1100)]  # 1100 > one row-sweep tile (1024 columns)
    C0 = [rng.standard_normal(sh) for sh in shapes]
    Cd = [E.to_dev(c) for c in C0]
    keep, probs, ref = [], [], [c.copy() for c in C0]
    for n in range(45):
        t = n % 3
        er, ec = shapes[t]
        M, K = int(rng.integers(1, min(er, 200))), int(rng.integers(1, 120))
        rows = np.sort(rng.choice(er, M, replace=False))
        A = rng.standard_normal((M, K))
        if n % 4 == 0 and M > 3:  # repeated target rows carrying exact-zero products
            rows[1:3] = rows[0]
            A[1:3] = 0.0
            rows = np.sort(rows)
            A[1:3] = 0.0
        rows = rows.astype(np.int32)
        B = rng.standard_normal((K, ec))
        dA, dB, dr = E.to_dev(A), E.to_dev(B), E.to_dev(rows)
        keep += [dA, dB, dr]
        q = E.gemm_problems(1)
        q["A"], q["B"], q["C"], q["c_rows"] = dA.data_ptr(), dB.data_ptr(), Cd[t].data_ptr(), dr.data_ptr()
        q["M"], q["N"], q["K"], q["lda"], q["ldb"], q["ldc"] = M, ec, K, K, ec, ec
        q["batch"], q["atomic"], q["alpha"], q["beta"], q["ext_r"], q["ext_c"] = 1, 1, 1.0, 1.0, er, ec
        probs.append(q)
        prod = A @ B
        for i, r in enumerate(rows):
            ref[t][r] += prod[i]
    P = np.concatenate(probs)
    outs = []
    for _ in range(3):
        for t in range(3):
            Cd[t].copy_(E.to_dev(C0[t]))
        E.gemm_grouped(P)
        outs.append([c.cpu().numpy() for c in Cd])
    for o in outs[1:]:
        for t in range(3):
            assert np.array_equal(o[t], outs[0][t])
    for t in range(3):
        assert relerr(outs[0][t], ref[t]) < 1e-14


def test_dense_cholesky_golden(cuda):
    from paper_1507_05593_b200 import kernels as K

    g = golden("kernels.npz")
    for n in (1, 7, 23, 50, 64, 65, 130, 256):
        assert relerr(K.dense_cholesky(g[f"chol_in_{n}"]), g[f"chol_out_{n}"]) < 1e-12, n


def test_dense_cholesky_kats(cuda):
    from paper_1507_05593_b200 import kernels as K
    from paper_1507_05593_b200.errors import IndefiniteError

    assert np.allclose(K.dense_cholesky(np.array([[4.0, 2.0], [2.0, 3.0]])), [[2, 0], [1, np.sqrt(2)]])
    assert np.allclose(K.dense_cholesky(np.array([[4.0, 99.0], [2.0, 3.0]])), [[2, 0], [1, np.sqrt(2)]])
    assert np.array_equal(K.dense_cholesky(np.eye(5)), np.eye(5))
    with pytest.raises(IndefiniteError) as e:
        K.dense_cholesky(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.pivot == 1
    with pytest.raises(IndefiniteError) as e:
        K.dense_cholesky(np.zeros((3, 3)))
    assert e.value.pivot == 0
    # pivot failure deep inside a later 64-block
    rng = np.random.default_rng(3)
    M = rng.standard_normal((150, 150))
    M = M @ M.T + 150 * np.eye(150)
    M[100, 100] = -1e6
    with pytest.raises(IndefiniteError) as e:
        K.dense_cholesky(M)
    assert e.value.pivot == 100
    assert K.dense_cholesky(np.zeros((0, 0))).shape == (0, 0)


def test_tri_solve_golden(cuda):
    from paper_1507_05593_b200 import kernels as K
    from paper_1507_05593_b200.errors import SingularDiagonal

    g = golden("kernels.npz")
    L, B = g["tri_L"], g["tri_B"]
    assert relerr(K.tri_solve(L, B), g["tri_left"]) < 1e-13
    assert relerr(K.tri_solve(L, B, transpose=True), g["tri_left_t"]) < 1e-13
    assert relerr(K.tri_solve(L, B.T, transpose=True, side="right"), g["tri_right_t"]) < 1e-13
    assert relerr(K.tri_solve(L, B.T, side="right"), g["tri_right"]) < 1e-13
    X = K.tri_solve(np.array([[2.0, 0.0], [1.0, 1.0]]), np.array([[2.0, 3.0]]), transpose=True, side="right")
    assert np.allclose(X, [[1, 2]])
    with pytest.raises(SingularDiagonal):
        K.tri_solve(np.array([[1.0, 0.0], [3.0, 0.0]]), np.ones((2, 1)))
    v = K.tri_solve(L, B[:, 0])
    assert v.shape == (150,) and relerr(v, g["tri_left"][:, 0]) < 1e-13


def test_orthonormalize_golden_ranks(cuda):
    from paper_1507_05593_b200 import kernels as K

    g = golden("kernels.npz")
    for tag in "abc":
        Q = K.orthonormalize(g[f"orth_in_{tag}"])
        Qr = g[f"orth_out_{tag}"]
        assert Q.shape == Qr.shape, tag
        assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() < 1e-13
        assert relerr(Q @ Q.T, Qr @ Qr.T) < 1e-10
    e1 = np.zeros((4, 1))
    e1[0] = 1.0
    Q = K.orthonormalize(np.hstack([e1, 2 * e1]))
    assert Q.shape == (4, 1) and abs(abs(Q[0, 0]) - 1) < 1e-14
    assert K.orthonormalize(np.zeros((5, 2))).shape == (5, 0)


def test_low_rank_approx_golden(cuda):
    from paper_1507_05593_b200 import kernels as K

    g = golden("kernels.npz")
    V, U = K.low_rank_approx(g["lra_in"], 30, power_iters=1, seed=5)
    assert U.shape == g["lra_U"].shape
    assert relerr(V @ U.T, g["lra_V"] @ g["lra_U"].T) < 1e-10
    rng = np.random.default_rng(2)
    B = np.outer(rng.standard_normal(30), rng.standard_normal(12))
    V, U = K.low_rank_approx(B, rank=4, seed=0)
    assert relerr(V @ U.T, B) < 1e-10
    V, U = K.low_rank_approx(np.zeros((10, 6)), rank=3, seed=0)
    assert np.linalg.norm(V @ U.T) == 0.0


@pytest.mark.parametrize("m,k,true_rank", [(1000, 300, None), (2100, 130, 90), (300, 700, 150)])
def test_orthonormalize_multi_cta_path(cuda, m, k, true_rank):
    """Sketches beyond one SM's shared memory go through the cooperative QR."""
    from oracle import kernels as ok
    from paper_1507_05593_b200 import kernels as K

    rng = np.random.default_rng(m + k)
    if true_rank is None:
        G = rng.standard_normal((m, k))
    else:
        G = rng.standard_normal((m, true_rank)) @ rng.standard_normal((true_rank, k)) + 1e-15 * rng.standard_normal(
            (m, k))
    Q = K.orthonormalize(G)
    Qo = ok.orth(G)
    assert Q.shape == Qo.shape
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() < 1e-12
    assert relerr(Q @ (Q.T @ G), Qo @ (Qo.T @ G)) < 1e-10


@pytest.mark.parametrize("m,k,true_rank", [(4096, 600, 250), (1000, 300, None), (30000, 96, 40),
                                             (8000, 1000, 300), (6000, 700, None)])
def test_orthonormalize_cooperative_kernel(cuda, monkeypatch, m, k, true_rank):
    """The cooperative multi-CTA QRCP itself (cluster path disabled): shared-memory
    column groups of ~100 CTAs (4096 x 600: more per-CTA pivot candidates than one
    warp's lanes) and the global-memory column path (30000 x 96: one column per CTA;
    8000 x 1000 and 6000 x 700: 5-7 columns per CTA, the CTA-cooperative update with
    the reflector staged in shared memory).  Kept rank exact,
    span to 1e-10 against the oracle."""
    from oracle import kernels as ok
    from paper_1507_05593_b200 import kernels as K

    monkeypatch.setenv("RSC_QR_NOCLUSTER", "1")
    rng = np.random.default_rng(m + 7 * k)
    if true_rank is None:
        G = rng.standard_normal((m, k))
    else:
        G = rng.standard_normal((m, true_rank)) @ rng.standard_normal((true_rank, k))
    Q = K.orthonormalize(G)
    Qo = ok.orth(G)
    assert Q.shape == Qo.shape
    assert np.abs(Q.T @ Q - np.eye(Q.shape[1])).max() < 1e-12
    assert relerr(Q @ (Q.T @ G), Qo @ (Qo.T @ G)) < 1e-10


def test_qrcp_batched_mixed_sizes_concurrent(cuda):
    """One batched call mixing one-CTA sketches and multi-CTA groups (run concurrently)."""
    import torch
    from oracle import kernels as ok
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(9)
    shapes = [(256, 58), (300, 120), (2048, 40), (700, 333), (64, 16), (1500, 210), (260, 101)]
    Gs = []
    for i, (m, k) in enumerate(shapes):
        r = min(m, k) if i % 2 == 0 else max(2, min(m, k) // 2)
        Gs.append(rng.standard_normal((m, r)) @ rng.standard_normal((r, k)))
    Gd = [E.to_dev(G) for G in Gs]
    Qd = [E.empty(*G.shape) for G in Gs]
    rank = E.zeros(len(Gs), dtype=E.I32)
    work = E.qrcp_batched([g.data_ptr() for g in Gd], [s[0] for s in shapes], [s[1] for s in shapes],
                          [s[1] for s in shapes], [q.data_ptr() for q in Qd], [s[1] for s in shapes], rank)
    torch.cuda.synchronize()
    ranks = rank.cpu().numpy()
    for i, G in enumerate(Gs):
        Qo = ok.orth(G)
        assert ranks[i] == Qo.shape[1], (i, ranks[i], Qo.shape)
        Q = Qd[i][:, :ranks[i]].cpu().numpy()
        assert relerr(Q @ (Q.T @ G), Qo @ (Qo.T @ G)) < 1e-10
    del work


@pytest.mark.parametrize("n", [1, 37, 64, 100, 256, 300, 320, 321, 400])
def test_trsm_right_fused_shapes(cuda, n):
    """X = B L^{-T} for a batch of panels with ragged m and n (the strip-resident kernel
    for n <= 320, the blocked path above), in place and out of place."""
    import torch

    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(n)
    ms = [1, 63, 64, 65, 700]
    Ls, Dinvs, Bs = [], [], []
    for m in ms:
        G = rng.standard_normal((n, n))
        A = G @ G.T / n + np.eye(n)
        Ad = E.to_dev(A)
        Dv = E.zeros(max(n, 1), 64)
        info = E.zeros(1, dtype=E.I32)
        E.potrf_batched([Ad.data_ptr()], [n], [n], [Dv.data_ptr()], info)
        Ls.append(Ad)
        Dinvs.append(Dv)
        Bs.append(rng.standard_normal((m, n)))
    Bd = [E.to_dev(B) for B in Bs]
    Xd = [torch.full_like(b, float("nan")) for b in Bd]
    args = ([L.data_ptr() for L in Ls], [n] * len(ms), [n] * len(ms), [d.data_ptr() for d in Dinvs])
    if n <= 320:
        E.trsm_right(*args, [b.data_ptr() for b in Bd], [x.data_ptr() for x in Xd], ms, [n] * len(ms))
    E.trsm_batched("right", 1, *args, [b.data_ptr() for b in Bd], ms, [n] * len(ms))  # in place
    torch.cuda.synchronize()
    for L, B, b, x in zip(Ls, Bs, Bd, Xd):
        Lh = np.tril(L.cpu().numpy())
        ref = np.linalg.solve(Lh, B.T).T  # B L^{-T}
        assert relerr(b.cpu().numpy(), ref) < 1e-12
        if n <= 320:
            assert np.array_equal(x.cpu().numpy(), b.cpu().numpy())  # same kernel, same bits
    if n > 320:
        from paper_1507_05593_b200 import _lib

        with pytest.raises(RuntimeError):
            E.trsm_right(*args, None, [b.data_ptr() for b in Bd], ms, [n] * len(ms))


def test_gemv_multi_modes_against_numpy(cuda):
    """rsc_gemv_multi: every mode (plain, transposed, lower/upper triangular, assign,
    gathers/scatters) on narrow / mid / wide panels, mixed in one launch."""
    import torch

    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200._lib import int_array, ptr_array

    lib = _lib.load()
    rng = np.random.default_rng(7)
    shapes = [(300, 7), (1000, 40), (257, 64), (65, 65), (500, 200), (130, 300), (64, 1000), (3, 2500)]
    items, refs = [], []
    keep = []
    for si, (r, c) in enumerate(shapes):
        for mode in (0, 1, 4, 6, 12):
            if mode in (6, 12) and r != c:
                rr = cc = min(r, c)
            else:
                rr, cc = r, c
            Mh = rng.standard_normal((rr, cc + 3))  # ld > cols
            trans = mode & 1
            xlen, ylen = (rr, cc) if trans else (cc, rr)
            xh = rng.standard_normal(xlen + 5)
            yh = rng.standard_normal(ylen + 5)
            xi = rng.permutation(xlen + 5)[:xlen].astype(np.int32) if si % 2 else None
            yi = rng.permutation(ylen + 5)[:ylen].astype(np.int32) if (si % 3 == 0 and not mode & 4) else None
            alpha = -1.5 if si % 2 else 0.75
            Mv = Mh[:, :cc]
            if mode & 2:
                Mv = np.tril(Mv)
            if mode & 8:
                Mv = np.triu(Mv)
            xv = xh[xi] if xi is not None else xh[:xlen]
            prod = (Mv.T @ xv) if trans else (Mv @ xv)
            ref = yh.copy()
            tgt = yi if yi is not None else np.arange(ylen)
            if mode & 4:
                ref[tgt] = alpha * prod
            else:
                ref[tgt] += alpha * prod
            Md, xd, yd = (torch.from_numpy(v).cuda() for v in (Mh, xh, yh))
            xid = torch.from_numpy(xi).cuda() if xi is not None else None
            yid = torch.from_numpy(yi).cuda() if yi is not None else None
            keep += [Md, xd, yd, xid, yid]
            items.append((Md.data_ptr(), rr, cc, cc + 3, xd.data_ptr(), xid.data_ptr() if xid is not None else 0,
                          yd.data_ptr(), yid.data_ptr() if yid is not None else 0, mode, alpha))
            refs.append((yd, ref))
    cols = list(zip(*items))
    arrs = [ptr_array(cols[0]), int_array(cols[1]), int_array(cols[2]), int_array(cols[3]), ptr_array(cols[4]),
            ptr_array(cols[5]), ptr_array(cols[6]), ptr_array(cols[7]), int_array(cols[8]),
            np.asarray(cols[9], dtype=np.float64)]
    rc = lib.rsc_gemv_multi(len(items), *[a.ctypes.data for a in arrs], torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    for yd, ref in refs:
        assert relerr(yd.cpu().numpy(), ref) < 1e-13


@pytest.mark.parametrize("n", [1, 37, 64, 100, 256, 300, 320, 400])
def test_trsm_left_shapes(cuda, n):
    """L X = B and L^T X = B for batches with ragged n and column counts (the
    strip-resident kernel for n <= 320, the blocked GEMM chain above)."""
    import torch

    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(100 + n)
    ms = [1, 31, 32, 33, 200]
    Ls, Dv = [], []
    for _ in ms:
        G = rng.standard_normal((n, n))
        Ad = E.to_dev(G @ G.T / n + np.eye(n))
        D = E.zeros(max(n, 1), 64)
        info = E.zeros(1, dtype=E.I32)
        E.potrf_batched([Ad.data_ptr()], [n], [n], [D.data_ptr()], info)
        Ls.append(Ad)
        Dv.append(D)
    for trans in (0, 1):
        Bs = [rng.standard_normal((n, m + 3)) for m in ms]   # ld > cols
        Bd = [E.to_dev(B) for B in Bs]
        E.trsm_batched("left", trans, [L.data_ptr() for L in Ls], [n] * len(ms), [n] * len(ms),
                       [d.data_ptr() for d in Dv], [b.data_ptr() for b in Bd], ms, [m + 3 for m in ms])
        torch.cuda.synchronize()
        for L, B, b, m in zip(Ls, Bs, Bd, ms):
            Lh = np.tril(L.cpu().numpy())
            ref = np.linalg.solve(Lh.T if trans else Lh, B[:, :m])
            got = b.cpu().numpy()
            assert relerr(got[:, :m], ref) < 1e-11
            assert np.array_equal(got[:, m:], B[:, m:])  # columns past m untouched


def test_potrf_fused_batch_mixed_sizes_lda_and_failures(cuda):
    """One batched call over orders 1..256 (the fused one-CTA path), odd and padded
    leading dimensions, failing pivots in several 64-blocks: L vs numpy (lower, upper
    zeroed), the stored inverse diagonal blocks, and LAPACK-style 1-based info."""
    import torch
    from paper_1507_05593_b200 import engine as E

    rng = np.random.default_rng(7)
    sizes = [1, 2, 7, 31, 63, 64, 65, 96, 127, 128, 129, 191, 200, 255, 256, 256, 100, 130]
    fail_at = {2: 0, 12: 5, 13: 70, 14: 255, 16: 64}  # batch index -> 0-based pivot
    mats, lds, ptrs, dinv = [], [], [], []
    for i, n in enumerate(sizes):
        G = rng.standard_normal((n, n))
        S = G @ G.T / max(n, 1) + np.eye(n)
        if i in fail_at:
            p = fail_at[i]
            S[p, p] = -1.0 if p == 0 else S[p, p] - 1e6
        ld = n + (i % 3)  # odd / padded leading dimensions
        buf = np.full((n, ld), np.nan)
        buf[:, :n] = S
        t = E.to_dev(buf)
        mats.append((S, t))
        lds.append(ld)
        ptrs.append(t.data_ptr())
        d = torch.full((max(n, 1), 64), float("nan"), dtype=torch.float64, device="cuda")
        dinv.append(d)
    info = torch.zeros(len(sizes), dtype=torch.int32, device="cuda")
    E.potrf_batched(ptrs, sizes, lds, [d.data_ptr() for d in dinv], info)
    torch.cuda.synchronize()
    info = info.cpu().numpy()
    for i, (n, (S, t)) in enumerate(zip(sizes, mats)):
        if i in fail_at:
            assert info[i] == fail_at[i] + 1, (i, n, info[i])
            continue
        assert info[i] == 0, (i, n, info[i])
        L = t.cpu().numpy()[:, :n]
        Lref = np.linalg.cholesky(S)
        assert relerr(L, Lref) < 1e-13, (i, n, relerr(L, Lref))
        D = dinv[i].cpu().numpy()
        for j0 in range(0, n, 64):
            nb = min(64, n - j0)
            blk = D[j0:j0 + nb, :]
            inv = np.linalg.inv(Lref[j0:j0 + nb, j0:j0 + nb])
            assert relerr(blk[:, :nb], inv) < 1e-12, (i, n, j0)
            assert np.all(blk[:, nb:] == 0.0) and np.all(np.triu(blk[:, :nb], 1) == 0.0)


def test_copy2d_batched_copy_and_transpose(cuda):
    """rsc_copy2d_batched: strided rectangular copies and transposes, mixed shapes in
    one launch (row tiles dealt over gridDim.y), more matrices than one parameter block."""
    import torch

    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200._lib import int_array, ptr_array

    lib = _lib.load()
    rng = np.random.default_rng(21)
    shapes = [(1, 1), (31, 33), (64, 64), (700, 45), (45, 700), (3000, 17), (2, 513)] + [(5, 7)] * 800
    for trans in (0, 1):
        src = [torch.from_numpy(rng.standard_normal((r, c + 2))).cuda() for r, c in shapes]
        dst = [torch.full((c if trans else r, (r if trans else c) + 3), -7.0, dtype=torch.float64, device="cuda")
               for r, c in shapes]
        arrs = [ptr_array([s.data_ptr() for s in src]), ptr_array([d.data_ptr() for d in dst]),
                int_array([r for r, _ in shapes]), int_array([c for _, c in shapes]),
                int_array([c + 2 for _, c in shapes]), int_array([d.shape[1] for d in dst])]
        rc = lib.rsc_copy2d_batched(len(shapes), *[a.ctypes.data for a in arrs], trans,
                                    torch.cuda.current_stream().cuda_stream)
        assert rc == 0
        torch.cuda.synchronize()
        for (r, c), s, d in zip(shapes[:8], src, dst):
            want = s[:, :c].T if trans else s[:, :c]
            got = d[:, :want.shape[1]]
            assert torch.equal(got, want)
            assert bool((d[:, want.shape[1]:] == -7.0).all())  # nothing written past the block
