// Plan-level C-ABI entries (SURVEY §8(b) "what a C-ABI replacement must export"):
// the numeric steps of the reference's sweep as calls a non-Python caller can drive
// from the plan's index arrays, composed from the batched kernels of this library.
//
//   rsc_schur_update        Schur assembly of one supernode (factor.py:383-398)
//   rsc_offdiag_products    the source terms of Alg. 2 / its mirror (factor.py:427-483)
//   rsc_interior_factor_batched   L_B and Y_B of interior blocks (interior.py:105-156)
//   rsc_tree_trsm           Alg. 4 on one diagonal block tree (diagblocks.py:192-273)
//   rsc_apply_sweep         one sweep (forward or backward) of the apply (factor.py:175-218)
//   rsc_nccl_*              communicator / all-reduce / broadcast for the multi-GPU path
//
// Every entry is stream-ordered and re-entrant; device pointers, int dimensions,
// 0 = ok, < 0 bad argument, > 0 error code of the underlying call.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

rsc_gemm_problem problem(const double *A, int lda, const double *B, int ldb, double *C, int ldc, int M, int N, int K,
                         double alpha, double beta) {
    rsc_gemm_problem p;
    std::memset(&p, 0, sizeof(p));
    p.A = A; p.B = B; p.C = C;
    p.lda = lda > 0 ? lda : 1; p.ldb = ldb > 0 ? ldb : 1; p.ldc = ldc > 0 ? ldc : 1;
    p.M = M; p.N = N; p.K = K;
    p.batch = 1;
    p.alpha = alpha; p.beta = beta;
    return p;
}

}  // namespace

extern "C" {

int rsc_schur_update(double *UD, int ld_ud, int nc, double *UO, int ld_uo, int nr, int nsrc,
                     const double *const *eff, const double *const *raw, const int *ld, const int *w, const int *lo,
                     const int *nrd, const int *nro, const int *const *cpos, const int *const *rpos, void *stream) {
    if (nsrc < 0 || nc < 0 || nr < 0) return -1;
    if (nsrc == 0) return 0;
    if (!eff || !raw || !ld || !w || !lo || !nrd || !nro || !cpos || !rpos) return -2;
    std::vector<rsc_gemm_problem> ps;
    ps.reserve(2 * (size_t)nsrc);
    // UD first, then UO: each target keeps its sources in the caller's (reference) order
    for (int q = 0; q < nsrc && UD; ++q) {
        if (w[q] <= 0 || nrd[q] <= 0) continue;
        const double *A = eff[q] + (long long)lo[q] * ld[q], *B = raw[q] + (long long)lo[q] * ld[q];
        rsc_gemm_problem p = problem(A, ld[q], B, ld[q], UD, ld_ud, nrd[q], nrd[q], w[q], -1.0, 1.0);
        p.c_rows = cpos[q]; p.c_cols = cpos[q]; p.atomic = 1; p.ext_r = nc; p.ext_c = nc;
        ps.push_back(p);
    }
    for (int q = 0; q < nsrc && UO; ++q) {
        if (w[q] <= 0 || nrd[q] <= 0 || nro[q] <= 0) continue;
        const double *A = eff[q] + (long long)(lo[q] + nrd[q]) * ld[q], *B = raw[q] + (long long)lo[q] * ld[q];
        rsc_gemm_problem p = problem(A, ld[q], B, ld[q], UO, ld_uo, nro[q], nrd[q], w[q], -1.0, 1.0);
        p.c_rows = rpos[q]; p.c_cols = cpos[q]; p.atomic = 1; p.ext_r = nr; p.ext_c = nc;
        ps.push_back(p);
    }
    if (ps.empty()) return 0;
    return rsc_gemm_grouped(0, 1, ps.data(), (int)ps.size(), stream);
}

int rsc_offdiag_products(int trans, double *W, int ldw, int wr, int wc, const double *G, int ldg, int r, int nsrc,
                         const double *const *eff, const double *const *raw, const int *ld, const int *w,
                         const int *lo, const int *nrd, const int *nro, const int *const *cpos,
                         const int *const *rpos, double *T, void *stream) {
    if (nsrc < 0 || r < 0) return -1;
    if (nsrc == 0 || r == 0) return 0;
    if (!W || !G || !T || !eff || !raw || !ld || !w || !lo || !nrd || !nro || !cpos || !rpos) return -2;
    std::vector<rsc_gemm_problem> p1, p2;
    long long toff = 0, tot = 0;
    for (int q = 0; q < nsrc; ++q)
        if (w[q] > 0 && nrd[q] > 0 && nro[q] > 0) tot += (long long)w[q] * r;
    cudaError_t e = cudaMemsetAsync(T, 0, (size_t)tot * 8, (cudaStream_t)stream);
    if (e != cudaSuccess) return (int)e;
    for (int q = 0; q < nsrc; ++q) {
        if (w[q] <= 0 || nrd[q] <= 0 || nro[q] <= 0) continue;
        const double *raw_lo = raw[q] + (long long)lo[q] * ld[q];
        const double *eff_hi = eff[q] + (long long)(lo[q] + nrd[q]) * ld[q];
        double *tq = T + toff;
        toff += (long long)w[q] * r;
        // trans = 0: T = V[lo:hi]^T G[cpos] ; W[rpos] -= E[hi:] T   (off_diagonal_multiply)
        // trans = 1: T = E[hi:]^T G[rpos]   ; W[cpos] -= V[lo:hi] T  (..._trans)
        rsc_gemm_problem a = problem(trans ? eff_hi : raw_lo, ld[q], G, ldg, tq, r, w[q], r,
                                     trans ? nro[q] : nrd[q], 1.0, 0.0);
        a.b_rows = trans ? rpos[q] : cpos[q];
        a.atomic = 1;  // T is zeroed: the product accumulates (its K may be split)
        rsc_gemm_problem b = problem(trans ? raw_lo : eff_hi, ld[q], tq, r, W, ldw, trans ? nrd[q] : nro[q], r, w[q],
                                     -1.0, 1.0);
        b.c_rows = trans ? cpos[q] : rpos[q];
        b.atomic = 1; b.ext_r = wr; b.ext_c = wc;
        p1.push_back(a);
        p2.push_back(b);
    }
    if (p1.empty()) return 0;
    int rc = rsc_gemm_grouped(1, 0, p1.data(), (int)p1.size(), stream);
    if (rc) return rc;
    return rsc_gemm_grouped(0, 0, p2.data(), (int)p2.size(), stream);
}

int rsc_interior_factor_batched(int count, double *const *L, const int *n, const int *ldl, double *const *Dinv,
                                double *const *Y, const int *m, const int *ldy, int *info_dev, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    int rc = rsc_potrf_batched(count, L, n, ldl, Dinv, info_dev, stream);
    if (rc) return rc;
    if (!Y) return 0;
    // Y_B = A(off_rows, C_B) L_B^{-T}: right solve, in place
    std::vector<const double *> Lc(L, L + count), Dc(Dinv, Dinv + count);
    std::vector<double *> Yv(Y, Y + count);
    return rsc_trsm_batched(1, 1, count, Lc.data(), n, ldl, Dc.data(), Yv.data(), m, ldy, stream);
}

// ---------------------------------------------------------------------------
// Alg. 4 on one block tree (in-order numbered blocks; internal block s couples its
// left subtree's columns [lo, split) to its right subtree's rows [split, hi)).

namespace {

struct Tree {
    const int *lo, *hi, *split, *left, *right;
    const double *const *L;
    const int *ldl;
    const double *const *Dinv;
    const double *const *B;   // dense coupling (split - lo columns x hi - split rows... row-major: rows x cols)
    const int *ldb;
    const double *const *V;   // low rank: B = V U^T (V: rows x k, U: cols x k)
    const double *const *U;
    const int *ldv, *ldu, *k;
    double *X;
    int ldx, r;
    double *tws;
    cudaStream_t s;
};

int tree_rec(const Tree &t, int nd, int trans) {
    const int lo = t.lo[nd], hi = t.hi[nd], sp = t.split[nd];
    if (sp < 0) {  // leaf: X[lo:hi] <- L^{-1} X or L^{-T} X
        const int n = hi - lo;
        double *Xp = t.X + (long long)lo * t.ldx;
        const double *Lp = t.L[nd], *Dp = t.Dinv[nd];
        return rsc_trsm_batched(0, trans, 1, &Lp, &n, &t.ldl[nd], &Dp, &Xp, &t.r, &t.ldx, t.s);
    }
    const int nl = sp - lo, nr = hi - sp;
    double *X1 = t.X + (long long)lo * t.ldx, *X2 = t.X + (long long)sp * t.ldx;
    auto couple = [&](bool tr) -> int {
        // forward: X2 -= B X1 ;  transposed: X1 -= B^T X2   (B: nr x nl)
        if (t.k && t.V[nd]) {
            const int k = t.k[nd];
            if (k == 0) return 0;
            rsc_gemm_problem a, b;
            if (!tr) {  // tws = U^T X1 (k x r); X2 -= V tws
                a = problem(t.U[nd], t.ldu[nd], X1, t.ldx, t.tws, t.r, k, t.r, nl, 1.0, 0.0);
                b = problem(t.V[nd], t.ldv[nd], t.tws, t.r, X2, t.ldx, nr, t.r, k, -1.0, 1.0);
            } else {    // tws = V^T X2 ; X1 -= U tws
                a = problem(t.V[nd], t.ldv[nd], X2, t.ldx, t.tws, t.r, k, t.r, nr, 1.0, 0.0);
                b = problem(t.U[nd], t.ldu[nd], t.tws, t.r, X1, t.ldx, nl, t.r, k, -1.0, 1.0);
            }
            int rc = rsc_gemm_grouped(1, 0, &a, 1, t.s);
            if (rc) return rc;
            return rsc_gemm_grouped(0, 0, &b, 1, t.s);
        }
        rsc_gemm_problem p = !tr ? problem(t.B[nd], t.ldb[nd], X1, t.ldx, X2, t.ldx, nr, t.r, nl, -1.0, 1.0)
                                 : problem(t.B[nd], t.ldb[nd], X2, t.ldx, X1, t.ldx, nl, t.r, nr, -1.0, 1.0);
        return rsc_gemm_grouped(tr ? 1 : 0, 0, &p, 1, t.s);
    };
    int rc;
    if (!trans) {
        if ((rc = tree_rec(t, t.left[nd], 0))) return rc;
        if ((rc = couple(false))) return rc;
        return tree_rec(t, t.right[nd], 0);
    }
    if ((rc = tree_rec(t, t.right[nd], 1))) return rc;
    if ((rc = couple(true))) return rc;
    return tree_rec(t, t.left[nd], 1);
}

}  // namespace

int rsc_tree_trsm(int trans, int nnodes, int root, const int *lo, const int *hi, const int *split, const int *left,
                  const int *right, const double *const *L, const int *ldl, const double *const *Dinv,
                  const double *const *B, const int *ldb, const double *const *V, const double *const *U,
                  const int *ldv, const int *ldu, const int *k, double *X, int ldx, int r, double *tws,
                  void *stream) {
    if (nnodes <= 0 || root < 0 || root >= nnodes || r < 0) return -1;
    if (r == 0) return 0;
    if (!lo || !hi || !split || !left || !right || !L || !ldl || !Dinv || !X) return -2;
    Tree t{lo, hi, split, left, right, L, ldl, Dinv, B, ldb, V, U, ldv, ldu, k, X, ldx, r, tws, (cudaStream_t)stream};
    if (k && !tws) return -2;
    return tree_rec(t, root, trans ? 1 : 0);
}

int rsc_apply_sweep(int nphases, const int *phase_count, const double *const *M, const int *rows, const int *cols,
                    const int *ldm, const double *const *x, const int *const *xidx, double *const *y,
                    const int *const *yidx, const int *modes, const double *alphas, void *stream) {
    if (nphases < 0) return -1;
    long long o = 0;
    for (int ph = 0; ph < nphases; ++ph) {
        const int c = phase_count[ph];
        if (c < 0) return -1;
        if (c) {
            const int rc = rsc_gemv_multi(c, M + o, rows + o, cols + o, ldm + o, x + o, xidx + o, y + o, yidx + o,
                                          modes + o, alphas + o, stream);
            if (rc) return rc;
        }
        o += c;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// NCCL (resolved at run time from libnccl.so.2, or RSC_NCCL_LIB)

namespace {

struct NcclId { char internal[128]; };  // ncclUniqueId, passed by value
typedef int (*nccl_get_id_t)(void *);
typedef int (*nccl_init_t)(void **, int, NcclId, int);
typedef int (*nccl_allreduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_bcast_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*nccl_destroy_t)(void *);

struct Nccl {
    void *h = nullptr;
    nccl_get_id_t get_id = nullptr;
    nccl_init_t init = nullptr;
    nccl_allreduce_t allreduce = nullptr;
    nccl_bcast_t bcast = nullptr;
    nccl_destroy_t destroy = nullptr;
};

Nccl *nccl() {
    static Nccl n;
    static bool tried = false;
    if (!tried) {
        tried = true;
        const char *p = getenv("RSC_NCCL_LIB");
        n.h = dlopen(p ? p : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (n.h) {
            n.get_id = (nccl_get_id_t)dlsym(n.h, "ncclGetUniqueId");
            n.init = (nccl_init_t)dlsym(n.h, "ncclCommInitRank");
            n.allreduce = (nccl_allreduce_t)dlsym(n.h, "ncclAllReduce");
            n.bcast = (nccl_bcast_t)dlsym(n.h, "ncclBroadcast");
            n.destroy = (nccl_destroy_t)dlsym(n.h, "ncclCommDestroy");
        }
    }
    return (n.get_id && n.init && n.allreduce && n.bcast && n.destroy) ? &n : nullptr;
}

constexpr int NCCL_FLOAT64 = 8, NCCL_SUM = 0;

}  // namespace

int rsc_nccl_available() { return nccl() != nullptr; }

int rsc_nccl_unique_id(char *id128) {
    Nccl *n = nccl();
    if (!n) return -20;
    return n->get_id(id128);
}

int rsc_nccl_comm_init(int nranks, const char *id128, int rank, void **comm) {
    Nccl *n = nccl();
    if (!n) return -20;
    if (!id128 || !comm || nranks < 1 || rank < 0 || rank >= nranks) return -1;
    NcclId id;
    std::memcpy(id.internal, id128, 128);
    return n->init(comm, nranks, id, rank);
}

int rsc_nccl_allreduce_sum_f64(void *comm, const double *send, double *recv, long long count, void *stream) {
    Nccl *n = nccl();
    if (!n) return -20;
    if (!comm || count < 0) return -1;
    return n->allreduce(send, recv, (size_t)count, NCCL_FLOAT64, NCCL_SUM, comm, (cudaStream_t)stream);
}

int rsc_nccl_broadcast_f64(void *comm, const double *send, double *recv, long long count, int root, void *stream) {
    Nccl *n = nccl();
    if (!n) return -20;
    if (!comm || count < 0) return -1;
    return n->bcast(send, recv, (size_t)count, NCCL_FLOAT64, root, comm, (cudaStream_t)stream);
}

int rsc_nccl_comm_destroy(void *comm) {
    Nccl *n = nccl();
    if (!n) return -20;
    return comm ? n->destroy(comm) : -1;
}

}  // extern "C"
