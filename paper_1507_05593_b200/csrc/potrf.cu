// Batched blocked Cholesky (POTRF) and triangular solves (TRSM) on FP64 DMMA.
//
// Blocked left-looking over 64-column panels.  For panel s (columns j0..j0+nb):
//   1. A[j0:n, j0:j0+nb] -= L[j0:n, 0:j0] @ L[j0:j0+nb, 0:j0]^T      (grouped DMMA GEMM)
//   2. factor the nb x nb diagonal block in shared memory and form its inverse
//      (potrf_diag_kernel, one CTA per matrix)                           -> Dinv_s
//   3. L[j0+nb:n, j0:j0+nb] = A[j0+nb:n, j0:j0+nb] @ Dinv_s^T           (grouped DMMA GEMM)
// The inverse diagonal blocks are kept (n x 64 per factor) so every later
// triangular solve with this factor is a chain of DMMA GEMMs, not a scalar
// substitution.  Pivot failure follows LAPACK dpotrf: info = 1-based column of the
// first pivot that is not > 0 (NaN included); the failing matrix is then skipped.
// Reference: kernels.py:22-39 (dense_cholesky), kernels.py:42-64 (tri_solve).
#include <cstdlib>
#include <vector>
#include "common.cuh"

namespace {

constexpr int NB = 64;
constexpr int MAXB = 600;  // whole level / batch per launch

struct DiagArgs {
    int count;
    int step;
    double *A[MAXB];
    double *Dinv[MAXB];
    int n[MAXB];
    int lda[MAXB];
    int base;  // index of A[0] within the caller's info array
};

// 64x64 diagonal block in shared memory, 256 threads: thread t owns row
// i = t >> 2 and the columns j == (t & 3) mod 4.  L lives in the lower triangle;
// its inverse is kept transposed in the strict upper part plus the pad column:
// inv[i][c] (i >= c) lives at s[c][i + 1].
// Right-looking Cholesky, then column-parallel forward substitution L X = I.
// Returns the 0-based failing pivot or -1.
__device__ int factor_invert_64(double (*s)[NB + 1], int nb, bool factor) {
    // warp w owns rows i == w (mod 8), lanes run along the row (conflict-free rows)
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (factor) {
        for (int k = 0; k < nb; ++k) {
            const double piv = s[k][k];
            if (!(piv > 0.0)) return k;  // uniform: every thread read the same value
            const double d = sqrt(piv), rd = 1.0 / d;  // dpotf2 scales by 1/ajj
            __syncthreads();
            for (int i = k + 1 + t; i < nb; i += blockDim.x) s[i][k] *= rd;
            if (t == 0) s[k][k] = d;
            __syncthreads();
            for (int i = k + 1 + w; i < nb; i += 8) {
                const double lik = s[i][k];
                for (int j = k + 1 + lane; j <= i; j += 32) s[i][j] -= lik * s[j][k];
            }
            __syncthreads();
        }
    }
    // X = L^{-1} (X[i][c] at s[c][i+1]); row k of X is final once rows < k are in
    for (int i = w; i < nb; i += 8)
        for (int c = lane; c <= i; c += 32) s[c][i + 1] = (c == i) ? 1.0 : 0.0;
    __syncthreads();
    for (int k = 0; k < nb; ++k) {
        const double rk = 1.0 / s[k][k];
        for (int c = t; c <= k; c += blockDim.x) s[c][k + 1] *= rk;
        __syncthreads();
        for (int i = k + 1 + w; i < nb; i += 8) {
            const double lik = s[i][k];
            for (int c = lane; c <= k; c += 32) s[c][i + 1] -= lik * s[c][k + 1];
        }
        __syncthreads();
    }
    return -1;
}

// One CTA per matrix: factor the diagonal block of panel `step` and invert it.
__global__ void __launch_bounds__(256) potrf_diag_kernel(const __grid_constant__ DiagArgs args,
                                                          int *info) {
    __shared__ double s[NB][NB + 1];
    const int b = blockIdx.x;
    const int n = args.n[b];
    const int j0 = args.step * NB;
    if (j0 >= n) return;
    if (info[args.base + b] != 0) return;
    const int nb = min(NB, n - j0);
    double *A = args.A[b];
    const int lda = args.lda[b];
    const int t = threadIdx.x;
    for (int e = t; e < NB * NB; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        s[i][j] = (i < nb && j <= i) ? A[(long long)(j0 + i) * lda + j0 + j] : 0.0;
    }
    __syncthreads();
    const int bad = factor_invert_64(s, nb, true);
    if (bad >= 0) {
        if (t == 0) info[args.base + b] = j0 + bad + 1;
        return;
    }
    for (int e = t; e < nb * NB; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        if (j < nb) A[(long long)(j0 + i) * lda + j0 + j] = (j <= i) ? s[i][j] : 0.0;
        args.Dinv[b][(long long)(j0 + i) * NB + j] = (j < nb && j <= i) ? s[j][i + 1] : 0.0;
    }
    // zero the strict upper triangle right of the diagonal block (dpotrf "clean")
    const int rest = n - j0 - nb;
    for (long long e = t; e < (long long)nb * rest; e += blockDim.x) {
        const int i = (int)(e / rest), j = (int)(e % rest);
        A[(long long)(j0 + i) * lda + j0 + nb + j] = 0.0;
    }
}

// Inverse diagonal blocks of an existing lower triangle (no factorization):
// grid = (blocks, matrices).  Used when a triangle arrives from outside
// (tri_solve on a caller-supplied L).
__global__ void __launch_bounds__(256) trtri_diag_kernel(const __grid_constant__ DiagArgs args) {
    __shared__ double s[NB][NB + 1];
    const int b = blockIdx.y;
    const int n = args.n[b];
    const int j0 = blockIdx.x * NB;
    if (j0 >= n) return;
    const int nb = min(NB, n - j0);
    const double *A = args.A[b];
    const int lda = args.lda[b];
    const int t = threadIdx.x;
    for (int e = t; e < NB * NB; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        s[i][j] = (i < nb && j <= i) ? A[(long long)(j0 + i) * lda + j0 + j] : 0.0;
    }
    __syncthreads();
    factor_invert_64(s, nb, false);
    for (int e = t; e < nb * NB; e += blockDim.x) {
        const int i = e >> 6, j = e & 63;
        args.Dinv[b][(long long)(j0 + i) * NB + j] = (j < nb && j <= i) ? s[j][i + 1] : 0.0;
    }
}

inline rsc_gemm_problem make_prob(const double *A, int lda, const double *B, int ldb, double *C,
                                  int ldc, int M, int N, int K, double alpha, double beta) {
    rsc_gemm_problem p{};
    p.A = A; p.B = B; p.C = C;
    p.lda = lda; p.ldb = ldb; p.ldc = ldc;
    p.M = M; p.N = N; p.K = K;
    p.alpha = alpha; p.beta = beta;
    p.batch = 1;
    return p;
}

}  // namespace

int rsc_potrf_fused(int count, double *const *A, const int *n, const int *lda, double *const *Dinv,
                    int *info_dev, cudaStream_t s);

extern "C" int rsc_potrf_batched(int count, double *const *A, const int *n, const int *lda,
                                 double *const *Dinv, int *info_dev, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!A) return -2;
    if (!n) return -3;
    if (!lda) return -4;
    if (!Dinv) return -5;
    if (!info_dev) return -6;
    cudaStream_t s = (cudaStream_t)stream;
    int maxn = 0;
    for (int i = 0; i < count; ++i) {
        if (n[i] < 0 || lda[i] < n[i]) return -3;
        maxn = n[i] > maxn ? n[i] : maxn;
    }
    cudaMemsetAsync(info_dev, 0, sizeof(int) * count, s);
    if (maxn <= 256 && !getenv("RSC_POTRF_UNFUSED")) return rsc_potrf_fused(count, A, n, lda, Dinv, info_dev, s);
    const int steps = (maxn + NB - 1) / NB;
    std::vector<rsc_gemm_problem> probs;
    probs.reserve(count);
    static thread_local DiagArgs da;
    for (int st = 0; st < steps; ++st) {
        const int j0 = st * NB;
        // 1. left-looking panel update
        if (j0 > 0) {
            probs.clear();
            for (int i = 0; i < count; ++i) {
                if (n[i] <= j0) continue;
                const int nb = n[i] - j0 < NB ? n[i] - j0 : NB;
                double *Ai = A[i];
                const long long l = lda[i];
                probs.push_back(make_prob(Ai + j0 * l, lda[i], Ai + j0 * l, lda[i], Ai + j0 * l + j0,
                                          lda[i], n[i] - j0, nb, j0, -1.0, 1.0));
            }
            int rc = rsc_gemm_grouped(0, 1, probs.data(), (int)probs.size(), stream);
            if (rc) return rc;
        }
        // 2. diagonal block factor + inverse
        for (int c0 = 0; c0 < count; c0 += MAXB) {
            const int cnt = count - c0 < MAXB ? count - c0 : MAXB;
            da.count = cnt;
            da.step = st;
            da.base = c0;
            for (int i = 0; i < cnt; ++i) {
                da.A[i] = A[c0 + i];
                da.Dinv[i] = Dinv[c0 + i];
                da.n[i] = n[c0 + i];
                da.lda[i] = lda[c0 + i];
            }
            potrf_diag_kernel<<<cnt, 256, 0, s>>>(da, info_dev);
            RSC_CHECK_LAUNCH();
        }
        // 3. panel below the diagonal block: X = X @ Dinv^T (in place, one column tile)
        probs.clear();
        for (int i = 0; i < count; ++i) {
            if (n[i] <= j0 + NB) continue;
            double *Ai = A[i];
            const long long l = lda[i];
            probs.push_back(make_prob(Ai + (j0 + NB) * l + j0, lda[i], Dinv[i] + (long long)j0 * NB, NB,
                                      Ai + (j0 + NB) * l + j0, lda[i], n[i] - j0 - NB, NB, NB, 1.0, 0.0));
        }
        int rc = rsc_gemm_grouped(0, 1, probs.data(), (int)probs.size(), stream);
        if (rc) return rc;
    }
    return 0;
}

int rsc_trsm_right_fused(int count, const double *const *L, const int *n, const int *ldl,
                         const double *const *Dinv, const double *const *Bsrc, double *const *B,
                         const int *m, const int *ldb, cudaStream_t s);
int rsc_trsm_left_fused(int trans, int count, const double *const *L, const int *n, const int *ldl,
                        const double *const *Dinv, double *const *B, const int *m, const int *ldb,
                        cudaStream_t s);

extern "C" int rsc_trsm_right_batched(int count, const double *const *L, const int *n, const int *ldl,
                                      const double *const *Dinv, const double *const *Bsrc,
                                      double *const *B, const int *m, const int *ldb, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!L || !n || !ldl || !Dinv || !B || !m || !ldb) return -2;
    const int rc = rsc_trsm_right_fused(count, L, n, ldl, Dinv, Bsrc, B, m, ldb, (cudaStream_t)stream);
    return rc == -1000 ? -3 : rc;  // some n > 320: use rsc_trsm_batched
}

extern "C" int rsc_trsm_batched(int side, int trans, int count, const double *const *L,
                                const int *n, const int *ldl, const double *const *Dinv,
                                double *const *B, const int *m, const int *ldb, void *stream) {
    if (side != 0 && side != 1) return -1;
    if (trans != 0 && trans != 1) return -2;
    if (side == 1 && trans == 0) return -2;
    if (count < 0) return -3;
    if (count == 0) return 0;
    if (!L || !n || !ldl || !Dinv || !B || !m || !ldb) return -4;
    if (side == 1) {  // fused strip-resident kernels when every triangle has n <= 320
        const int rc = rsc_trsm_right_fused(count, L, n, ldl, Dinv, nullptr, B, m, ldb, (cudaStream_t)stream);
        if (rc != -1000) return rc;
    } else {
        const int rc = rsc_trsm_left_fused(trans, count, L, n, ldl, Dinv, B, m, ldb, (cudaStream_t)stream);
        if (rc != -1000) return rc;
    }
    int maxn = 0;
    for (int i = 0; i < count; ++i) maxn = n[i] > maxn ? n[i] : maxn;
    const int steps = (maxn + NB - 1) / NB;
    std::vector<rsc_gemm_problem> upd, dia;
    upd.reserve(count);
    dia.reserve(count);
    for (int it = 0; it < steps; ++it) {
        upd.clear();
        dia.clear();
        for (int i = 0; i < count; ++i) {
            const int ni = n[i];
            const int nst = (ni + NB - 1) / NB;
            if (it >= nst || m[i] <= 0) continue;
            // left-trans runs the panels backwards
            const int st = (side == 0 && trans == 1) ? nst - 1 - it : it;
            const int j0 = st * NB;
            const int nb = ni - j0 < NB ? ni - j0 : NB;
            const double *Li = L[i];
            const long long ll = ldl[i], lb = ldb[i];
            double *Bi = B[i];
            const double *Di = Dinv[i] + (long long)j0 * NB;
            if (side == 1) {
                // X L^T = B ; B is m x n.  X_s = (B_s - X_{<s} L_{s,<s}^T) Dinv_s^T
                if (j0 > 0)
                    upd.push_back(make_prob(Bi, ldb[i], Li + j0 * ll, ldl[i], Bi + j0, ldb[i], m[i], nb, j0,
                                            -1.0, 1.0));
                dia.push_back(make_prob(Bi + j0, ldb[i], Di, NB, Bi + j0, ldb[i], m[i], nb, nb, 1.0, 0.0));
            } else if (trans == 0) {
                // L X = B ; B is n x m.  X_s = Dinv_s (B_s - L_{s,<s} X_{<s})
                if (j0 > 0)
                    upd.push_back(make_prob(Li + j0 * ll, ldl[i], Bi, ldb[i], Bi + j0 * lb, ldb[i], nb, m[i], j0,
                                            -1.0, 1.0));
                dia.push_back(make_prob(Di, NB, Bi + j0 * lb, ldb[i], Bi + j0 * lb, ldb[i], nb, m[i], nb, 1.0,
                                        0.0));
            } else {
                // L^T X = B.  X_s = Dinv_s^T (B_s - L_{>s,s}^T X_{>s})
                const int rest = ni - j0 - nb;
                if (rest > 0)
                    upd.push_back(make_prob(Li + (j0 + nb) * ll + j0, ldl[i], Bi + (j0 + nb) * lb, ldb[i],
                                            Bi + j0 * lb, ldb[i], nb, m[i], rest, -1.0, 1.0));
                dia.push_back(make_prob(Di, NB, Bi + j0 * lb, ldb[i], Bi + j0 * lb, ldb[i], nb, m[i], nb, 1.0,
                                        0.0));
            }
        }
        int rc;
        if (!upd.empty()) {
            if (side == 1) rc = rsc_gemm_grouped(0, 1, upd.data(), (int)upd.size(), stream);
            else if (trans == 0) rc = rsc_gemm_grouped(0, 0, upd.data(), (int)upd.size(), stream);
            else rc = rsc_gemm_grouped(1, 0, upd.data(), (int)upd.size(), stream);
            if (rc) return rc;
        }
        if (!dia.empty()) {
            if (side == 1) rc = rsc_gemm_grouped(0, 1, dia.data(), (int)dia.size(), stream);
            else if (trans == 0) rc = rsc_gemm_grouped(0, 0, dia.data(), (int)dia.size(), stream);
            else rc = rsc_gemm_grouped(1, 0, dia.data(), (int)dia.size(), stream);
            if (rc) return rc;
        }
    }
    return 0;
}

extern "C" int rsc_trtri_diag_batched(int count, const double *const *L, const int *n, const int *ldl,
                                      double *const *Dinv, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!L || !n || !ldl || !Dinv) return -2;
    static thread_local DiagArgs da;
    for (int c0 = 0; c0 < count; c0 += MAXB) {
        const int cnt = count - c0 < MAXB ? count - c0 : MAXB;
        int maxn = 1;
        da.count = cnt;
        da.step = 0;
        da.base = c0;
        for (int i = 0; i < cnt; ++i) {
            da.A[i] = const_cast<double *>(L[c0 + i]);
            da.Dinv[i] = Dinv[c0 + i];
            da.n[i] = n[c0 + i];
            da.lda[i] = ldl[c0 + i];
            maxn = n[c0 + i] > maxn ? n[c0 + i] : maxn;
        }
        dim3 grid((maxn + NB - 1) / NB, cnt);
        trtri_diag_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(da);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}
