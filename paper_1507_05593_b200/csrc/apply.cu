// HBM-streaming kernels of the preconditioner application (factor.py:175-218):
// batched triangular solves with a single right-hand side and batched
// gather/scatter matrix-vector products.  Every matrix element is read exactly
// once per sweep, along its contiguous (row-major) dimension.
//
//  trsv_batched : one CTA per dense lower triangle.  Blocked by the 64x64 diagonal
//                 blocks whose inverses the factorization stored: forward
//                 x_j = Dinv_j (b_j - L_{j,<j} x_{<j}), backward
//                 x_j = Dinv_j^T (b_j - L_{>j,j}^T x_{>j}); x stays in shared memory.
//  gemv_batched : y[yidx[r]] += alpha * M[r,:] . x[xidx]     (trans = 0, warp per row)
//                 y[c]       += alpha * sum_r M[r,c] x[xidx[r]]  (trans = 1, thread per column)
//                 FP64 atomics on the output (units of one level share target rows).
#include "common.cuh"

namespace {

constexpr int NB = 64;
constexpr int T = 256;
constexpr int MAXP = 240;

struct TrsvArgs {
    int count;
    const double *L[MAXP];
    const double *Dinv[MAXP];
    double *x[MAXP];
    int n[MAXP], ldl[MAXP];
};

__global__ void __launch_bounds__(T) trsv_kernel(const __grid_constant__ TrsvArgs a, int trans) {
    extern __shared__ double xs[];  // n + 64 doubles
    __shared__ double part[8][NB];
    const int b = blockIdx.x;
    const int n = a.n[b], ld = a.ldl[b];
    const double *L = a.L[b];
    const double *Di = a.Dinv[b];
    double *x = a.x[b];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    double *tb = xs + n;  // 64-entry block right-hand side
    for (int i = t; i < n; i += T) xs[i] = x[i];
    __syncthreads();
    const int nbk = (n + NB - 1) / NB;
    for (int it = 0; it < nbk; ++it) {
        const int jb = trans ? nbk - 1 - it : it;
        const int j0 = jb * NB, nbj = min(NB, n - j0);
        if (!trans) {
            // t = b_j - L[j0:j0+nbj, 0:j0] x[0:j0]  (warp per row, lanes along the row)
            for (int r = w; r < nbj; r += 8) {
                const double *Lr = L + (long long)(j0 + r) * ld;
                double s = 0.0;
                for (int c = lane; c < j0; c += 32) s += Lr[c] * xs[c];
                s = warp_sum(s);
                if (lane == 0) tb[r] = xs[j0 + r] - s;
            }
        } else {
            // t = b_j - L[j0+nbj:n, j0:j0+nbj]^T x[j0+nbj:n]  (warp w sums rows w, w+8, ..)
            const int c0 = lane, c1 = lane + 32;
            double s0 = 0.0, s1 = 0.0;
            for (int r = j0 + nbj + w; r < n; r += 8) {
                const double *Lr = L + (long long)r * ld + j0;
                const double xr = xs[r];
                if (c0 < nbj) s0 += Lr[c0] * xr;
                if (c1 < nbj) s1 += Lr[c1] * xr;
            }
            part[w][c0] = s0;
            part[w][c1] = s1;
            __syncthreads();
            if (t < nbj) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < 8; ++q) s += part[q][t];
                tb[t] = xs[j0 + t] - s;
            }
        }
        __syncthreads();
        // x_j = Dinv_j t   or   Dinv_j^T t
        const double *D = Di + (long long)j0 * NB;
        if (!trans) {
            for (int r = w; r < nbj; r += 8) {
                double s = 0.0;
                for (int c = lane; c <= r; c += 32) s += D[r * NB + c] * tb[c];
                s = warp_sum(s);
                if (lane == 0) xs[j0 + r] = s;
            }
        } else {
            for (int c = w; c < nbj; c += 8) {
                double s = 0.0;
                for (int r = c + lane; r < nbj; r += 32) s += D[r * NB + c] * tb[r];
                s = warp_sum(s);
                if (lane == 0) xs[j0 + c] = s;
            }
        }
        __syncthreads();
    }
    for (int i = t; i < n; i += T) x[i] = xs[i];
}

struct GemvArgs {
    int count;
    long long blk_begin[MAXP + 1];
    const double *M[MAXP];
    const double *x[MAXP];
    double *y[MAXP];
    const int *xidx[MAXP];
    const int *yidx[MAXP];
    int rows[MAXP], cols[MAXP], ldm[MAXP];
    double alpha;
};

constexpr int ROWS_T0 = 16;  // transpose 0: 8 warps x 2 rows per CTA
constexpr int ROWS_T1 = 64;  // transpose 1: 64-row slab, thread per column

__device__ __forceinline__ double ldnc(const double *p) { return __ldg(p); }

// mode bit 0: transpose; bit 1: M is lower triangular (read c <= r only);
// bit 2: assign instead of atomic accumulate (transpose 0 only: one warp owns a row);
// bit 3: M is upper triangular (transpose 0 only: read c >= r only).
// Inner loops are unrolled 4x so each lane keeps four independent 8-byte loads in
// flight (the kernel is latency-bound otherwise).
__global__ void __launch_bounds__(T) gemv_kernel(const __grid_constant__ GemvArgs a, int mode) {
    const bool trans = mode & 1, lower = mode & 2, assign = mode & 4, upper = mode & 8;
    __shared__ double xr[ROWS_T1];
    int lo = 0, hi = a.count - 1;
    const long long blk = blockIdx.x;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.blk_begin[mid] <= blk) lo = mid; else hi = mid - 1;
    }
    const int p = lo;
    const int rows = a.rows[p], cols = a.cols[p], ld = a.ldm[p];
    const double *M = a.M[p];
    const double *x = a.x[p];
    double *y = a.y[p];
    const int *xi = a.xidx[p];
    const int *yi = a.yidx[p];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    if (!trans) {
        const int r0 = (int)(blk - a.blk_begin[p]) * ROWS_T0;
        const int r1 = min(rows, r0 + ROWS_T0);
        for (int r = r0 + w; r < r1; r += 8) {
            const double *Mr = M + (long long)r * ld;
            const int cend = lower ? min(cols, r + 1) : cols;
            int c = (upper ? r : 0) + lane;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            if (xi) {
                for (; c + 96 < cend; c += 128) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + 32), m2 = ldnc(Mr + c + 64),
                                 m3 = ldnc(Mr + c + 96);
                    s0 += m0 * x[xi[c]];
                    s1 += m1 * x[xi[c + 32]];
                    s2 += m2 * x[xi[c + 64]];
                    s3 += m3 * x[xi[c + 96]];
                }
                for (; c < cend; c += 32) s0 += ldnc(Mr + c) * x[xi[c]];
            } else {
                for (; c + 96 < cend; c += 128) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + 32), m2 = ldnc(Mr + c + 64),
                                 m3 = ldnc(Mr + c + 96);
                    s0 += m0 * x[c];
                    s1 += m1 * x[c + 32];
                    s2 += m2 * x[c + 64];
                    s3 += m3 * x[c + 96];
                }
                for (; c < cend; c += 32) s0 += ldnc(Mr + c) * x[c];
            }
            const double s = warp_sum((s0 + s1) + (s2 + s3));
            if (lane == 0) {
                double *dst = y + (yi ? yi[r] : r);
                if (assign) *dst = a.alpha * s;
                else atomicAdd(dst, a.alpha * s);
            }
        }
    } else {
        const int r0 = (int)(blk - a.blk_begin[p]) * ROWS_T1;
        const int r1 = min(rows, r0 + ROWS_T1);
        for (int r = r0 + t; r < r1; r += T) xr[r - r0] = xi ? x[xi[r]] : x[r];
        __syncthreads();
        for (int c = t; c < cols; c += T) {
            int r = lower ? max(r0, c) : r0;
            if (r >= r1) continue;
            const double *Mc = M + (long long)r * ld + c;
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            for (; r + 3 < r1; r += 4, Mc += 4LL * ld) {
                const double m0 = ldnc(Mc), m1 = ldnc(Mc + ld), m2 = ldnc(Mc + 2LL * ld), m3 = ldnc(Mc + 3LL * ld);
                s0 += m0 * xr[r - r0];
                s1 += m1 * xr[r + 1 - r0];
                s2 += m2 * xr[r + 2 - r0];
                s3 += m3 * xr[r + 3 - r0];
            }
            for (; r < r1; ++r, Mc += ld) s0 += ldnc(Mc) * xr[r - r0];
            atomicAdd(y + (yi ? yi[c] : c), a.alpha * ((s0 + s1) + (s2 + s3)));
        }
    }
}

}  // namespace

extern "C" int rsc_trsv_batched(int count, const double *const *L, const int *n, const int *ldl,
                                const double *const *Dinv, double *const *x, int trans, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!L || !n || !ldl || !Dinv || !x) return -2;
    static thread_local TrsvArgs a;
    for (int c0 = 0; c0 < count; c0 += MAXP) {
        const int cnt = count - c0 < MAXP ? count - c0 : MAXP;
        int maxn = 1;
        a.count = cnt;
        for (int i = 0; i < cnt; ++i) {
            a.L[i] = L[c0 + i]; a.Dinv[i] = Dinv[c0 + i]; a.x[i] = x[c0 + i];
            a.n[i] = n[c0 + i]; a.ldl[i] = ldl[c0 + i];
            maxn = n[c0 + i] > maxn ? n[c0 + i] : maxn;
        }
        const size_t smem = (size_t)(maxn + NB) * sizeof(double);
        if (smem > 200 * 1024) return -3;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(trsv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            attr = true;
        }
        trsv_kernel<<<cnt, T, smem, (cudaStream_t)stream>>>(a, trans);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

extern "C" int rsc_gemv_batched(int count, const double *const *M, const int *rows, const int *cols,
                                const int *ldm, const double *const *x, const int *const *xidx,
                                double *const *y, const int *const *yidx, int mode, double alpha,
                                void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!M || !rows || !cols || !ldm || !x || !y) return -2;
    static thread_local GemvArgs a;
    int i = 0;
    while (i < count) {
        a.count = 0;
        a.alpha = alpha;
        long long blocks = 0;
        while (i < count && a.count < MAXP) {
            const int c = a.count;
            if (rows[i] <= 0 || cols[i] <= 0) { ++i; continue; }
            a.M[c] = M[i]; a.x[c] = x[i]; a.y[c] = y[i];
            a.xidx[c] = xidx ? xidx[i] : nullptr;
            a.yidx[c] = yidx ? yidx[i] : nullptr;
            a.rows[c] = rows[i]; a.cols[c] = cols[i]; a.ldm[c] = ldm[i];
            a.blk_begin[c] = blocks;
            const int rpc = (mode & 1) ? ROWS_T1 : ROWS_T0;
            blocks += (rows[i] + rpc - 1) / rpc;
            ++a.count;
            ++i;
        }
        if (a.count == 0) continue;
        a.blk_begin[a.count] = blocks;
        gemv_kernel<<<(unsigned)blocks, T, 0, (cudaStream_t)stream>>>(a, mode);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}
