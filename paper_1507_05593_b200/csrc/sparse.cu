// HBM-bound kernels: CSR block scatter, SpMM / SpMV, row gather / scatter-add and
// the PCG vector updates.  Grids are sized in multiples of the SM count and every
// kernel streams its operands once (coalesced along the dense row).
#include <atomic>
#include <vector>
#include "common.cuh"

namespace {

constexpr int MAXB = 256;

struct CsrDenseArgs {
    int count;
    const int *rowptr[MAXB];
    const int *colidx[MAXB];
    const double *values[MAXB];
    double *D[MAXB];
    int nrows[MAXB];
    int ldd[MAXB];
};

__global__ void csr_to_dense_kernel(const __grid_constant__ CsrDenseArgs a) {
    const int b = blockIdx.y;
    const int nr = a.nrows[b];
    const int *rp = a.rowptr[b];
    const int *ci = a.colidx[b];
    const double *v = a.values[b];
    double *D = a.D[b];
    const long long ld = a.ldd[b];
    for (int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); r < nr;
         r += gridDim.x * (blockDim.x / 32)) {
        for (int p = rp[r] + (threadIdx.x & 31); p < rp[r + 1]; p += 32) D[r * ld + ci[p]] = v[p];
    }
}

struct SpmmArgs {
    int count;
    const int *rowptr[MAXB];
    const int *colidx[MAXB];
    const double *values[MAXB];
    const double *X[MAXB];
    double *Y[MAXB];
    int nrows[MAXB], r[MAXB], ldx[MAXB], ldy[MAXB];
    double alpha, beta;
};

// grouped SpMM: blockIdx.y = problem, warps stride over its rows
__global__ void spmm_csr_batched_kernel(const __grid_constant__ SpmmArgs a) {
    const int b = blockIdx.y;
    const int nr = a.nrows[b], r = a.r[b];
    const int *rp = a.rowptr[b];
    const int *ci = a.colidx[b];
    const double *v = a.values[b];
    const double *X = a.X[b];
    double *Y = a.Y[b];
    const int ldx = a.ldx[b], ldy = a.ldy[b];
    const int wpb = blockDim.x / 32;
    for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < nr; row += gridDim.x * wpb) {
        const int p0 = rp[row], p1 = rp[row + 1];
        for (int c = threadIdx.x & 31; c < r; c += 32) {
            double acc = 0.0;
            for (int p = p0; p < p1; ++p) acc += v[p] * X[(long long)ci[p] * ldx + c];
            double *y = Y + (long long)row * ldy + c;
            *y = (a.beta == 0.0) ? a.alpha * acc : a.alpha * acc + a.beta * (*y);
        }
    }
}

// one warp per output row; lanes stride over the dense columns
__global__ void spmm_csr_kernel(int nrows, int r, const int *__restrict__ rp,
                                const int *__restrict__ ci, const double *__restrict__ v,
                                const double *__restrict__ X, int ldx, double alpha, double beta,
                                double *__restrict__ Y, int ldy) {
    const int wpb = blockDim.x / 32;
    for (int row = blockIdx.x * wpb + (threadIdx.x >> 5); row < nrows; row += gridDim.x * wpb) {
        const int p0 = rp[row], p1 = rp[row + 1];
        for (int c = threadIdx.x & 31; c < r; c += 32) {
            double acc = 0.0;
            for (int p = p0; p < p1; ++p) acc += v[p] * X[(long long)ci[p] * ldx + c];
            double *y = Y + (long long)row * ldy + c;
            *y = (beta == 0.0) ? alpha * acc : alpha * acc + beta * (*y);
        }
    }
}

// vector CSR SpMV: 8 lanes per row (stencil rows hold 7..81 entries)
__global__ void spmv_csr_kernel(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                                const double *__restrict__ v, const double *__restrict__ x,
                                double *__restrict__ y) {
    const int sub = threadIdx.x & 7;
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    // warp-uniform loop: each warp owns 4 consecutive rows per trip
    for (long long base = warp * 4; base < n; base += nwarps * 4) {
        const long long row = base + ((threadIdx.x & 31) >> 3);
        double acc = 0.0;
        if (row < n) {
            const int p0 = rp[row], p1 = rp[row + 1];
            for (int p = p0 + sub; p < p1; p += 8) acc += v[p] * x[ci[p]];
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, 8);
        if (sub == 0 && row < n) y[row] = acc;
    }
}

__global__ void gather_rows_kernel(int nrows, int ncols, const int *__restrict__ idx,
                                   const double *__restrict__ src, int lds, double *__restrict__ dst,
                                   int ldd) {
    const long long tot = (long long)nrows * ncols;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / ncols), j = (int)(e % ncols);
        dst[(long long)i * ldd + j] = src[(long long)idx[i] * lds + j];
    }
}

__global__ void scatter_add_rows_kernel(int nrows, int ncols, const int *__restrict__ idx,
                                        double alpha, const double *__restrict__ src, int lds,
                                        double *__restrict__ dst, int ldd) {
    const long long tot = (long long)nrows * ncols;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < tot;
         e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / ncols), j = (int)(e % ncols);
        dst[(long long)idx[i] * ldd + j] += alpha * src[(long long)i * lds + j];
    }
}

constexpr int DOT_BLOCKS = 296;  // 2 x 148 SMs
constexpr int DOT_THREADS = 512;

__global__ void dot_partial_kernel(int n, const double *__restrict__ x, const double *__restrict__ y,
                                   double *__restrict__ part) {
    __shared__ double red[32];
    double s = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        s += x[i] * y[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void dot_final_kernel(int nparts, const double *__restrict__ part, double *__restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) s += part[i];
    s = block_sum(s, red);
    if (threadIdx.x == 0) out[0] = s;
}

// x += a p ; r -= a Ap with a = rz / pAp (pcg.py:109-111)
__global__ void pcg_update_xr_kernel(int n, const double *rz, const double *pap, double *x, double *r,
                                     const double *p, const double *ap) {
    const double a = rz[0] / pap[0];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        x[i] += a * p[i];
        r[i] -= a * ap[i];
    }
}

// p = z + (rz_new / rz) p (pcg.py:127)
__global__ void pcg_update_p_kernel(int n, const double *rznew, const double *rz, const double *z,
                                    double *p) {
    const double beta = rznew[0] / rz[0];
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

inline int grid_for(long long work, int threads, int cap = 148 * 16) {
    long long g = (work + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (int)g;
}

}  // namespace

extern "C" int rsc_csr_to_dense_batched(int count, const int *const *rowptr, const int *const *colidx,
                                        const double *const *values, const int *nrows, double *const *D,
                                        const int *ldd, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!rowptr || !colidx || !values || !nrows || !D || !ldd) return -2;
    static thread_local CsrDenseArgs a;
    for (int c0 = 0; c0 < count; c0 += MAXB) {
        const int cnt = count - c0 < MAXB ? count - c0 : MAXB;
        a.count = cnt;
        int maxr = 1;
        for (int i = 0; i < cnt; ++i) {
            a.rowptr[i] = rowptr[c0 + i];
            a.colidx[i] = colidx[c0 + i];
            a.values[i] = values[c0 + i];
            a.D[i] = D[c0 + i];
            a.nrows[i] = nrows[c0 + i];
            a.ldd[i] = ldd[c0 + i];
            maxr = nrows[c0 + i] > maxr ? nrows[c0 + i] : maxr;
        }
        dim3 grid((maxr + 7) / 8 < 64 ? (maxr + 7) / 8 : 64, cnt);
        csr_to_dense_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

extern "C" int rsc_spmm_csr_batched(int count, const int *const *rowptr, const int *const *colidx,
                                    const double *const *values, const int *nrows, const int *r,
                                    const double *const *X, const int *ldx, double alpha, double beta,
                                    double *const *Y, const int *ldy, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!rowptr || !colidx || !values || !nrows || !r || !X || !ldx || !Y || !ldy) return -2;
    static thread_local SpmmArgs a;
    for (int c0 = 0; c0 < count; c0 += MAXB) {
        const int cnt = count - c0 < MAXB ? count - c0 : MAXB;
        a.count = cnt;
        a.alpha = alpha;
        a.beta = beta;
        int maxr = 1;
        for (int i = 0; i < cnt; ++i) {
            a.rowptr[i] = rowptr[c0 + i]; a.colidx[i] = colidx[c0 + i]; a.values[i] = values[c0 + i];
            a.X[i] = X[c0 + i]; a.Y[i] = Y[c0 + i];
            a.nrows[i] = nrows[c0 + i]; a.r[i] = r[c0 + i]; a.ldx[i] = ldx[c0 + i]; a.ldy[i] = ldy[c0 + i];
            maxr = nrows[c0 + i] > maxr ? nrows[c0 + i] : maxr;
        }
        dim3 grid((maxr + 7) / 8 < 128 ? (maxr + 7) / 8 : 128, cnt);
        spmm_csr_batched_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

extern "C" int rsc_spmm_csr(int nrows, int r, const int *rowptr_dev, const int *colidx_dev,
                            const double *values_dev, const double *X_dev, int ldx, double alpha,
                            double beta, double *Y_dev, int ldy, void *stream) {
    if (nrows < 0) return -1;
    if (r < 0) return -2;
    if (nrows == 0 || r == 0) return 0;
    const int threads = 256;
    spmm_csr_kernel<<<grid_for((long long)nrows * 32, threads), threads, 0, (cudaStream_t)stream>>>(
        nrows, r, rowptr_dev, colidx_dev, values_dev, X_dev, ldx, alpha, beta, Y_dev, ldy);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_spmv_csr(int n, const int *rowptr_dev, const int *colidx_dev, const double *values_dev,
                            const double *x_dev, double *y_dev, void *stream) {
    if (n < 0) return -1;
    if (n == 0) return 0;
    const int threads = 256;
    spmv_csr_kernel<<<grid_for((long long)n * 8, threads), threads, 0, (cudaStream_t)stream>>>(
        n, rowptr_dev, colidx_dev, values_dev, x_dev, y_dev);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_gather_rows(int nrows, int ncols, const int *idx_dev, const double *src_dev, int lds,
                               double *dst_dev, int ldd, void *stream) {
    if (nrows < 0 || ncols < 0) return -1;
    if (nrows == 0 || ncols == 0) return 0;
    gather_rows_kernel<<<grid_for((long long)nrows * ncols, 256), 256, 0, (cudaStream_t)stream>>>(
        nrows, ncols, idx_dev, src_dev, lds, dst_dev, ldd);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_scatter_add_rows(int nrows, int ncols, const int *idx_dev, double alpha,
                                    const double *src_dev, int lds, double *dst_dev, int ldd, void *stream) {
    if (nrows < 0 || ncols < 0) return -1;
    if (nrows == 0 || ncols == 0) return 0;
    scatter_add_rows_kernel<<<grid_for((long long)nrows * ncols, 256), 256, 0, (cudaStream_t)stream>>>(
        nrows, ncols, idx_dev, alpha, src_dev, lds, dst_dev, ldd);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_dot(int n, const double *x_dev, const double *y_dev, double *out_dev, double *work_dev,
                       void *stream) {
    if (n < 0) return -1;
    cudaStream_t s = (cudaStream_t)stream;
    dot_partial_kernel<<<DOT_BLOCKS, DOT_THREADS, 0, s>>>(n, x_dev, y_dev, work_dev);
    dot_final_kernel<<<1, DOT_THREADS, 0, s>>>(DOT_BLOCKS, work_dev, out_dev);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_pcg_update_xr(int n, const double *rz_dev, const double *pap_dev, double *x_dev,
                                 double *r_dev, const double *p_dev, const double *ap_dev, void *stream) {
    if (n <= 0) return n < 0 ? -1 : 0;
    pcg_update_xr_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, rz_dev, pap_dev, x_dev, r_dev,
                                                                            p_dev, ap_dev);
    RSC_CHECK_LAUNCH();
    return 0;
}

extern "C" int rsc_pcg_update_p(int n, const double *rznew_dev, const double *rz_dev, const double *z_dev,
                                double *p_dev, void *stream) {
    if (n <= 0) return n < 0 ? -1 : 0;
    pcg_update_p_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, rznew_dev, rz_dev, z_dev, p_dev);
    RSC_CHECK_LAUNCH();
    return 0;
}

static std::atomic<long long> g_launches{0};
void rsc_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

extern "C" long long rsc_launch_counter(int reset) {
    return reset ? g_launches.exchange(0) : g_launches.load();
}

extern "C" const char *rsc_version(void) { return "rsc_b200 0.1 (sm_100a, FP64 DMMA)"; }

extern "C" int rsc_device_arch(void) {
#if defined(__CUDA_ARCH__)
    return __CUDA_ARCH__;
#else
    return 1000;
#endif
}
