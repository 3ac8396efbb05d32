// Multi-CTA column-pivoted Householder QR for sketches too large for one SM
// (e.g. 2048 x 508 off-diagonal sketches of the top separators).
//
// Same arithmetic contract as qrcp_kernel (LAPACK dlaqp2 pivoting, dlarfg
// reflectors, partial-norm downdating with the sqrt(eps) recomputation test,
// dorg2r for the kept columns; reference kernels.py:67-82), distributed by
// COLUMN OWNERSHIP: CTA b owns physical columns [b*cpc, (b+1)*cpc) and keeps them in
// shared memory for the whole factorization.  Pivoting never moves data: every CTA
// keeps the same position->column permutation and applies LAPACK's swap sequence
// to it redundantly, so the "first position of the largest partial norm" rule is
// reproduced exactly.  Per step: the owner of the pivot column forms the
// reflector and publishes it (v, tau) -> grid sync -> every CTA updates its own
// columns and downdates their norms -> grid sync.
//
// Q is formed afterwards by an ordinary kernel: column j of Q is
// H_0 ... H_j e_j applied right-to-left (dorg2r order), one warp per column.
#include <cooperative_groups.h>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int CT = 256;  // threads per CTA (8 warps)
constexpr double EPS = 2.220446049250313e-16;
constexpr double TOL3Z = 1.0536712127723509e-08;

struct CoopArgs {
    const double *G;
    int ldg, m, k, ldw, cpc;
    double *W;      // global column-major spill (ldw x k): reflectors for the Q kernel
    double *vn1, *vn2, *tau, *diagR, *vbuf;
    int *perm;      // final position -> physical column
};

template <bool SMEM>
__global__ void __launch_bounds__(CT) qrcp_coop_kernel(const CoopArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double sm[];
    const int m = a.m, k = a.k, ldw = a.ldw, cpc = a.cpc;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = CT / 32;
    const int c0 = blockIdx.x * cpc, c1 = min(k, c0 + cpc);
    double *cols = SMEM ? sm : a.W + (long long)c0 * ldw;            // owned columns
    double *v = SMEM ? sm + (long long)cpc * ldw : nullptr;            // reflector copy
    int *pos2phys = reinterpret_cast<int *>(SMEM ? v + m : sm);
    int *posof = pos2phys + k;
    __shared__ double red[32];
    __shared__ int piv_s;
    __shared__ double vsm_fallback[1];
    (void)vsm_fallback;

    // load owned columns (transposed from row-major G) and their norms
    for (long long e = t; e < (long long)m * (c1 - c0); e += CT) {
        const int r = (int)(e / (c1 - c0)), j = (int)(e % (c1 - c0));
        cols[(long long)j * ldw + r] = a.G[(long long)r * a.ldg + c0 + j];
    }
    for (int j = t; j < k; j += CT) { pos2phys[j] = j; posof[j] = j; }
    __syncthreads();
    for (int j = warp; j < c1 - c0; j += nw) {
        const double *cj = cols + (long long)j * ldw;
        double s = 0.0;
        for (int r = lane; r < m; r += 32) s += cj[r] * cj[r];
        s = sqrt(warp_sum(s));
        if (lane == 0) { a.vn1[c0 + j] = s; a.vn2[c0 + j] = s; }
    }
    grid.sync();

    const int kmin = m < k ? m : k;
    for (int i = 0; i < kmin; ++i) {
        // 1. pivot: first position j >= i with the largest vn1 (identical in every CTA)
        if (warp == 0) {
            double best = -1.0;
            int bp = k;
            for (int j = i + lane; j < k; j += 32) {
                const double vv = __ldcg(a.vn1 + pos2phys[j]);
                if (vv > best) { best = vv; bp = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
            }
            if (lane == 0) {
                if (bp >= k) bp = i;  // NaN norms: keep the order
                const int ci = pos2phys[i], cp = pos2phys[bp];
                pos2phys[i] = cp; pos2phys[bp] = ci;
                posof[cp] = i; posof[ci] = bp;
                piv_s = cp;
            }
        }
        __syncthreads();
        const int pc = piv_s;
        // 2. the owner of the pivot column forms and publishes the reflector
        if (pc >= c0 && pc < c1) {
            double *ci = cols + (long long)(pc - c0) * ldw;
            double part = 0.0;
            for (int r = i + 1 + t; r < m; r += CT) part += ci[r] * ci[r];
            const double xnorm = sqrt(block_sum(part, red));
            const double alpha = ci[i];
            double tau = 0.0, beta = alpha, scal = 0.0;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            __syncthreads();
            for (int r = i + 1 + t; r < m; r += CT) {
                const double x = (xnorm != 0.0) ? ci[r] * scal : ci[r];
                ci[r] = x;
                a.vbuf[r] = x;
            }
            if (t == 0) {
                ci[i] = beta;
                a.vbuf[i] = 1.0;
                a.tau[i] = tau;
                a.diagR[i] = beta;
            }
            __threadfence();
        }
        grid.sync();
        // 3. every CTA applies H_i^T to its unchosen columns and downdates their norms
        const double tau = __ldcg(a.tau + i);
        const double *vsrc;
        if (SMEM) {
            for (int r = i + t; r < m; r += CT) v[r] = __ldcg(a.vbuf + r);
            __syncthreads();
            vsrc = v;
        } else {
            vsrc = a.vbuf;
        }
        for (int j = warp; j < c1 - c0; j += nw) {
            const int phys = c0 + j;
            if (posof[phys] <= i) continue;
            double *cj = cols + (long long)j * ldw;
            if (tau != 0.0) {
                double w = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) w += (SMEM ? vsrc[r] : __ldcg(vsrc + r)) * cj[r];
                w = warp_sum(w) + cj[i];
                const double f = tau * w;
                for (int r = i + 1 + lane; r < m; r += 32) cj[r] -= f * (SMEM ? vsrc[r] : __ldcg(vsrc + r));
                __syncwarp();
                if (lane == 0) cj[i] -= f;
                __syncwarp();
            }
            const double v1 = a.vn1[phys];
            if (v1 != 0.0) {
                double temp = fabs(cj[i]) / v1;
                temp = 1.0 - temp * temp;
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = v1 / a.vn2[phys];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= TOL3Z) {
                    double s = 0.0;
                    for (int r = i + 1 + lane; r < m; r += 32) s += cj[r] * cj[r];
                    s = (i + 1 < m) ? sqrt(warp_sum(s)) : 0.0;
                    if (lane == 0) { a.vn1[phys] = s; a.vn2[phys] = s; }
                } else if (lane == 0) {
                    a.vn1[phys] = v1 * sqrt(temp);
                }
            }
            __syncwarp();
        }
        __threadfence();
        grid.sync();
    }
    // spill the owned columns (reflectors) for the Q kernel; publish the permutation
    if (SMEM)
        for (long long e = t; e < (long long)ldw * (c1 - c0); e += CT) a.W[(long long)c0 * ldw + e] = cols[e];
    if (blockIdx.x == 0)
        for (int j = t; j < k; j += CT) a.perm[j] = pos2phys[j];
}

// Q[:, j] = H_0 ... H_j e_j for j < rank; one warp per output column, the column
// lives in shared memory.  Also writes the kept rank (every CTA computes it).
__global__ void __launch_bounds__(CT) qr_form_q_kernel(const double *__restrict__ W, int ldw, int m, int k,
                                                        const int *__restrict__ perm,
                                                        const double *__restrict__ tau,
                                                        const double *__restrict__ diagR, double *Q, int ldq,
                                                        int *rank_out, int warps_per_cta) {
    extern __shared__ __align__(16) double qcol[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ int rank_s;
    if (threadIdx.x == 0) {
        const double d0 = fabs(diagR[0]);
        const int kmin = m < k ? m : k;
        int r = 0;
        if (d0 != 0.0) {
            const double cut = (double)(m > k ? m : k) * EPS * d0;
            for (int i = 0; i < kmin; ++i)
                if (fabs(diagR[i]) > cut) ++r;
        }
        rank_s = r;
        if (blockIdx.x == 0) *rank_out = r;
    }
    __syncthreads();
    const int rank = rank_s;
    if (warp >= warps_per_cta) return;
    const int j = blockIdx.x * warps_per_cta + warp;
    if (j >= rank) return;
    double *q = qcol + (long long)warp * m;
    for (int r = lane; r < m; r += 32) q[r] = (r == j) ? 1.0 : 0.0;
    __syncwarp();
    for (int i = j; i >= 0; --i) {
        const double *vi = W + (long long)perm[i] * ldw;  // v_i[i] = 1 implicitly
        const double ti = tau[i];
        double w = 0.0;
        for (int r = i + 1 + lane; r < m; r += 32) w += vi[r] * q[r];
        w = warp_sum(w) + q[i];
        const double f = ti * w;
        __syncwarp();
        for (int r = i + 1 + lane; r < m; r += 32) q[r] -= f * vi[r];
        if (lane == 0) q[i] -= f;
        __syncwarp();
    }
    for (int r = lane; r < m; r += 32) Q[(long long)r * ldq + j] = q[r];
}

}  // namespace

// workspace doubles of one cooperative QR
long long rsc_qrcp_coop_doubles(int m, int k) {
    const long long ldw = m | 1;
    return ldw * k + 4LL * k + m + k + 64;
}

int rsc_qrcp_coop(const double *G, int m, int k, int ldg, double *Q, int ldq, int *rank_dev, double *work,
                  cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    CoopArgs a;
    a.G = G; a.ldg = ldg; a.m = m; a.k = k; a.ldw = m | 1;
    a.W = work;
    a.vn1 = work + (long long)a.ldw * k;
    a.vn2 = a.vn1 + k;
    a.tau = a.vn2 + k;
    a.diagR = a.tau + k;
    a.vbuf = a.diagR + k;
    a.perm = reinterpret_cast<int *>(a.vbuf + m);
    int cpc = (k + nsm - 1) / nsm;
    const size_t idx_bytes = sizeof(int) * 2 * (size_t)k;
    size_t smem = (size_t)cpc * a.ldw * 8 + (size_t)m * 8 + idx_bytes;
    const bool use_smem = smem <= 200 * 1024;
    void *fn;
    if (use_smem) {
        fn = (void *)qrcp_coop_kernel<true>;
    } else {
        smem = idx_bytes;
        fn = (void *)qrcp_coop_kernel<false>;
    }
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, CT, smem);
    if (per_sm < 1) return 77;
    // enough CTAs to own every column, never more than can be co-resident
    int nblk = (k + cpc - 1) / cpc;
    while (nblk > nsm * per_sm) {
        ++cpc;
        nblk = (k + cpc - 1) / cpc;
    }
    if (use_smem) {
        smem = (size_t)cpc * a.ldw * 8 + (size_t)m * 8 + idx_bytes;
        if (smem > 200 * 1024) return 78;
    }
    a.cpc = cpc;
    void *args[] = {&a};
    cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(nblk), dim3(CT), args, smem, s);
    rsc_count_launch();
    if (e != cudaSuccess) return (int)e;
    // Q formation
    int wpc = (int)((200 * 1024) / ((size_t)m * 8));
    wpc = wpc < 1 ? 1 : (wpc > CT / 32 ? CT / 32 : wpc);
    if ((size_t)m * 8 > 200 * 1024) return 79;
    const size_t qsmem = (size_t)wpc * m * 8;
    cudaFuncSetAttribute(qr_form_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsmem);
    const int kmin = m < k ? m : k;
    const int qblocks = (kmin + wpc - 1) / wpc;
    qr_form_q_kernel<<<qblocks > 0 ? qblocks : 1, CT, qsmem, s>>>(a.W, a.ldw, m, k, a.perm, a.tau, a.diagR, Q, ldq,
                                                                  rank_dev, wpc);
    RSC_CHECK_LAUNCH();
    return 0;
}
