// Fused batched Cholesky for n <= 256: one CTA (8 warps) factors one matrix in a
// single launch -- the whole blocked left-looking algorithm of potrf.cu without the
// 3 launches per 64-column panel.
//
// Reference: kernels.py:22-39 (dense_cholesky = LAPACK dpotrf lower + clean; info
// = 1-based first non-positive pivot).  Used for every POTRF of the path whose
// order is <= 256: config[1]'s 256x256 diagonal blocks, the sparse sweep's dense
// node diagonals (nc <= tau_D), diagonal-tree leaves and interior blocks.
//
// Per 64-column panel s (columns j0 = 64 s .. j0 + nb):
//   1. update   P = A[j0:n, panel] - L[j0:n, 0:j0] L[j0:j0+64, 0:j0]^T
//      DMMA.8x8x4; warp w owns panel rows 32w..32w+31 (accumulators in registers);
//      the K = j0 operand columns stream through a 3-stage cp.async ring in shared
//      memory -- rows 0..63 of each staged chunk are also the B operand.
//   2. factor + invert the 64x64 diagonal block in shared memory with all 256
//      threads as 2x2 blocks of 32: each 32x32 diagonal block right-looking with the
//      forward substitution for its inverse fused into the same sweep (one CTA
//      barrier per column), the off-diagonal blocks as small FMA products.  (A
//      row-per-thread Crout variant on 64 threads and a 64-wide right-looking sweep
//      were both latency-bound: with one CTA per SM nothing hides a long serial
//      column chain.)
//   3. below    L[j0+64:n, panel] = P_below Dinv^T   (DMMA, B = Dinv from smem)
// The matrix (<= 512 KB) stays L2-resident between the phases, so the panel rows
// round-trip through L2, not HBM.  Rows past n of a partial last panel are treated
// as identity rows, so the 64-row algorithm needs no special case.
#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int PF_THREADS = 256;
constexpr int PF_MAXB = 600;
constexpr int PF_KC = 8;       // k columns per staged chunk
constexpr int PF_LDS = 12;     // staged row stride (doubles): conflict-free fragments, 16 B rows
constexpr int PF_LDD = 68;     // inverse block stride (doubles): conflict-free fragments
constexpr int PF_LDF = 68;     // factor block stride (4 threads per row: conflict-free)
constexpr int PF_STAGES = 3;
constexpr int PF_STAGE_ROWS = 256;
constexpr int PF_STAGE_DBL = PF_STAGE_ROWS * PF_LDS;
constexpr int PF_SMEM = (PF_STAGES * PF_STAGE_DBL + 64 * PF_LDF + 64 * PF_LDD + 64) * 8 + 16;

struct PfArgs {
    int count;
    int base;
    double *A[PF_MAXB];
    double *Dinv[PF_MAXB];
    int n[PF_MAXB];
    int lda[PF_MAXB];
};

__device__ __forceinline__ void cp_async_16(void *smem, const double *gmem, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0));
}

// Stage rows [0, R) of columns [kc, kc+8) of the row-major block at src (leading
// dim ld) into buf (stride PF_LDS); rows [R, Rpad) are zero-filled.
__device__ __forceinline__ void stage_chunk(double *buf, const double *src, int ld, int R, int Rpad, int kc,
                                            bool vec16) {
    const int t = threadIdx.x;
    if (vec16) {
        for (int e = t; e < Rpad * 4; e += PF_THREADS) {
            const int r = e >> 2, c = (e & 3) * 2;
            const bool ok = r < R;
            cp_async_16(buf + r * PF_LDS + c, ok ? src + (long long)r * ld + kc + c : src, ok);
        }
    } else {
        for (int e = t; e < Rpad * 8; e += PF_THREADS) {
            const int r = e >> 3, c = e & 7;
            const bool ok = r < R;
            cp_async_8(buf + r * PF_LDS + c, ok ? src + (long long)r * ld + kc + c : src, ok);
        }
    }
}

// acc[rt][ct] += (-1 if NEG) A_stage[rows of warp] * B^T, one staged chunk (k = 8).
// A rows: warp w rows 32w + 8rt + g of abuf; B rows 8ct + g of bbuf (stride ldb).
template <bool NEG>
__device__ __forceinline__ void chunk_mma(double (&acc)[4][8][2], const double *abuf, const double *bbuf,
                                          int ldb, int warp, int lane) {
    const int g = lane >> 2, q = lane & 3;
#pragma unroll
    for (int kk = 0; kk < PF_KC; kk += 4) {
        double a[4], b[8];
#pragma unroll
        for (int rt = 0; rt < 4; ++rt) {
            const double x = abuf[(32 * warp + 8 * rt + g) * PF_LDS + kk + q];
            a[rt] = NEG ? -x : x;
        }
#pragma unroll
        for (int ct = 0; ct < 8; ++ct) b[ct] = bbuf[(8 * ct + g) * ldb + kk + q];
#pragma unroll
        for (int rt = 0; rt < 4; ++rt)
#pragma unroll
            for (int ct = 0; ct < 8; ++ct) dmma_8x8x4(acc[rt][ct][0], acc[rt][ct][1], a[rt], b[ct]);
    }
}

// Cholesky + inverse of the 32x32 diagonal block at offset o of Ds (stride PF_LDF,
// lower part in place -> L) with the inverse written to Is[o.., o..] (stride PF_LDD).
// Right-looking on unscaled columns with the forward substitution fused in: at step
// j every row i > j applies f = A_ij / d_j to A_ik -= f A_kj (j < k <= i) and
// B_ic -= f B_jc (c <= j, B = I); then L_ik = A_ik / sqrt(d_k), X_ic = B_ic / L_ii.
// 8 threads per row, one CTA barrier per column.  Returns the failing pivot (block
// relative) or -1, uniformly.
__device__ int chol_inv_32(double *Ds, double *Is, int o, double *rsv) {
    const int t = threadIdx.x, i = t >> 3, sub = t & 7;
    double *Ri = Ds + (o + i) * PF_LDF + o;
    double *Bi = Is + (o + i) * PF_LDD + o;
    for (int k = sub; k < 32; k += 8) Bi[k] = (k == i) ? 1.0 : 0.0;
    for (int j = 0; j < 32; ++j) {
        __syncthreads();
        const double dj = Ds[(o + j) * PF_LDF + o + j];
        if (!(dj > 0.0)) return j;  // uniform: every thread read dj
        if (i > j) {
            const double f = Ri[j] * (1.0 / dj);
            const double *Cj = Ds + o * PF_LDF + o + j;  // column j, row stride PF_LDF
            const double *Bj = Is + (o + j) * PF_LDD + o;
            const int k0 = j + 1 + ((sub - j - 1) & 7);
            double x[4], y[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // at most 4 columns per thread: loads first
                const int k = k0 + 8 * u, c = sub + 8 * u;
                x[u] = (k <= i) ? Cj[k * PF_LDF] : 0.0;
                y[u] = (c <= j) ? Bj[c] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int k = k0 + 8 * u, c = sub + 8 * u;
                if (k <= i) Ri[k] = fma(-f, x[u], Ri[k]);
                if (c <= j) Bi[c] = fma(-f, y[u], Bi[c]);
            }
        }
    }
    __syncthreads();
    if (t < 32) rsv[t] = rsqrt(Ds[(o + t) * PF_LDF + o + t]);
    __syncthreads();
    const double ri = rsv[i];
    for (int k = sub; k < 32; k += 8) {
        if (k <= i) {
            Ri[k] *= (k == i) ? ri : rsv[k];
            Bi[k] *= ri;
        } else {
            Bi[k] = 0.0;
        }
    }
    __syncthreads();
    return -1;
}

__device__ unsigned long long pf_phase_cycles[8];  // RSC_POTRF_TIMING diagnostics (CTA 0)

template <bool TIMING>
__global__ void __launch_bounds__(PF_THREADS, 1) potrf_fused_kernel(const __grid_constant__ PfArgs args,
                                                                     int *info) {
    extern __shared__ __align__(16) double sm[];
    double *stage = sm;                                    // PF_STAGES x PF_STAGE_DBL
    double *Ds = stage + PF_STAGES * PF_STAGE_DBL;          // 64 x PF_LDF: diagonal block / L
    double *Is = Ds + 64 * PF_LDF;                          // 64 x PF_LDD: its inverse
    double *invd = Is + 64 * PF_LDD;                        // 64: 1 / L_jj
    int *fail_s = reinterpret_cast<int *>(invd + 64);

    const int b = blockIdx.x;
    const int n = args.n[b];
    if (n <= 0) return;
    double *A = args.A[b];
    const int lda = args.lda[b];
    double *Dinv = args.Dinv[b];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int g = lane >> 2, q = lane & 3;
    const bool vec16 = ((lda & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);

    long long tp = TIMING ? clock64() : 0;
    auto mark = [&](int ph) {
        if (TIMING && threadIdx.x == 0 && blockIdx.x == 0) {
            const long long now = clock64();
            atomicAdd(&pf_phase_cycles[ph], (unsigned long long)(now - tp));
            tp = now;
        }
    };
    for (int j0 = 0; j0 < n; j0 += 64) {
        mark(7);
        const int M = n - j0;             // panel rows
        const int nb = M < 64 ? M : 64;   // panel columns
        double *P = A + (long long)j0 * lda + j0;  // panel origin
        // ---- 1. left-looking update of the panel --------------------------------------
        double acc[4][8][2];
        const bool active = 32 * warp < M;
#pragma unroll
        for (int rt = 0; rt < 4; ++rt)
#pragma unroll
            for (int ct = 0; ct < 8; ++ct) {
                const int r = 32 * warp + 8 * rt + g, c = 8 * ct + 2 * q;
                acc[rt][ct][0] = (r < M && c < nb) ? P[(long long)r * lda + c] : 0.0;
                acc[rt][ct][1] = (r < M && c + 1 < nb) ? P[(long long)r * lda + c + 1] : 0.0;
            }
        if (j0 > 0) {
            const double *Lrows = A + (long long)j0 * lda;  // L[j0:n, 0:j0]
            const int Rpad = M < 64 ? 64 : M;
            const int nch = j0 / PF_KC;
#pragma unroll
            for (int s = 0; s < PF_STAGES - 1; ++s) {
                if (s < nch) stage_chunk(stage + s * PF_STAGE_DBL, Lrows, lda, M, Rpad, s * PF_KC, vec16);
                cp_async_commit();
            }
            for (int c = 0; c < nch; ++c) {
                cp_async_wait<PF_STAGES - 2>();
                __syncthreads();
                const int nx = c + PF_STAGES - 1;
                if (nx < nch)
                    stage_chunk(stage + (nx % PF_STAGES) * PF_STAGE_DBL, Lrows, lda, M, Rpad, nx * PF_KC, vec16);
                cp_async_commit();
                const double *buf = stage + (c % PF_STAGES) * PF_STAGE_DBL;
                if (active) chunk_mma<true>(acc, buf, buf, PF_LDS, warp, lane);
            }
            cp_async_wait<0>();
        }
        // rows 0..63 of the panel -> Ds; the rest back to the panel in L2 (for phase 3)
        if (warp < 2) {
#pragma unroll
            for (int rt = 0; rt < 4; ++rt)
#pragma unroll
                for (int ct = 0; ct < 8; ++ct) {
                    const int r = 32 * warp + 8 * rt + g, c = 8 * ct + 2 * q;
                    Ds[r * PF_LDF + c] = acc[rt][ct][0];
                    Ds[r * PF_LDF + c + 1] = acc[rt][ct][1];
                }
        } else if (active && j0 > 0) {
#pragma unroll
            for (int rt = 0; rt < 4; ++rt)
#pragma unroll
                for (int ct = 0; ct < 8; ++ct) {
                    const int r = 32 * warp + 8 * rt + g, c = 8 * ct + 2 * q;
                    if (r < M) {
                        P[(long long)r * lda + c] = acc[rt][ct][0];
                        P[(long long)r * lda + c + 1] = acc[rt][ct][1];
                    }
                }
        }
        __syncthreads();
        mark(0);
        // ---- 2. factor + invert the diagonal block (all 256 threads) -----------------
        // 2x2 blocks of 32: chol+inv(D11); L21 = A21 inv11^T; A22 -= L21 L21^T;
        // chol+inv(A22); X21 = -inv22 L21 inv11.  Rows past nb are identity rows.
        {
            for (int e = t; e < 64 * 64; e += PF_THREADS) {
                const int i = e >> 6, k = e & 63;
                if (i >= nb) Ds[i * PF_LDF + k] = (k == i) ? 1.0 : 0.0;
            }
            double *T = stage;  // 32 x 33 scratch (the staging ring is idle here)
            int bad = chol_inv_32(Ds, Is, 0, invd);
            if (bad < 0) {
                // L21 = A21 inv11^T : L21[i][k] = sum_{m<=k} A21[i][m] inv11[k][m]
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = t + PF_THREADS * u, i = e >> 5, k = e & 31;
                    const double *a = Ds + (32 + i) * PF_LDF, *w = Is + k * PF_LDD;
                    double s0 = 0.0, s1 = 0.0;
                    int m = 0;
                    for (; m + 1 <= k; m += 2) { s0 = fma(a[m], w[m], s0); s1 = fma(a[m + 1], w[m + 1], s1); }
                    if (m <= k) s0 = fma(a[m], w[m], s0);
                    v[u] = s0 + s1;
                }
                __syncthreads();
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int e = t + PF_THREADS * u, i = e >> 5, k = e & 31;
                    Ds[(32 + i) * PF_LDF + k] = v[u];
                }
                __syncthreads();
                // A22 -= L21 L21^T (lower part incl. diagonal)
                for (int e = t; e < 32 * 32; e += PF_THREADS) {
                    const int i = e >> 5, j = e & 31;
                    if (j > i) continue;
                    const double *li = Ds + (32 + i) * PF_LDF, *lj = Ds + (32 + j) * PF_LDF;
                    double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
                    for (int m = 0; m < 32; m += 2) { s0 = fma(li[m], lj[m], s0); s1 = fma(li[m + 1], lj[m + 1], s1); }
                    Ds[(32 + i) * PF_LDF + 32 + j] -= s0 + s1;
                }
                bad = chol_inv_32(Ds, Is, 32, invd);
                if (bad >= 0) bad += 32;
            }
            if (bad < 0) {
                // T = L21 inv11 : T[i][c] = sum_{k>=c} L21[i][k] inv11[k][c]
                for (int e = t; e < 32 * 32; e += PF_THREADS) {
                    const int i = e >> 5, c = e & 31;
                    const double *l = Ds + (32 + i) * PF_LDF;
                    double s0 = 0.0, s1 = 0.0;
                    int k = c;
                    for (; k + 1 < 32; k += 2) {
                        s0 = fma(l[k], Is[k * PF_LDD + c], s0);
                        s1 = fma(l[k + 1], Is[(k + 1) * PF_LDD + c], s1);
                    }
                    if (k < 32) s0 = fma(l[k], Is[k * PF_LDD + c], s0);
                    T[i * 33 + c] = s0 + s1;
                }
                __syncthreads();
                // X21 = -inv22 T : X21[i][c] = -sum_{m<=i} inv22[i][m] T[m][c]
                for (int e = t; e < 32 * 32; e += PF_THREADS) {
                    const int i = e >> 5, c = e & 31;
                    const double *w = Is + (32 + i) * PF_LDD + 32;
                    double s0 = 0.0, s1 = 0.0;
                    int m = 0;
                    for (; m + 1 <= i; m += 2) {
                        s0 = fma(w[m], T[m * 33 + c], s0);
                        s1 = fma(w[m + 1], T[(m + 1) * 33 + c], s1);
                    }
                    if (m <= i) s0 = fma(w[m], T[m * 33 + c], s0);
                    Is[(32 + i) * PF_LDD + c] = -(s0 + s1);
                }
                __syncthreads();
                // zero the upper off-diagonal block and everything past nb
                for (int e = t; e < 64 * 64; e += PF_THREADS) {
                    const int i = e >> 6, k = e & 63;
                    if ((i < 32 && k >= 32) || i >= nb || k >= nb) Is[i * PF_LDD + k] = 0.0;
                }
                if (t == 0) *fail_s = -1;
            } else if (t == 0) {
                info[args.base + b] = j0 + bad + 1;
                *fail_s = bad;
            }
        }
        __syncthreads();
        mark(1);
        if (*fail_s >= 0) return;
        // diagonal block (upper zeroed), its inverse, and the clean strict upper part
        for (int e = t; e < nb * 64; e += PF_THREADS) {
            const int i = e >> 6, j = e & 63;
            if (j < nb) P[(long long)i * lda + j] = (j <= i) ? Ds[i * PF_LDF + j] : 0.0;
            Dinv[(long long)(j0 + i) * 64 + j] = Is[i * PF_LDD + j];
        }
        const int rest = n - j0 - nb;
        for (int e = t; e < nb * rest; e += PF_THREADS) {
            const int i = e / rest, j = e - i * rest;
            P[(long long)i * lda + nb + j] = 0.0;
        }
        mark(2);
        // ---- 3. rows below the diagonal block: X = P_below Dinv^T ---------------------
        const int M3 = M - 64;
        if (M3 > 0) {
            double *Pb = P + 64LL * lda;
            double acc3[4][8][2];
#pragma unroll
            for (int rt = 0; rt < 4; ++rt)
#pragma unroll
                for (int ct = 0; ct < 8; ++ct) acc3[rt][ct][0] = acc3[rt][ct][1] = 0.0;
            const bool act3 = 32 * warp < M3;
            constexpr int nch = 64 / PF_KC;
#pragma unroll
            for (int s = 0; s < PF_STAGES - 1; ++s) {
                stage_chunk(stage + s * PF_STAGE_DBL, Pb, lda, M3, M3, s * PF_KC, vec16);
                cp_async_commit();
            }
            for (int c = 0; c < nch; ++c) {
                cp_async_wait<PF_STAGES - 2>();
                __syncthreads();
                const int nx = c + PF_STAGES - 1;
                if (nx < nch) stage_chunk(stage + (nx % PF_STAGES) * PF_STAGE_DBL, Pb, lda, M3, M3, nx * PF_KC, vec16);
                cp_async_commit();
                if (act3)
                    chunk_mma<false>(acc3, stage + (c % PF_STAGES) * PF_STAGE_DBL, Is + c * PF_KC, PF_LDD, warp,
                                     lane);
            }
            cp_async_wait<0>();
            if (act3) {
#pragma unroll
                for (int rt = 0; rt < 4; ++rt)
#pragma unroll
                    for (int ct = 0; ct < 8; ++ct) {
                        const int r = 32 * warp + 8 * rt + g, c = 8 * ct + 2 * q;
                        if (r < M3) {
                            Pb[(long long)r * lda + c] = acc3[rt][ct][0];
                            Pb[(long long)r * lda + c + 1] = acc3[rt][ct][1];
                        }
                    }
            }
        }
        __syncthreads();
    }
}

}  // namespace

// Fused path of rsc_potrf_batched (every n <= 256); info must be zeroed by the caller.
int rsc_potrf_fused(int count, double *const *A, const int *n, const int *lda, double *const *Dinv,
                    int *info_dev, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(potrf_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
        cudaFuncSetAttribute(potrf_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
        attr = true;
    }
    static thread_local PfArgs pa;
    for (int c0 = 0; c0 < count; c0 += PF_MAXB) {
        const int cnt = count - c0 < PF_MAXB ? count - c0 : PF_MAXB;
        pa.count = cnt;
        pa.base = c0;
        for (int i = 0; i < cnt; ++i) {
            pa.A[i] = A[c0 + i];
            pa.Dinv[i] = Dinv[c0 + i];
            pa.n[i] = n[c0 + i];
            pa.lda[i] = lda[c0 + i];
        }
        static const bool timing = getenv("RSC_POTRF_TIMING") != nullptr;
        if (timing) potrf_fused_kernel<true><<<cnt, PF_THREADS, PF_SMEM, s>>>(pa, info_dev);
        else potrf_fused_kernel<false><<<cnt, PF_THREADS, PF_SMEM, s>>>(pa, info_dev);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

extern "C" int rsc_potrf_phase_cycles(unsigned long long *out8, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out8, pf_phase_cycles, 8 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[8] = {};
        cudaMemcpyToSymbol(pf_phase_cycles, z, sizeof(z));
    }
    return (int)e;
}
