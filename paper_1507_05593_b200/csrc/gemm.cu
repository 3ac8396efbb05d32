// Grouped FP64 DMMA GEMM with optional gather (rows of op(B)) and scatter (rows /
// columns of C) index maps and an atomic-accumulate epilogue.
//
// This is the workhorse of the numeric factorization: every Schur update
// (gather panel rows -> DMMA -> scatter-subtract into the target block), every
// implicit sketch product and every blocked triangular solve step is one problem of
// a grouped launch.  One CTA computes one 64x64 tile of one problem; the problem
// descriptors travel in the kernel parameter block (__grid_constant__, up to
// RSC_GEMM_MAXP per launch), so a launch needs no descriptor upload.
//
// Tile: 64x64x16, 128 threads = 2x2 warps of 32x32 (4x4 DMMA.8x8x4 fragments,
// 32 FP64 accumulators per thread).  Operands are staged global->shared with
// 8-byte cp.async (zero-filled at the ragged edges) in a 2-stage pipeline.  The
// shared layouts are chosen per transpose case so both the cp.async stores and the
// fragment loads are bank-conflict-free (a 32-lane FP64 fragment load = 2
// wavefronts, the minimum).
#include "common.cuh"

namespace {

#ifndef RSC_GEMM_BK
#define RSC_GEMM_BK 16
#endif
constexpr int BM = 64, BN = 64, BK = RSC_GEMM_BK, NT = 128;
constexpr int PADK = BK + 4;   // [m][k] / [n][k] row stride (doubles)
constexpr int PADM = BM + 4;   // [k][m] / [k][n] row stride: 2*PADM = 8 mod 32 banks
constexpr int A_SZ = (BM * PADK > BK * PADM) ? BM * PADK : BK * PADM;
constexpr int B_SZ = A_SZ;
constexpr int MAXP = 192;
#ifndef RSC_GEMM_STAGES
#define RSC_GEMM_STAGES 2
#endif
constexpr int STAGES = RSC_GEMM_STAGES;
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_SZ + B_SZ) * sizeof(double);

struct GemmArgs {
    int count;
    long long tile_begin[MAXP + 1];
    rsc_gemm_problem p[MAXP];
};

template <bool TA, bool TB>
__device__ __forceinline__ void load_tiles(const rsc_gemm_problem &P, const double *A,
                                           const double *B, int m0, int n0, int k0,
                                           double *sA, double *sB) {
    const int t = threadIdx.x;
    if (!TA) {  // A row-major M x K, contiguous along k
        const int k = t % BK, mr = t / BK;
#pragma unroll
        for (int i = 0; i < BM * BK / NT; ++i) {
            const int m = mr + (NT / BK) * i;
            const bool v = (m0 + m < P.M) && (k0 + k < P.K);
            const double *src = v ? A + (long long)(m0 + m) * P.lda + (k0 + k) : A;
            cp_async_8(&sA[m * PADK + k], src, v);
        }
    } else {  // A stored K x M, contiguous along m
        const int m = t & 63, kr = t >> 6;
#pragma unroll
        for (int i = 0; i < BK / 2; ++i) {
            const int k = kr + 2 * i;
            const bool v = (m0 + m < P.M) && (k0 + k < P.K);
            const double *src = v ? A + (long long)(k0 + k) * P.lda + (m0 + m) : A;
            cp_async_8(&sA[k * PADM + m], src, v);
        }
    }
    if (!TB) {  // op(B) = B (K x N), contiguous along n, optional row gather
        const int n = t & 63, kr = t >> 6;
#pragma unroll
        for (int i = 0; i < BK / 2; ++i) {
            const int k = kr + 2 * i;
            const bool v = (n0 + n < P.N) && (k0 + k < P.K);
            const double *src = B;
            if (v) {
                const int row = P.b_rows ? __ldg(P.b_rows + k0 + k) : (k0 + k);
                src = B + (long long)row * P.ldb + (n0 + n);
            }
            cp_async_8(&sB[k * PADM + n], src, v);
        }
    } else {  // op(B) = B^T with B stored N x K, contiguous along k
        const int k = t % BK, nr = t / BK;
#pragma unroll
        for (int i = 0; i < BN * BK / NT; ++i) {
            const int n = nr + (NT / BK) * i;
            const bool v = (n0 + n < P.N) && (k0 + k < P.K);
            const double *src = v ? B + (long long)(n0 + n) * P.ldb + (k0 + k) : B;
            cp_async_8(&sB[n * PADK + k], src, v);
        }
    }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT) gemm_grouped_kernel(const __grid_constant__ GemmArgs args) {
    extern __shared__ __align__(16) double gsm[];
    double(*sA)[A_SZ] = reinterpret_cast<double(*)[A_SZ]>(gsm);
    double(*sB)[B_SZ] = reinterpret_cast<double(*)[B_SZ]>(gsm + STAGES * A_SZ);

    // locate problem: last p with tile_begin[p] <= blockIdx.x
    const long long tile = blockIdx.x;
    int lo = 0, hi = args.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (args.tile_begin[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const rsc_gemm_problem &P = args.p[lo];
    const long long local = tile - args.tile_begin[lo];
    const int tm = (P.M + BM - 1) / BM, tn = (P.N + BN - 1) / BN;
    const int b = (int)(local / ((long long)tm * tn));
    const int rem = (int)(local - (long long)b * tm * tn);
    const int m0 = (rem / tn) * BM, n0 = (rem % tn) * BN;

    const double *A = P.A + (long long)b * P.strideA;
    const double *B = P.B + (long long)b * P.strideB;
    double *C = P.C + (long long)b * P.strideC;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = (P.K + BK - 1) / BK;
    if (nk > 0) {
        // STAGES-deep cp.async pipeline, one CTA barrier per k-tile
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nk) load_tiles<TA, TB>(P, A, B, m0, n0, s * BK, sA[s], sB[s]);
            cp_async_commit();
        }
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();  // tile kt landed; everyone is done with tile kt-1's stage
            const int pf = kt + STAGES - 1;
            if (pf < nk) load_tiles<TA, TB>(P, A, B, m0, n0, pf * BK, sA[pf % STAGES], sB[pf % STAGES]);
            cp_async_commit();
            const double *a_s = sA[kt % STAGES];
            const double *b_s = sB[kt % STAGES];
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double af[4], bf[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = wm + i * 8 + g;
                    af[i] = TA ? a_s[(kk + q) * PADM + m] : a_s[m * PADK + kk + q];
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int n = wn + j * 8 + g;
                    bf[j] = TB ? b_s[n * PADK + kk + q] : b_s[(kk + q) * PADM + n];
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
    }

    // epilogue
    const double alpha = P.alpha, beta = P.beta;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm + i * 8 + g;
        if (row >= P.M) continue;
        const long long crow = (long long)(P.c_rows ? __ldg(P.c_rows + row) : row) * P.ldc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = n0 + wn + j * 8 + 2 * q + e;
                if (col >= P.N) continue;
                const int ccol = P.c_cols ? __ldg(P.c_cols + col) : col;
                double *dst = C + crow + ccol;
                const double v = alpha * acc[i][j][e];
                if (P.atomic) {
                    atomicAdd(dst, v);
                } else if (beta == 0.0) {
                    *dst = v;
                } else {
                    *dst = v + beta * (*dst);
                }
            }
        }
    }
}

template <bool TA, bool TB>
int launch_chunk(GemmArgs &args, long long tiles, cudaStream_t s) {
    if (tiles <= 0) return 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_grouped_kernel<TA, TB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
        attr = true;
    }
    gemm_grouped_kernel<TA, TB><<<(unsigned)tiles, NT, SMEM_BYTES, s>>>(args);
    RSC_CHECK_LAUNCH();
    return 0;
}

}  // namespace

extern "C" int rsc_gemm_grouped(int transA, int transB, const rsc_gemm_problem *problems,
                                int count, void *stream) {
    if (count < 0) return -4;
    if (count == 0) return 0;
    if (!problems) return -3;
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local GemmArgs args;  // ~30 KB; copied into the launch parameter block
    int i = 0;
    while (i < count) {
        args.count = 0;
        long long tiles = 0;
        while (i < count && args.count < MAXP) {
            const rsc_gemm_problem &p = problems[i++];
            if (p.M <= 0 || p.N <= 0 || p.batch <= 0) continue;
            if (transB && p.b_rows) return -3;
            if (p.K < 0) return -3;
            const long long tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
            args.tile_begin[args.count] = tiles;
            args.p[args.count] = p;
            tiles += tm * tn * p.batch;
            args.count++;
        }
        if (args.count == 0) continue;
        args.tile_begin[args.count] = tiles;
        int rc;
        if (!transA && !transB) rc = launch_chunk<false, false>(args, tiles, s);
        else if (!transA && transB) rc = launch_chunk<false, true>(args, tiles, s);
        else if (transA && !transB) rc = launch_chunk<true, false>(args, tiles, s);
        else rc = launch_chunk<true, true>(args, tiles, s);
        if (rc) return rc;
    }
    return 0;
}
