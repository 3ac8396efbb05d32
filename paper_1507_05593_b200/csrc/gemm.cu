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

// Per-thread operand loader: the 8 A and 8 B elements a thread stages per k-tile sit
// at fixed (row, column) offsets of the tile, so their addresses, smem slots and the
// M / N validity are computed once per CTA; a k-tile only advances the pointers and
// checks the K bound.  (Recomputing all of that per element per tile, with a branch
// per gathered row, had the k-loop at ~11 instructions per DMMA.)
template <bool TA, bool TB, bool GATHER>
struct Loader {
    const double *a;      // element 0 of this thread's A slots at k0 = 0
    const double *b;      // element 0 of this thread's B slots (no gather) / column base (gather)
    const int *rows;      // b_rows (gather) or nullptr
    long long a_i, a_k;   // A: stride between the 8 slots, advance per k-tile
    long long b_i, b_k;
    long long ldb;
    unsigned amask, bmask;  // M / N validity of the 8 slots
    int ka, kb;           // k offset of slot 0 within the tile (A / B); slots add 2*i when k varies
    int sa, sb;           // smem offset of slot 0; slot stride below
    int K;
    int grow[8];          // gathered B rows of the NEXT load() (prefetched one k-tile ahead)

    // indices of the 8 gathered op(B) rows this thread stages for k-tile kt: loaded
    // one load() ahead so the dependent index read never sits in front of the
    // cp.async issue (it cost 10-20% on the gathered sweep products)
    __device__ __forceinline__ void fetch_rows(int kt) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int k = kt * BK + kb + 2 * i;
            grow[i] = ((bmask & 1) && k < K) ? __ldg(rows + k) : -1;
        }
    }

    __device__ __forceinline__ void init(const rsc_gemm_problem &P, const double *A, const double *B, int m0,
                                         int n0) {
        const int t = threadIdx.x;
        K = P.K;
        amask = bmask = 0;
        if (!TA) {  // A row-major M x K: slot i = row (t/BK) + 8i, column k = t%BK
            const int k = t % BK, mr = t / BK;
            a = A + (long long)(m0 + mr) * P.lda + k;
            a_i = (long long)(NT / BK) * P.lda;
            a_k = BK;
            ka = k;
            sa = mr * PADK + k;
#pragma unroll
            for (int i = 0; i < BM * BK / NT; ++i)
                if (m0 + mr + (NT / BK) * i < P.M) amask |= 1u << i;
        } else {    // A stored K x M: slot i = k row (t>>6) + 2i, column m = t&63
            const int m = t & 63, kr = t >> 6;
            a = A + (long long)kr * P.lda + m0 + m;
            a_i = 2LL * P.lda;
            a_k = (long long)BK * P.lda;
            ka = kr;
            sa = kr * PADM + m;
            if (m0 + m < P.M) amask = 0xffu;
        }
        rows = nullptr;
        ldb = P.ldb;
        if (!TB) {  // op(B) = B (K x N): slot i = k row (t>>6) + 2i, column n = t&63
            const int n = t & 63, kr = t >> 6;
            rows = GATHER ? P.b_rows : nullptr;
            b = rows ? B + n0 + n : B + (long long)kr * P.ldb + n0 + n;
            b_i = 2LL * P.ldb;
            b_k = (long long)BK * P.ldb;
            kb = kr;
            sb = kr * PADM + n;
            if (n0 + n < P.N) bmask = 0xffu;
            if (GATHER && rows) fetch_rows(0);
        } else {    // op(B) = B^T, B stored N x K: slot i = row (t/BK) + 8i, column k = t%BK
            const int k = t % BK, nr = t / BK;
            b = B + (long long)(n0 + nr) * P.ldb + k;
            b_i = (long long)(NT / BK) * P.ldb;
            b_k = BK;
            kb = k;
            sb = nr * PADK + k;
#pragma unroll
            for (int i = 0; i < BN * BK / NT; ++i)
                if (n0 + nr + (NT / BK) * i < P.N) bmask |= 1u << i;
        }
    }

    // stage k-tile kt into sA / sB
    __device__ __forceinline__ void load(int kt, double *sA, double *sB) {
        const int k0 = kt * BK;
        if (!TA) {
            const double *p = a + (long long)kt * a_k;
            const bool kv = k0 + ka < K;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool v = kv && ((amask >> i) & 1);
                cp_async_8(&sA[sa + i * (NT / BK) * PADK], v ? p + i * a_i : a, v);
            }
        } else {
            const double *p = a + (long long)kt * a_k;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool v = (amask & 1) && (k0 + ka + 2 * i < K);
                cp_async_8(&sA[sa + 2 * i * PADM], v ? p + i * a_i : a, v);
            }
        }
        if (!TB) {
            if (GATHER && rows) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool v = grow[i] >= 0;
                    cp_async_8(&sB[sb + 2 * i * PADM], b + (long long)(v ? grow[i] : 0) * ldb, v);
                }
                fetch_rows(kt + 1);  // load() is called for consecutive k-tiles
            } else {
                const double *p = b + (long long)kt * b_k;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const bool v = (bmask & 1) && (k0 + kb + 2 * i < K);
                    cp_async_8(&sB[sb + 2 * i * PADM], v ? p + i * b_i : b, v);
                }
            }
        } else {
            const double *p = b + (long long)kt * b_k;
            const bool kv = k0 + kb < K;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const bool v = kv && ((bmask >> i) & 1);
                cp_async_8(&sB[sb + i * (NT / BK) * PADK], v ? p + i * b_i : b, v);
            }
        }
    }
};

template <bool TA, bool TB, bool GATHER>
#ifndef RSC_GEMM_MINB
#define RSC_GEMM_MINB 1
#endif
__global__ void __launch_bounds__(NT, RSC_GEMM_MINB) gemm_grouped_kernel(const __grid_constant__ GemmArgs args) {
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
    Loader<TA, TB, GATHER> ld;
    ld.init(P, A, B, m0, n0);
    if (nk > 0) {
        // STAGES-deep cp.async pipeline, one CTA barrier per k-tile
#pragma unroll
        for (int s = 0; s < STAGES - 1; ++s) {
            if (s < nk) ld.load(s, sA[s], sB[s]);
            cp_async_commit();
        }
        for (int kt = 0; kt < nk; ++kt) {
            cp_async_wait<STAGES - 2>();
            __syncthreads();  // tile kt landed; everyone is done with tile kt-1's stage
            const int pf = kt + STAGES - 1;
            if (pf < nk) ld.load(pf, sA[pf % STAGES], sB[pf % STAGES]);
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

template <bool TA, bool TB, bool GATHER>
int launch_chunk(GemmArgs &args, long long tiles, cudaStream_t s) {
    if (tiles <= 0) return 0;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_grouped_kernel<TA, TB, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
        attr = true;
    }
    gemm_grouped_kernel<TA, TB, GATHER><<<(unsigned)tiles, NT, SMEM_BYTES, s>>>(args);
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
        bool gather = false;
        while (i < count && args.count < MAXP) {
            const rsc_gemm_problem &p = problems[i++];
            if (p.M <= 0 || p.N <= 0 || p.batch <= 0) continue;
            if (transB && p.b_rows) return -3;
            if (p.K < 0) return -3;
            const long long tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
            args.tile_begin[args.count] = tiles;
            args.p[args.count] = p;
            gather |= p.b_rows != nullptr;
            tiles += tm * tn * p.batch;
            args.count++;
        }
        if (args.count == 0) continue;
        args.tile_begin[args.count] = tiles;
        int rc;
        // the gathered-B loader is its own instantiation: its index prefetch costs the
        // plain kernels ~2.5% (registers), it is only used for launches that gather
        if (!transA && !transB) rc = gather ? launch_chunk<false, false, true>(args, tiles, s)
                                            : launch_chunk<false, false, false>(args, tiles, s);
        else if (!transA && transB) rc = launch_chunk<false, true, false>(args, tiles, s);
        else if (transA && !transB) rc = gather ? launch_chunk<true, false, true>(args, tiles, s)
                                                : launch_chunk<true, false, false>(args, tiles, s);
        else rc = launch_chunk<true, true, false>(args, tiles, s);
        if (rc) return rc;
    }
    return 0;
}
