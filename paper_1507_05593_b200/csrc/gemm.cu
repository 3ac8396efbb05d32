// Grouped FP64 DMMA GEMM with optional gather (rows of op(B)) and scatter (rows /
// columns of C) index maps, and a DETERMINISTIC ordered accumulation for problems
// that share a target block.
//
// This is the workhorse of the numeric factorization: every Schur update
// (gather panel rows -> DMMA -> scatter-subtract into the target block), every
// implicit sketch product and every blocked triangular solve step is one problem of
// a grouped launch.  One CTA computes one 64x64 tile of one problem; the problem
// descriptors travel in the kernel parameter block (__grid_constant__, up to
// MAXP per launch), so a launch needs no descriptor upload.
//
// Tile: 64x64x16, 128 threads = 2x2 warps of 32x32 (4x4 DMMA.8x8x4 fragments,
// 32 FP64 accumulators per thread).  Operands are staged global->shared with
// 8-byte cp.async (zero-filled at the ragged edges) in a 2-stage pipeline.  The
// shared layouts are chosen per transpose case so both the cp.async stores and the
// fragment loads are bank-conflict-free (a 32-lane FP64 fragment load = 2
// wavefronts, the minimum).
//
// Accumulating problems (atomic != 0: Schur sums over update sources, implicit
// products over sources, split-K slabs) never race on C.  The host wrapper
// redirects each such problem's product to a private dense partial in the stream's
// workspace (plain coalesced stores), and ordered_reduce_kernel then adds the
// partials into C: one CTA owns a band of TR target rows of one target block and
// walks that block's problems in launch order, so every element of C receives
// C + P_1 + P_2 + ... in a fixed order -- the left-to-right `UD -= ...` order of
// the reference loops (factor.py:389-398, 445-455; diagblocks.py:231-262), and
// bit-identical results from run to run.  (Round 1 used FP64 atomicAdd here; the
// summation order then varied between runs and moved QRCP rank decisions that sit
// within rounding of the cutoff.)
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

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
    // a dependent ordered reduce (launched with programmatic stream serialization)
    // may start its list building while the last GEMM tiles run
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
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

    // epilogue (accumulating problems were redirected to private partials by the
    // host wrapper: here every problem is a plain store / read-modify-write)
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
                if (P.atomic) {  // diagnostic only (RSC_GEMM_ATOMIC=1): unordered FP64 atomics
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

// ---------------------------------------------------------------------------
// ordered reduction of the partials of accumulating problems

struct RedProb {
    const double *P;      // partial: batch x M x N, dense
    const int *c_rows;    // non-decreasing (or null = identity)
    const int *c_cols;    // strictly increasing (or null = identity)
    int M, N, g;          // g: group index
};

struct RedGroup {
    double *C;            // target block (all problems of the group share it)
    long long sC;         // batch stride of C
    int *rtab;            // [ext_r][np]: first local row of problem q mapped to target row t, or -1
    int *ctab;            // [np][ext_c]: local column of problem q mapped to target column c, or -1
    int ldc, ext_r, ext_c, batch, p0, np, TR, CW;
    int uniform;          // no column maps and every partial is ext_c wide (row-sweep fast path)
};

struct RedArgs {
    int count;            // groups
    int nprob;
    long long cta_begin[MAXP + 1];
    RedGroup g[MAXP];
    RedProb p[MAXP];
};

constexpr int RT = 256;
#ifndef RED_EPT
#define RED_EPT 1  // target elements per reduce thread
#endif
#ifndef RED_U
#define RED_U 16   // partial loads in flight per element
#endif
constexpr int TR_MAX = 64;
constexpr int MW = (MAXP + 31) / 32;  // problem-mask words per row

// Inverse maps of every mapped problem of the chunk (tables pre-set to -1).
__global__ void __launch_bounds__(RT) reduce_tables_kernel(const __grid_constant__ RedArgs a) {
    const RedProb &P = a.p[blockIdx.x];
    const RedGroup &G = a.g[P.g];
    const int q = blockIdx.x - G.p0;
    if (G.rtab) {
        for (int i = threadIdx.x; i < P.M; i += RT) {
            const int t = P.c_rows ? __ldg(P.c_rows + i) : i;
            // a run of repeated rows is represented by its first local row; the run
            // length rides in the high 8 bits (repeats: interior-block rows outside
            // the target structure, whose products are exact zeros)
            if (t < G.ext_r && (i == 0 || !P.c_rows || __ldg(P.c_rows + i - 1) != t)) {
                int run = 1;
                if (P.c_rows)
                    while (i + run < P.M && run < 255 && __ldg(P.c_rows + i + run) == t) ++run;
                G.rtab[(long long)t * G.np + q] = i | (run << 24);
            }
        }
    }
    if (G.ctab) {
        for (int j = threadIdx.x; j < P.N; j += RT) {
            const int c = P.c_cols ? __ldg(P.c_cols + j) : j;
            if (c < G.ext_c) G.ctab[(long long)q * G.ext_c + c] = j;
        }
    }
}

// One CTA owns a TR x CW tile of one target block; every element is a register sum
// C + P_q1 + P_q2 + ... over the problems that reach it, in problem order.  Per row
// of the tile the contributing (problem, first local row, run length) entries are
// collected once, in problem order, into shared memory by one warp per row (ballot
// + popc compaction).
//   Groups without column maps (the common case: sketch products scattered by row)
// store each entry as the address of the partial row itself (run length in the top
// byte): per partial element one shared-memory list read and one coalesced load, no
// map or descriptor lookups (the kernel was issue-bound at ~20 instructions per
// partial element).  Column-mapped groups keep the per-element lookup.
constexpr int LIST_MAX = 4096;  // entries per CTA (TR x np bounded by the host)

__global__ void __launch_bounds__(RT) ordered_reduce_kernel(const __grid_constant__ RedArgs a) {
    __shared__ unsigned long long s_buf[LIST_MAX];  // fast path: packed row pointers; else s_q | s_i
    __shared__ int s_cnt[TR_MAX];
    int *s_q = reinterpret_cast<int *>(s_buf);
    int *s_i = s_q + LIST_MAX;
    const long long cta = blockIdx.x;
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.cta_begin[mid] <= cta) lo = mid; else hi = mid - 1;
    }
    const RedGroup &G = a.g[lo];
    const long long local = cta - a.cta_begin[lo];
    const int nbr = (G.ext_r + G.TR - 1) / G.TR, nbc = (G.ext_c + G.CW - 1) / G.CW;
    const int b = (int)(local / ((long long)nbr * nbc));
    const int rem = (int)(local - (long long)b * nbr * nbc);
    const int t0 = (rem / nbc) * G.TR, c0 = (rem % nbc) * G.CW;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool fast = G.uniform != 0;
    if (fast) {
        // uniform group (no column maps, every partial ext_c wide): target column c is
        // column c of every contributing partial row.  One warp per tile row collects
        // the row's contributor list as packed partial-row addresses (the rtab row is
        // read in one go: every round's load in flight before the ballots); then the
        // tile's elements are dealt to threads, UF partial loads in flight per
        // element, summed in problem order.
        constexpr int UF = 8, QMAX = (MAXP + 31) / 32;
        for (int tt = warp; tt < G.TR; tt += RT / 32) {
            const int t = t0 + tt;
            int n = 0;
            if (t < G.ext_r) {
                int pre[QMAX];
#pragma unroll
                for (int r = 0; r < QMAX; ++r) {
                    const int q = r * 32 + lane;
                    pre[r] = -1;
                    if (q < G.np) {
                        if (G.rtab) pre[r] = __ldg(G.rtab + (long long)t * G.np + q);
                        else pre[r] = t < a.p[G.p0 + q].M ? (t | (1 << 24)) : -1;
                    }
                }
#pragma unroll
                for (int r = 0; r < QMAX; ++r) {
                    const int q = r * 32 + lane, i = pre[r];
                    const unsigned bal = __ballot_sync(0xffffffffu, i >= 0);
                    if (i >= 0) {
                        const RedProb &P = a.p[G.p0 + q];
                        const double *row = P.P + (long long)b * P.M * P.N + (long long)(i & 0xffffff) * P.N;
                        s_buf[tt * G.np + n + __popc(bal & ((1u << lane) - 1u))] =
                            (unsigned long long)row | ((unsigned long long)((unsigned)i >> 24) << 56);
                    }
                    n += __popc(bal);
                }
            }
            if (lane == 0) s_cnt[tt] = n;
        }
        asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the partials are written
        __syncthreads();
        const long long N = G.ext_c;
        double *C = G.C + (long long)b * G.sC;
        for (int e = threadIdx.x; e < G.TR * G.CW; e += RT) {
            const int tt = e / G.CW, t = t0 + tt, c = c0 + (e - tt * G.CW);
            const int n = s_cnt[tt];
            if (n == 0 || t >= G.ext_r || c >= G.ext_c) continue;
            const unsigned long long *lst = s_buf + tt * G.np;
            double *dst = C + (long long)t * G.ldc + c;
            double acc = *dst;
            for (int k0 = 0; k0 < n; k0 += UF) {
                double x[UF];
#pragma unroll
                for (int u = 0; u < UF; ++u) {
                    x[u] = 0.0;
                    if (k0 + u < n) {
                        const unsigned long long en = lst[k0 + u];
                        const double *src = reinterpret_cast<const double *>(en & 0x00ffffffffffffffULL) + c;
                        x[u] = src[0];
                        const int run = (int)(en >> 56);
                        for (int r = 1; r < run; ++r) x[u] += src[r * N];  // exact-zero repeats
                    }
                }
#pragma unroll
                for (int u = 0; u < UF; ++u)
                    if (k0 + u < n) acc += x[u];
            }
            *dst = acc;
        }
        return;
    }
    // per-row contributor lists: row tt owns entries [tt * np, tt * np + s_cnt[tt])
    for (int tt = warp; tt < G.TR; tt += RT / 32) {
        const int t = t0 + tt;
        int n = 0;
        if (t < G.ext_r) {
            for (int q0 = 0; q0 < G.np; q0 += 32) {
                const int q = q0 + lane;
                int i = -1;  // packed: first local row | run length << 24
                if (q < G.np) {
                    if (G.rtab) i = __ldg(G.rtab + (long long)t * G.np + q);
                    else i = t < a.p[G.p0 + q].M ? (t | (1 << 24)) : -1;
                }
                const unsigned bal = __ballot_sync(0xffffffffu, i >= 0);
                if (i >= 0) {
                    const int pos = tt * G.np + n + __popc(bal & ((1u << lane) - 1u));
                    s_q[pos] = q;
                    s_i[pos] = i;
                }
                n += __popc(bal);
            }
        }
        if (lane == 0) s_cnt[tt] = n;
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the partials are written
    __syncthreads();
    double *C = G.C + (long long)b * G.sC;
    constexpr int U = RED_U;
    for (int e = threadIdx.x; e < G.TR * G.CW; e += RT) {
        const int tt = e / G.CW, t = t0 + tt, c = c0 + (e - tt * G.CW);
        const int n = s_cnt[tt];
        if (n == 0 || t >= G.ext_r || c >= G.ext_c) continue;
        const int *lq = s_q + tt * G.np, *li = s_i + tt * G.np;
        double *dst = C + (long long)t * G.ldc + c;
        double acc = *dst;
        unsigned any = 0;
        for (int k0 = 0; k0 < n; k0 += U) {
            // U independent partial loads in flight, then the in-order sum
            double v[U];
            unsigned ok = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                v[u] = 0.0;
                const int k = k0 + u;
                if (k < n) {
                    const int q = lq[k];
                    const RedProb &P = a.p[G.p0 + q];
                    const int j = G.ctab ? __ldg(G.ctab + (long long)q * G.ext_c + c) : (c < P.N ? c : -1);
                    if (j >= 0) {
                        const int packed = li[k], i = packed & 0xffffff, run = (unsigned)packed >> 24;
                        const double *src = P.P + (long long)b * P.M * P.N + (long long)i * P.N + j;
                        double x = src[0];
                        for (int r = 1; r < run; ++r) x += src[(long long)r * P.N];  // exact-zero repeats
                        v[u] = x;
                        ok |= 1u << u;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
                if ((ok >> u) & 1u) acc += v[u];
            any |= ok;
        }
        if (any) *dst = acc;
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
    static const bool log = getenv("RSC_GEMM_LOG") != nullptr;  // diagnostics: one line per launch
    if (log) {
        double fl = 0.0, pad = 0.0, pad32m = 0.0, pad32n = 0.0;
        int maxk = 0;
        for (int i = 0; i < args.count; ++i) {
            const rsc_gemm_problem &p = args.p[i];
            const double pk = (double)((p.K + BK - 1) / BK * BK) * p.batch;
            const double pm = (p.M + BM - 1) / BM * BM, pn = (p.N + BN - 1) / BN * BN;
            fl += 2.0 * p.M * p.N * (double)p.K * p.batch;
            pad += 2.0 * pm * pn * pk;
            pad32m += 2.0 * ((p.M + 31) / 32 * 32) * pn * pk;  // with 32-row tiles
            pad32n += 2.0 * pm * ((p.N + 31) / 32 * 32) * pk;  // with 32-column tiles
            maxk = std::max(maxk, p.K);
        }
        fprintf(stderr, "GEMMLOG %d %d %d tiles %lld probs %d flops %.0f padded %.0f maxk %d pad32m %.0f pad32n %.0f\n",
                (int)TA, (int)TB, (int)GATHER, tiles, args.count, fl, pad, maxk, pad32m, pad32n);
    }
    return 0;
}

struct WsEntry {
    void *stream;
    char *ptr;
    long long bytes;
};
std::mutex g_ws_mu;
std::vector<WsEntry> g_ws;
WsEntry g_ws_default{nullptr, nullptr, 0};

WsEntry lookup_ws(void *stream) {
    std::lock_guard<std::mutex> lk(g_ws_mu);
    for (const WsEntry &e : g_ws)
        if (e.stream == stream) return e;
    return g_ws_default;
}

// Build and launch the ordered reduction for the accumulating problems of one chunk
// (reds, in launch order; argi = their slot in the GEMM launch).  Groups = distinct
// (C, strideC, batch) targets, each keeping its problems in order.  A group with a
// single unmapped problem needs no ordering: that problem is switched back to a
// direct C += alpha op(A) op(B) in the GEMM launch itself (returned in `direct`).
// Tables for the inverse maps are carved from `tab` (bytes available: tab_bytes).
int plan_reduce(const std::vector<rsc_gemm_problem> &reds, const std::vector<const double *> &parts,
                char *tab, long long tab_bytes, RedArgs &ra, std::vector<int> &direct, long long &ctas,
                long long &tab_used) {
    const int n = (int)reds.size();
    std::vector<int> gid(n, -1);
    std::vector<int> gfirst;
    for (int i = 0; i < n; ++i) {
        const rsc_gemm_problem &p = reds[i];
        int g = -1;
        for (int k = (int)gfirst.size() - 1; k >= 0; --k) {
            const rsc_gemm_problem &f = reds[gfirst[k]];
            if (f.C == p.C && f.strideC == p.strideC && f.batch == p.batch) { g = k; break; }
        }
        if (g < 0) {
            g = (int)gfirst.size();
            gfirst.push_back(i);
        }
        gid[i] = g;
    }
    ra.count = 0;
    ra.nprob = 0;
    ctas = 0;
    tab_used = 0;
    direct.clear();
    for (int g = 0; g < (int)gfirst.size(); ++g) {
        const rsc_gemm_problem &f = reds[gfirst[g]];
        int np = 0, er = 0, ec = 0;
        bool rmap = false, cmap = false, sameN = true;
        for (int i = 0; i < n; ++i) {
            if (gid[i] != g) continue;
            const rsc_gemm_problem &p = reds[i];
            if (p.ldc != f.ldc) return -7;
            if ((p.c_rows && p.ext_r <= 0) || (p.c_cols && p.ext_c <= 0)) return -3;
            er = std::max(er, p.ext_r > 0 ? p.ext_r : p.M);
            ec = std::max(ec, p.ext_c > 0 ? p.ext_c : p.N);
            rmap |= p.c_rows != nullptr;
            cmap |= p.c_cols != nullptr;
            sameN &= p.N == f.N;
            ++np;
        }
        if (np == 1 && !rmap && !cmap) {
            direct.push_back(gfirst[g]);
            continue;
        }
        RedGroup &G = ra.g[ra.count];
        G.C = f.C;
        G.sC = f.strideC;
        G.ldc = f.ldc;
        G.batch = f.batch;
        G.ext_r = er;
        G.ext_c = ec;
        G.p0 = ra.nprob;
        G.np = np;
        G.uniform = !cmap && sameN && f.N == ec;
        if (G.uniform) {  // ~4 target elements per thread, at most one row per warp
            G.CW = std::min(ec, 4 * RT);
            G.TR = std::max(1, std::min(std::min(RT / 32, std::max(1, 4 * RT / G.CW)), LIST_MAX / np));
        } else {
            G.CW = std::min(ec, RT);
            G.TR = std::max(1, std::min(std::min(TR_MAX, (RT * RED_EPT) / G.CW), LIST_MAX / np));
        }
        G.rtab = G.ctab = nullptr;
        const long long rb = rmap ? ((long long)er * np * 4 + 255) / 256 * 256 : 0;
        const long long cb = cmap ? ((long long)ec * np * 4 + 255) / 256 * 256 : 0;
        if (tab_used + rb + cb > tab_bytes) return -6;
        if (rmap) G.rtab = (int *)(tab + tab_used);
        if (cmap) G.ctab = (int *)(tab + tab_used + rb);
        tab_used += rb + cb;
        for (int i = 0; i < n; ++i) {
            if (gid[i] != g) continue;
            const rsc_gemm_problem &p = reds[i];
            RedProb &rp = ra.p[ra.nprob++];
            rp.P = parts[i];
            rp.c_rows = p.c_rows;
            rp.c_cols = p.c_cols;
            rp.M = p.M;
            rp.N = p.N;
            rp.g = ra.count;
        }
        ra.cta_begin[ra.count] = ctas;
        ctas += (long long)((er + G.TR - 1) / G.TR) * ((ec + G.CW - 1) / G.CW) * G.batch;
        ++ra.count;
    }
    ra.cta_begin[ra.count] = ctas;
    return 0;
}

struct RedStats {
    long long launches = 0, ctas = 0, groups = 0, probs = 0, target_el = 0, partial_el = 0, direct = 0;
    long long hist[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // launches by CTA count: <8, <64, <512, <4096, ...
    ~RedStats() {
        if (!getenv("RSC_GEMM_STATS")) return;
        fprintf(stderr, "RSC_GEMM_STATS reduce launches %lld ctas %lld groups %lld probs %lld target_el %lld "
                "partial_el %lld direct %lld\n", launches, ctas, groups, probs, target_el, partial_el, direct);
        fprintf(stderr, "RSC_GEMM_STATS cta hist <8:%lld <64:%lld <512:%lld <4k:%lld <32k:%lld more:%lld\n", hist[0],
                hist[1], hist[2], hist[3], hist[4], hist[5]);
    }
};
RedStats g_rstats;

int launch_reduce(RedArgs &ra, long long ctas, char *tab, long long tab_used, cudaStream_t s) {
    if (ra.count == 0 || ctas <= 0) return 0;
    {
        g_rstats.launches++;
        g_rstats.ctas += ctas;
        g_rstats.groups += ra.count;
        g_rstats.probs += ra.nprob;
        for (int g = 0; g < ra.count; ++g) g_rstats.target_el += (long long)ra.g[g].ext_r * ra.g[g].ext_c * ra.g[g].batch;
        for (int q = 0; q < ra.nprob; ++q) g_rstats.partial_el += (long long)ra.p[q].M * ra.p[q].N;
        int h = 0;
        for (long long c = ctas; c >= 8 && h < 5; c >>= 3) ++h;
        g_rstats.hist[h]++;
        static const bool big = getenv("RSC_GEMM_STATS") != nullptr;
        if (big) {
            long long te = 0, pe = 0, mrow = 0;
            for (int g = 0; g < ra.count; ++g) te += (long long)ra.g[g].ext_r * ra.g[g].ext_c * ra.g[g].batch;
            for (int q = 0; q < ra.nprob; ++q) pe += (long long)ra.p[q].M * ra.p[q].N;
            for (int g = 0; g < ra.count; ++g) mrow = std::max(mrow, (long long)ra.g[g].np);
            if (pe > 20000000)
                fprintf(stderr, "RSC_GEMM_BIG groups %d probs %d maxnp %lld target_el %lld partial_el %lld ctas %lld "
                        "ext %dx%d TR %d CW %d rtab %d ctab %d\n", ra.count, ra.nprob, mrow, te, pe, ctas,
                        ra.g[0].ext_r, ra.g[0].ext_c, ra.g[0].TR, ra.g[0].CW, ra.g[0].rtab != nullptr,
                        ra.g[0].ctab != nullptr);
        }
    }
    static const bool dbg = getenv("RSC_GEMM_DEBUG") != nullptr;
    if (dbg) {  // diagnostics (syncs; not capturable): target overlap between groups
        for (int g = 0; g < ra.count; ++g)
            for (int h = g + 1; h < ra.count; ++h) {
                const RedGroup &G = ra.g[g], &H = ra.g[h];
                const char *lo1 = (const char *)G.C, *hi1 = lo1 + 8 * ((long long)(G.ext_r - 1) * G.ldc + G.ext_c);
                const char *lo2 = (const char *)H.C, *hi2 = lo2 + 8 * ((long long)(H.ext_r - 1) * H.ldc + H.ext_c);
                if (lo1 < hi2 && lo2 < hi1 && G.sC == 0 && H.sC == 0)
                    fprintf(stderr, "RSC_GEMM_DEBUG: groups %d/%d overlap\n", g, h);
            }
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    static const bool no_pdl = getenv("RSC_GEMM_NO_PDL") != nullptr;  // profiling: plain stream order
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.gridDim = dim3((unsigned)ctas);
    cfg.blockDim = dim3(RT);
    cfg.stream = s;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, ordered_reduce_kernel, ra);
    rsc_count_launch();
    return e == cudaSuccess ? 0 : (int)e;
}

// inverse-map tables of a chunk's reduce: depend only on the problems' maps, so they
// are built before the GEMM launch (the reduce then follows the GEMM directly)
int launch_reduce_tables(RedArgs &ra, char *tab, long long tab_used, cudaStream_t s) {
    if (ra.count == 0 || tab_used <= 0) return 0;
    cudaMemsetAsync(tab, 0xff, (size_t)tab_used, s);  // every table entry = -1
    reduce_tables_kernel<<<ra.nprob, RT, 0, s>>>(ra);
    RSC_CHECK_LAUNCH();
    return 0;
}

}  // namespace

// K balancing of one grouped launch (engine.balance_k / split_k_var, restated here
// so the host side of the sweep does not rebuild problem arrays in numpy): every
// accumulating problem (atomic, or beta = 1) whose single-tile k-loop exceeds ~1.5x
// the balanced per-CTA share is cut into K slabs of that share, in place and in
// order (each slab accumulates: the ordered reduction keeps the slab order).
extern "C" int rsc_gemm_grouped_balanced(int transA, int transB, const rsc_gemm_problem *problems, int count,
                                         int ctas, void *stream) {
    if (count < 0 || ctas <= 0) return -4;
    if (count == 0) return 0;
    double tot = 0.0;
    for (int i = 0; i < count; ++i) {
        const rsc_gemm_problem &p = problems[i];
        const double tiles = std::ceil(p.M / 64.0) * std::ceil(p.N / 64.0) * p.batch;
        tot += tiles * std::ceil(p.K / 16.0);
    }
    const long long target = std::max(8LL, (long long)std::ceil(tot / ctas));
    static thread_local std::vector<rsc_gemm_problem> q;
    q.clear();
    bool any = false;
    for (int i = 0; i < count; ++i) {
        const rsc_gemm_problem &p = problems[i];
        const double ks = std::ceil(p.K / 16.0);
        const bool need = (p.atomic == 1 || p.beta == 1.0) && ks > 1.5 * (double)target;
        if (!need) { q.push_back(p); continue; }
        const long long lim = 16 * target, K = p.K;
        const long long nsl = std::max(1LL, (K + lim - 1) / lim);
        if (nsl == 1) { q.push_back(p); continue; }
        any = true;
        for (long long sl = 0; sl < nsl; ++sl) {
            rsc_gemm_problem r = p;
            const long long k0 = sl * lim;
            r.K = (int)std::min(lim, K - k0);
            r.A = transA ? p.A + k0 * p.lda : p.A + k0;
            if (transB) r.B = p.B + k0;
            else if (p.b_rows) r.b_rows = p.b_rows + k0;
            else r.B = p.B + k0 * p.ldb;
            r.atomic = 1;
            r.beta = 1.0;
            q.push_back(r);
        }
    }
    if (!any) return rsc_gemm_grouped(transA, transB, problems, count, stream);
    return rsc_gemm_grouped(transA, transB, q.data(), (int)q.size(), stream);
}

extern "C" int rsc_gemm_set_workspace(void *stream, void *ws_dev, long long bytes, int as_default) {
    if (bytes < 0) return -3;
    std::lock_guard<std::mutex> lk(g_ws_mu);
    if (as_default) {
        g_ws_default = {nullptr, (char *)ws_dev, bytes};
        return 0;
    }
    for (WsEntry &e : g_ws)
        if (e.stream == stream) {
            e.ptr = (char *)ws_dev;
            e.bytes = bytes;
            return 0;
        }
    g_ws.push_back({stream, (char *)ws_dev, bytes});
    return 0;
}

extern "C" int rsc_gemm_grouped(int transA, int transB, const rsc_gemm_problem *problems,
                                int count, void *stream) {
    if (count < 0) return -4;
    if (count == 0) return 0;
    if (!problems) return -3;
    cudaStream_t s = (cudaStream_t)stream;
    static thread_local GemmArgs args;  // ~30 KB; copied into the launch parameter block
    static thread_local std::vector<rsc_gemm_problem> reds;
    static thread_local std::vector<const double *> parts;
    static thread_local std::vector<int> argi, direct;
    static thread_local RedArgs ra;
    static const bool atomic_diag = getenv("RSC_GEMM_ATOMIC") != nullptr;  // A/B diagnostics only
    WsEntry ws{nullptr, nullptr, 0};
    bool ws_looked = false;
    int i = 0;
    while (i < count) {
        args.count = 0;
        reds.clear();
        parts.clear();
        argi.clear();
        long long tiles = 0, used = 0;
        long long max_ext = 0;  // largest target extent (rows + cols) of the chunk's accumulating problems
        bool gather = false;
        while (i < count && args.count < MAXP) {
            const rsc_gemm_problem &p = problems[i];
            if (p.M <= 0 || p.N <= 0 || p.batch <= 0) { ++i; continue; }
            if (transB && p.b_rows) return -3;
            if (p.K < 0) return -3;
            rsc_gemm_problem q = p;
            if (p.atomic && !atomic_diag) {
                if (!ws_looked) { ws = lookup_ws(stream); ws_looked = true; }
                const long long need = (((long long)p.M * p.N * p.batch * 8) + 255) / 256 * 256;
                const long long ext = (long long)(p.ext_r > 0 ? p.ext_r : p.M) + (p.ext_c > 0 ? p.ext_c : p.N);
                // tables of the chunk: sum_g (ext_r + ext_c) np_g <= max ext x problems
                const long long tab2 = (4LL * std::max(max_ext, ext) + 512) * (long long)(reds.size() + 1);
                if (!ws.ptr || need + 4 * ext + 512 > ws.bytes) return -6;
                if (used + need + tab2 > ws.bytes) break;  // close the chunk; the rest follows in order
                max_ext = std::max(max_ext, ext);
                double *part = (double *)(ws.ptr + used);
                used += need;
                reds.push_back(p);
                parts.push_back(part);
                argi.push_back(args.count);
                q.C = part;
                q.ldc = p.N;
                q.strideC = (long long)p.M * p.N;
                q.c_rows = nullptr;
                q.c_cols = nullptr;
                q.atomic = 0;
                q.beta = 0.0;
            }
            ++i;
            const long long tm = (p.M + BM - 1) / BM, tn = (p.N + BN - 1) / BN;
            args.tile_begin[args.count] = tiles;
            args.p[args.count] = q;
            gather |= p.b_rows != nullptr;
            tiles += tm * tn * p.batch;
            args.count++;
        }
        if (args.count == 0) continue;
        args.tile_begin[args.count] = tiles;
        long long rctas = 0, tab_used = 0;
        int rc = 0;
        if (!reds.empty()) {
            rc = plan_reduce(reds, parts, ws.ptr + used, ws.bytes - used, ra, direct, rctas, tab_used);
            if (rc) return rc;
            g_rstats.direct += (long long)direct.size();
            for (int k : direct) {  // sole unmapped writer of its target: accumulate in place
                rsc_gemm_problem &q = args.p[argi[k]];
                const rsc_gemm_problem &p = reds[k];
                q.C = p.C;
                q.ldc = p.ldc;
                q.strideC = p.strideC;
                q.beta = 1.0;
            }
        }
        // longest k-loops first: the hardware dispatches CTAs in index order, so the
        // tiles of long-K problems start in the first wave and the short ones fill in
        // behind them (LPT order); the problems' results do not depend on the order
        // (each writes its own partial or target; the ordered reduce keeps its own
        // problem order)
        static const bool no_lpt = getenv("RSC_GEMM_NO_LPT") != nullptr;
        if (!no_lpt && args.count > 1) {
            static thread_local std::vector<int> ord;
            static thread_local std::vector<rsc_gemm_problem> tmp;
            ord.resize(args.count);
            for (int k = 0; k < args.count; ++k) ord[k] = k;
            std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return args.p[x].K > args.p[y].K; });
            tmp.assign(args.p, args.p + args.count);
            long long tb = 0;
            for (int k = 0; k < args.count; ++k) {
                const rsc_gemm_problem &q = tmp[ord[k]];
                args.p[k] = q;
                args.tile_begin[k] = tb;
                tb += (long long)((q.M + BM - 1) / BM) * ((q.N + BN - 1) / BN) * q.batch;
            }
            args.tile_begin[args.count] = tb;
        }
        if (!reds.empty() && (rc = launch_reduce_tables(ra, ws.ptr + used, tab_used, s))) return rc;
        // the gathered-B loader is its own instantiation: its index prefetch costs the
        // plain kernels ~2.5% (registers), it is only used for launches that gather
        if (!transA && !transB) rc = gather ? launch_chunk<false, false, true>(args, tiles, s)
                                            : launch_chunk<false, false, false>(args, tiles, s);
        else if (!transA && transB) rc = launch_chunk<false, true, false>(args, tiles, s);
        else if (transA && !transB) rc = gather ? launch_chunk<true, false, true>(args, tiles, s)
                                                : launch_chunk<true, false, false>(args, tiles, s);
        else rc = launch_chunk<true, true, false>(args, tiles, s);
        if (rc) return rc;
        if (!reds.empty() && (rc = launch_reduce(ra, rctas, ws.ptr + used, tab_used, s))) return rc;
    }
    return 0;
}
