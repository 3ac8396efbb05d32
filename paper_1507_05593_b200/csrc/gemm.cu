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
    const int *c_cols;
    int M, N;
};

struct RedGroup {
    double *C;            // target block (all problems of the group share it)
    long long sC;         // batch stride of C
    int ldc, ext_r, batch, TR, p0, np;
};

struct RedArgs {
    int count;            // groups
    long long cta_begin[MAXP + 1];
    RedGroup g[MAXP];
    RedProb p[MAXP];
};

constexpr int RT = 256;

__device__ __forceinline__ int lower_bound_dev(const int *a, int n, int x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(a + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(RT) ordered_reduce_kernel(const __grid_constant__ RedArgs a) {
    __shared__ int s_i0[MAXP], s_i1[MAXP];
    const long long cta = blockIdx.x;
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.cta_begin[mid] <= cta) lo = mid; else hi = mid - 1;
    }
    const RedGroup &G = a.g[lo];
    const long long local = cta - a.cta_begin[lo];
    const int nt = (G.ext_r + G.TR - 1) / G.TR;
    const int b = (int)(local / nt);
    const int t0 = (int)(local - (long long)b * nt) * G.TR;
    const int t1 = min(t0 + G.TR, G.ext_r);
    // local row range of every problem inside this band (maps are increasing)
    for (int q = threadIdx.x; q < G.np; q += RT) {
        const RedProb &P = a.p[G.p0 + q];
        int i0, i1;
        if (P.c_rows) {
            i0 = lower_bound_dev(P.c_rows, P.M, t0);
            i1 = i0 + lower_bound_dev(P.c_rows + i0, P.M - i0, t1);
        } else {
            i0 = min(t0, P.M);
            i1 = min(t1, P.M);
        }
        s_i0[q] = i0;
        s_i1[q] = i1;
    }
    __syncthreads();
    double *C = G.C + (long long)b * G.sC;
    for (int q = 0; q < G.np; ++q) {
        const int i0 = s_i0[q], i1 = s_i1[q];
        if (i0 >= i1) continue;  // block-uniform
        const RedProb &P = a.p[G.p0 + q];
        const int n = P.N;
        const double *src = P.P + (long long)b * P.M * n;
        const int cnt = (i1 - i0) * n;
        for (int e = threadIdx.x; e < cnt; e += RT) {
            const int di = e / n;
            const int i = i0 + di, j = e - di * n;
            const int c = P.c_cols ? __ldg(P.c_cols + j) : j;
            if (!P.c_rows) {
                C[(long long)i * G.ldc + c] += src[(long long)i * n + j];
                continue;
            }
            // Row maps are non-decreasing but may repeat: searchsorted maps of
            // interior-block rows outside the target's structure (their products are
            // exact zeros, see plan._build_targets).  The first local row of a run
            // sums the whole run, so no two threads ever update the same element.
            const int r = __ldg(P.c_rows + i);
            if (i > i0 && __ldg(P.c_rows + i - 1) == r) continue;
            double v = src[(long long)i * n + j];
            for (int k = i + 1; k < i1 && __ldg(P.c_rows + k) == r; ++k) v += src[(long long)k * n + j];
            C[(long long)r * G.ldc + c] += v;
        }
        __syncthreads();  // problem q+1 may hit the same elements through other threads
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
// (reds, in launch order).  Groups = distinct (C, strideC, batch) targets, each
// keeping its problems in order.
int launch_reduce(const std::vector<rsc_gemm_problem> &reds, const std::vector<const double *> &parts,
                  cudaStream_t s) {
    static thread_local RedArgs ra;
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
    ra.count = (int)gfirst.size();
    long long ctas = 0;
    int pos = 0;
    for (int g = 0; g < ra.count; ++g) {
        const rsc_gemm_problem &f = reds[gfirst[g]];
        RedGroup &G = ra.g[g];
        G.C = f.C;
        G.sC = f.strideC;
        G.ldc = f.ldc;
        G.batch = f.batch;
        G.p0 = pos;
        int er = 0, ec = 0;
        for (int i = 0; i < n; ++i) {
            if (gid[i] != g) continue;
            const rsc_gemm_problem &p = reds[i];
            if (p.ldc != f.ldc) return -7;
            if ((p.c_rows && p.ext_r <= 0) || (p.c_cols && p.ext_c <= 0)) return -3;
            er = std::max(er, p.ext_r > 0 ? p.ext_r : p.M);
            ec = std::max(ec, p.ext_c > 0 ? p.ext_c : p.N);
            RedProb &rp = ra.p[pos++];
            rp.P = parts[i];
            rp.c_rows = p.c_rows;
            rp.c_cols = p.c_cols;
            rp.M = p.M;
            rp.N = p.N;
        }
        G.np = pos - G.p0;
        G.ext_r = er;
        G.TR = std::max(4, std::min(64, 2048 / std::max(ec, 1)));
        ra.cta_begin[g] = ctas;
        ctas += (long long)((er + G.TR - 1) / G.TR) * G.batch;
    }
    ra.cta_begin[ra.count] = ctas;
    static const bool dbg = getenv("RSC_GEMM_DEBUG") != nullptr;
    if (dbg) {  // diagnostics: target overlap between groups, map monotonicity and range
        cudaStreamSynchronize(s);
        for (int g = 0; g < ra.count; ++g) {
            const RedGroup &G = ra.g[g];
            const char *lo1 = (const char *)G.C;
            const char *hi1 = lo1 + 8 * ((long long)(G.ext_r - 1) * G.ldc + 1);
            for (int h = g + 1; h < ra.count; ++h) {
                const RedGroup &H = ra.g[h];
                const char *lo2 = (const char *)H.C;
                const char *hi2 = lo2 + 8 * ((long long)(H.ext_r - 1) * H.ldc + 1);
                if (lo1 < hi2 && lo2 < hi1)
                    fprintf(stderr, "RSC_GEMM_DEBUG: groups %d/%d overlap (C %p ext %d ld %d / C %p ext %d ld %d)\n",
                            g, h, (void *)G.C, G.ext_r, G.ldc, (void *)H.C, H.ext_r, H.ldc);
            }
            for (int q = G.p0; q < G.p0 + G.np; ++q) {
                const RedProb &P = ra.p[q];
                for (int w = 0; w < 2; ++w) {
                    const int *mp = w ? P.c_cols : P.c_rows;
                    const int len = w ? P.N : P.M;
                    if (!mp) continue;
                    std::vector<int> hv(len);
                    cudaMemcpy(hv.data(), mp, sizeof(int) * len, cudaMemcpyDeviceToHost);
                    for (int t = 0; t < len; ++t) {
                        const bool bad = (t && (w ? hv[t] <= hv[t - 1] : hv[t] < hv[t - 1])) || hv[t] < 0;
                        if (bad) {
                            fprintf(stderr, "RSC_GEMM_DEBUG: group %d prob %d %s map bad at %d: %d (prev %d, ext_r %d)\n",
                                    g, q, w ? "col" : "row", t, hv[t], t ? hv[t - 1] : -1, G.ext_r);
                            break;
                        }
                    }
                }
            }
        }
    }
    if (ctas <= 0) return 0;
    ordered_reduce_kernel<<<(unsigned)ctas, RT, 0, s>>>(ra);
    RSC_CHECK_LAUNCH();
    return 0;
}

}  // namespace

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
    static const bool atomic_diag = getenv("RSC_GEMM_ATOMIC") != nullptr;  // A/B diagnostics only
    WsEntry ws{nullptr, nullptr, 0};
    bool ws_looked = false;
    int i = 0;
    while (i < count) {
        args.count = 0;
        reds.clear();
        parts.clear();
        long long tiles = 0, used = 0;
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
                if (!ws.ptr || need > ws.bytes) return -6;
                if (used + need > ws.bytes) break;  // close the chunk; the rest follows in order
                double *part = (double *)(ws.ptr + used);
                used += need;
                reds.push_back(p);
                parts.push_back(part);
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
        if (!reds.empty() && (rc = launch_reduce(reds, parts, s))) return rc;
    }
    return 0;
}
