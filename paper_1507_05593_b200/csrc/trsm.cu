// Fused right-side triangular solve  X = B L^{-T}  for batches of panels
// (reference kernels.py:42-64 tri_solve, used as L_O = A(R_j, C_j) L_D^{-T} at
// factor.py:414,633 and for every off-diagonal panel of a supernode).
//
// One CTA owns a 64-row strip of one panel B (m x n, n <= 320) and keeps the whole
// strip resident in shared memory while it runs the left-looking block recurrence
//
//     X_j = (B_j - sum_{i<j} X_i L_ji^T) Dinv_j^T          (64-column blocks j)
//
// with Dinv_j = L_jj^{-1} from rsc_potrf_batched.  The operand blocks L_ji / Dinv_j
// (64 x 64, shared by all strips of a panel, L2-resident) stream through a 2-stage
// cp.async pipeline that runs continuously across the phases of the recurrence; the
// strip itself is loaded one column block ahead of its use and each finished X_j is
// stored while later blocks compute, so B is read from HBM once and X written once,
// overlapped with the DMMA work, and a whole batch is one launch.
//
// 128 threads = 2 x 2 warps of 32 x 32 (4 x 4 DMMA.8x8x4 fragments per warp, 16
// independent accumulators: DMMA.8x8x4 issues every 16 cycles per SM sub-partition
// with ~26 cycles latency (tools/micro/dmma_micro.cu), so one warp per sub-partition
// keeps the FP64 pipe fed and the per-chunk control work stays small).
#include <vector>

#include "common.cuh"

#define RSC_TRSM_TOO_WIDE (-1000)

namespace {

#ifndef RSC_TRSM_ROWS
#define RSC_TRSM_ROWS 32
#endif
constexpr int SM_ROWS = RSC_TRSM_ROWS;  // strip height (32: two CTAs per SM)
constexpr int TNT = 128;
#ifndef RSC_TRSM_STAGES
#define RSC_TRSM_STAGES 2
#endif
constexpr int RST = RSC_TRSM_STAGES;          // operand pipeline depth (right solve)
constexpr int KB = RST == 3 ? 16 : (SM_ROWS == 32 ? 32 : 64);  // k extent of one chunk
constexpr int KPB = 64 / KB;                 // chunks per 64-wide operand block
constexpr int BPAD = KB + 4;  // [n][k] row stride of a staged operand block
constexpr int WTM = SM_ROWS / 2;             // warp tile rows (2 x 2 warps)
constexpr int FI = WTM / 8;
constexpr int TMAXN = 320;    // strip + 2 operand stages fit in shared memory
constexpr int MAXT = 520;

struct TrsmArgs {
    int count;
    int lds;                       // strip row stride (doubles)
    long long tile_begin[MAXT + 1];
    const double *L[MAXT];
    const double *Dinv[MAXT];
    const double *Bsrc[MAXT];
    double *B[MAXT];
    int n[MAXT], m[MAXT], ldl[MAXT], ldb[MAXT];
};

__device__ __forceinline__ void cp_async_16(void *smem, const double *gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
                 "r"(valid ? 16 : 0));
}

// stage a 64 (rows) x KB (k) operand slice  dst[r][k] = src[r * ld + k]  (r < rows,
// k < kmax; zero elsewhere); 16-byte copies when the rows are 16-byte aligned
__device__ __forceinline__ void load_opblock(double *dst, const double *src, long long ld, int rows, int kmax,
                                             bool vec) {
    const int t = threadIdx.x;
    if (vec) {
#pragma unroll
        for (int i = 0; i < 64 * KB / 2 / TNT; ++i) {
            const int e = t + TNT * i;
            const int r = e / (KB / 2), k = 2 * (e % (KB / 2));
            const bool v = r < rows && k < kmax;  // kmax is even on this path
            cp_async_16(&dst[r * BPAD + k], v ? src + (long long)r * ld + k : src, v);
        }
    } else {
#pragma unroll 8
        for (int i = 0; i < 64 * KB / TNT; ++i) {
            const int e = t + TNT * i;
            const int r = e / KB, k = e % KB;
            const bool v = r < rows && k < kmax;
            cp_async_8(&dst[r * BPAD + k], v ? src + (long long)r * ld + k : src, v);
        }
    }
}

__global__ void __launch_bounds__(TNT) trsm_right_kernel(const __grid_constant__ TrsmArgs a) {
    extern __shared__ __align__(16) double tsm[];
    const int lds = a.lds;
    double *S = tsm;
    double *sB = tsm + SM_ROWS * lds;

    const long long tile = blockIdx.x;
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.tile_begin[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int r0 = (int)(tile - a.tile_begin[b]) * SM_ROWS;
    const int n = a.n[b], m = a.m[b], ldb = a.ldb[b];
    const long long ldl = a.ldl[b];
    const int nblk = (n + 63) >> 6;
    const int rows = m - r0 < SM_ROWS ? m - r0 : SM_ROWS;
    const double *Bs = a.Bsrc[b] + (long long)r0 * ldb;
    double *Bd = a.B[b] + (long long)r0 * ldb;
    const double *L = a.L[b];
    const double *Dv = a.Dinv[b];

    const bool vec = ((ldb | n) & 1) == 0 && ((reinterpret_cast<uintptr_t>(Bs) & 15) == 0) &&
                     ((reinterpret_cast<uintptr_t>(Bd) & 15) == 0);
    const bool vecL = ((ldl | n) & 1) == 0 && ((reinterpret_cast<uintptr_t>(L) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(Dv) & 15) == 0);

    auto load_block = [&](int jb) {  // strip columns [64 jb, 64 jb + 64)
        const int c0 = jb * 64;
        if (vec) {
            for (int e = threadIdx.x; e < SM_ROWS * 32; e += TNT) {
                const int r = e >> 5, c = c0 + 2 * (e & 31);
                const bool v = r < rows && c < n;
                cp_async_16(&S[r * lds + c], v ? Bs + (long long)r * ldb + c : Bs, v);
            }
        } else {
            for (int e = threadIdx.x; e < SM_ROWS * 64; e += TNT) {
                const int r = e >> 6, c = c0 + (e & 63);
                const bool v = r < rows && c < n;
                cp_async_8(&S[r * lds + c], v ? Bs + (long long)r * ldb + c : Bs, v);
            }
        }
    };
    auto store_block = [&](int jb) {
        const int c0 = jb * 64;
        const int w = n - c0 < 64 ? n - c0 : 64;
        if (vec) {
            for (int e = threadIdx.x; e < rows * 32; e += TNT) {
                const int r = e >> 5, c = 2 * (e & 31);
                if (c < w)
                    *reinterpret_cast<double2 *>(Bd + (long long)r * ldb + c0 + c) =
                        *reinterpret_cast<const double2 *>(&S[r * lds + c0 + c]);
            }
        } else {
            for (int e = threadIdx.x; e < rows * 64; e += TNT) {
                const int r = e >> 6, c = e & 63;
                if (c < w) Bd[(long long)r * ldb + c0 + c] = S[r * lds + c0 + c];
            }
        }
    };

    // chunk sequence: block jb has KPB*jb update chunks (operand L_{jb, k}, k < 64 jb)
    // and KPB diagonal chunks (Dinv_jb); (pj, pi) walks it for the prefetcher
    int pj = 0, pi = 0;
    auto prefetch = [&](int stage) {
        if (pj < nblk) {
            const int j0 = pj * 64;
            const int w = n - j0 < 64 ? n - j0 : 64;
            double *dst = sB + stage * 64 * BPAD;
            const int nu = KPB * pj;
            if (pi < nu) load_opblock(dst, L + (long long)j0 * ldl + pi * KB, ldl, w, KB, vecL);
            else {
                const int k0 = (pi - nu) * KB;
                load_opblock(dst, Dv + (long long)j0 * 64 + k0, 64, w, w - k0, vecL && (w & 1) == 0);
            }
            // strip block pj+1 rides with the first chunk of block pj (pj >= 1); it is
            // first touched by block pj+1's update epilogue
            if (pi == 0 && pj >= 1 && pj + 1 < nblk) load_block(pj + 1);
            if (++pi >= KPB * (pj + 1)) {
                ++pj;
                pi = 0;
            }
        }
        cp_async_commit();
    };

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int wm = (warp >> 1) * WTM, wn = (warp & 1) * 32;

    load_block(0);
    if (nblk > 1) load_block(1);
    cp_async_commit();
#pragma unroll
    for (int st = 0; st < RST - 1; ++st) prefetch(st);

    double acc[FI][4][2];
#pragma unroll
    for (int i = 0; i < FI; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int cj = 0, ci = 0, stage = 0;  // chunk being computed
    while (cj < nblk) {
        cp_async_wait<RST - 2>();
        __syncthreads();  // chunk landed; the stage to refill is free; S writes are visible
        prefetch((stage + RST - 1) % RST);
        if (ci == 0 && cj >= 1) store_block(cj - 1);  // X_{cj-1} is final
        const int nu = KPB * cj;
        const bool diag = ci >= nu;
        const int j0 = cj * 64;
        const double *b_s = sB + stage * 64 * BPAD;
        const double *a_s = S + (diag ? j0 + (ci - nu) * KB : ci * KB);
#pragma unroll 4
        for (int kk = 0; kk < KB; kk += 4) {
            double af[FI], bf[4];
#pragma unroll
            for (int i = 0; i < FI; ++i) af[i] = a_s[(wm + i * 8 + g) * lds + kk + q];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = b_s[(wn + j * 8 + g) * BPAD + kk + q];
#pragma unroll
            for (int i = 0; i < FI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        if (ci + 1 == nu || ci + 1 == nu + KPB) {
            // last update chunk: B_j -= sum_{i<j} X_i L_ji^T (no warp reads block j yet);
            // last diagonal chunk: X_j = B_j Dinv_j^T once every warp is done reading B_j
            if (diag) __syncthreads();
#pragma unroll
            for (int i = 0; i < FI; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double &sv = S[(wm + i * 8 + g) * lds + j0 + wn + j * 8 + 2 * q + e];
                        sv = diag ? acc[i][j][e] : -acc[i][j][e] + sv;
                        acc[i][j][e] = 0.0;
                    }
        }
        stage = (stage + 1) % RST;
        if (++ci >= KPB * (cj + 1)) {
            ++cj;
            ci = 0;
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    store_block(nblk - 1);
}

// ---------------------------------------------------------------------------
// Left-side solves  X = L^{-1} B  (TRANS = 0)  and  X = L^{-T} B  (TRANS = 1)
// (tri_solve(side="left"), kernels.py:42-64: every diagonal solve of the sweep --
// Alg. 2's G1 = L_D^{-T} G, the tree leaves of Alg. 4, interior blocks).  One CTA
// owns a 32-column strip of B (all n <= 320 rows) in shared memory and runs the
// row-block recurrence
//     TRANS 0:  X_j = Dinv_j   (B_j - sum_{i<j} L_ji   X_i)      j = 0, 1, ...
//     TRANS 1:  X_j = Dinv_j^T (B_j - sum_{i>j} L_ij^T X_i)      j = nb-1, ...
// as DMMA products whose A operand (a 64x32 slice of L / Dinv, or its transpose)
// streams through a 2-stage cp.async pipeline and whose B operand is the resident
// strip.  One launch replaces the per-block chain of grouped GEMM launches.
constexpr int LCW = 32;            // strip width (columns of B)
constexpr int LKB = 32;            // k extent of one operand chunk
constexpr int LPK = LKB + 4;       // [m][k] row stride
constexpr int LPM = 64 + 4;        // [k][m] row stride (transposed staging)
constexpr int LSTAGE = 64 * LPK;   // doubles per stage (covers 64 x 36 and 32 x 68)

struct TrsmLArgs {
    int count;
    int lds;                       // strip row stride (doubles)
    long long tile_begin[MAXT + 1];
    const double *L[MAXT];
    const double *Dinv[MAXT];
    double *B[MAXT];
    int n[MAXT], m[MAXT], ldl[MAXT], ldb[MAXT];
};

// stage the operand chunk A[mm][kk] (mm < 64, kk < 32): TRANS 0 reads src[mm*ld + kk]
// (row-major slice), TRANS 1 reads src[kk*ld + mm] (the transposed slice); zero fill
// outside rows x kmax
template <int TRANS>
__device__ __forceinline__ void load_lop(double *dst, const double *src, long long ld, int rows, int kmax) {
    const int t = threadIdx.x;
    if (TRANS == 0) {
#pragma unroll
        for (int i = 0; i < 64 * LKB / TNT; ++i) {
            const int e = t + TNT * i;
            const int mm = e / LKB, kk = e % LKB;
            const bool v = mm < rows && kk < kmax;
            cp_async_8(&dst[mm * LPK + kk], v ? src + (long long)mm * ld + kk : src, v);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 64 * LKB / TNT; ++i) {
            const int e = t + TNT * i;
            const int kk = e / 64, mm = e % 64;
            const bool v = mm < rows && kk < kmax;
            cp_async_8(&dst[kk * LPM + mm], v ? src + (long long)kk * ld + mm : src, v);
        }
    }
}

template <int TRANS>
__global__ void __launch_bounds__(TNT) trsm_left_kernel(const __grid_constant__ TrsmLArgs a) {
    extern __shared__ __align__(16) double lsm[];
    const int lds = a.lds;
    const long long tile = blockIdx.x;
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.tile_begin[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const int b = lo;
    const int c0 = (int)(tile - a.tile_begin[b]) * LCW;
    const int n = a.n[b], m = a.m[b], ldb = a.ldb[b];
    const long long ldl = a.ldl[b];
    const int nblk = (n + 63) >> 6, npad = nblk * 64;
    const int cols = m - c0 < LCW ? m - c0 : LCW;
    double *S = lsm;                       // npad x lds
    double *sA = lsm + (size_t)npad * lds; // 2 stages
    double *Bp = a.B[b] + c0;
    const double *L = a.L[b];
    const double *Dv = a.Dinv[b];

    for (int e = threadIdx.x; e < npad * LCW; e += TNT) {
        const int r = e / LCW, c = e % LCW;
        const bool v = r < n && c < cols;
        cp_async_8(&S[r * lds + c], v ? Bp + (long long)r * ldb + c : Bp, v);
    }
    cp_async_commit();

    // chunk walk: block position p (row block j = p or nblk-1-p) has `nu` update
    // blocks (2 chunks each) then the diagonal block (2 chunks)
    auto jof = [&](int p) { return TRANS ? nblk - 1 - p : p; };
    auto nupd = [&](int p) { return p; };  // i < j (TRANS 0) or i > j (TRANS 1): p of them
    auto ublk = [&](int p, int u) { return TRANS ? nblk - 1 - u : u; };  // u-th update source block
    int pp = 0, pc = 0;  // prefetch position
    auto prefetch = [&](int stage) {
        if (pp < nblk) {
            const int j = jof(pp), j0 = j * 64;
            const int w = n - j0 < 64 ? n - j0 : 64;
            double *dst = sA + stage * LSTAGE;
            const int nu = nupd(pp);
            if (pc < 2 * nu) {
                const int i0 = ublk(pp, pc >> 1) * 64, k0 = (pc & 1) * LKB;
                const int kw = n - i0 - k0;
                if (TRANS == 0) load_lop<0>(dst, L + (long long)j0 * ldl + i0 + k0, ldl, w, kw);
                else load_lop<1>(dst, L + (long long)(i0 + k0) * ldl + j0, ldl, w, kw);
            } else {
                const int k0 = (pc - 2 * nu) * LKB;
                if (TRANS == 0) load_lop<0>(dst, Dv + (long long)j0 * 64 + k0, 64, w, w - k0);
                else load_lop<1>(dst, Dv + (long long)(j0 + k0) * 64, 64, w, w - k0);
            }
            if (++pc >= 2 * nu + 2) {
                ++pp;
                pc = 0;
            }
        }
        cp_async_commit();
    };

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, q = lane & 3;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 16;
    prefetch(0);
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    int cp = 0, cc = 0, stage = 0;
    while (cp < nblk) {
        cp_async_wait<0>();
        __syncthreads();
        prefetch(stage ^ 1);
        const int j = jof(cp), j0 = j * 64;
        const int nu = nupd(cp);
        const bool diag = cc >= 2 * nu;
        // B operand rows of this chunk in the strip
        const int br = diag ? j0 + (cc - 2 * nu) * LKB : ublk(cp, cc >> 1) * 64 + (cc & 1) * LKB;
        const double *a_s = sA + stage * LSTAGE;
#pragma unroll 4
        for (int kk = 0; kk < LKB; kk += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                af[i] = TRANS ? a_s[(kk + q) * LPM + wm + i * 8 + g] : a_s[(wm + i * 8 + g) * LPK + kk + q];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) bf[jj] = S[(br + kk + q) * lds + wn + jj * 8 + g];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj) dmma_8x8x4(acc[i][jj][0], acc[i][jj][1], af[i], bf[jj]);
        }
        if (cc + 1 == 2 * nu || cc + 1 == 2 * nu + 2) {
            if (diag) __syncthreads();  // every warp is done reading block j's rows
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int jj = 0; jj < 2; ++jj)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        double &sv = S[(j0 + wm + i * 8 + g) * lds + wn + jj * 8 + 2 * q + e];
                        sv = diag ? acc[i][jj][e] : -acc[i][jj][e] + sv;
                        acc[i][jj][e] = 0.0;
                    }
        }
        stage ^= 1;
        if (++cc >= 2 * nu + 2) {
            ++cp;
            cc = 0;
        }
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int e = threadIdx.x; e < n * LCW; e += TNT) {
        const int r = e / LCW, c = e % LCW;
        if (c < cols) Bp[(long long)r * ldb + c] = S[r * lds + c];
    }
}

}  // namespace

// Right-side X = B L^{-T} for panels with n <= 320 (returns RSC_TRSM_TOO_WIDE if some
// n is larger: the caller then uses the blocked path).  Bsrc may be NULL (in place)
// or a separate source array of the same shapes/ld as B.
int rsc_trsm_right_fused(int count, const double *const *L, const int *n, const int *ldl,
                         const double *const *Dinv, const double *const *Bsrc, double *const *B,
                         const int *m, const int *ldb, cudaStream_t s) {
    int maxn = 0;
    for (int i = 0; i < count; ++i) maxn = n[i] > maxn ? n[i] : maxn;
    if (maxn > TMAXN) return RSC_TRSM_TOO_WIDE;
    static thread_local TrsmArgs a;
    // the dynamic shared-memory cap is raised once, to the widest panel, so no
    // attribute call happens later (e.g. inside a CUDA-graph capture)
    static bool attr = false;
    if (!attr) {
        const int maxbytes = (SM_ROWS * (TMAXN + 4) + RST * 64 * BPAD) * (int)sizeof(double);
        cudaFuncSetAttribute(trsm_right_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, maxbytes);
        attr = true;
    }
    for (int c0 = 0; c0 < count;) {
        a.count = 0;
        long long tiles = 0;
        int mx = 0;
        for (; c0 < count && a.count < MAXT; ++c0) {
            if (m[c0] <= 0 || n[c0] <= 0) continue;
            const int c = a.count++;
            a.L[c] = L[c0];
            a.Dinv[c] = Dinv[c0];
            a.Bsrc[c] = Bsrc ? Bsrc[c0] : B[c0];
            a.B[c] = B[c0];
            a.n[c] = n[c0];
            a.m[c] = m[c0];
            a.ldl[c] = ldl[c0];
            a.ldb[c] = ldb[c0];
            a.tile_begin[c] = tiles;
            tiles += (m[c0] + SM_ROWS - 1) / SM_ROWS;
            mx = n[c0] > mx ? n[c0] : mx;
        }
        if (!a.count) continue;
        a.tile_begin[a.count] = tiles;
        a.lds = ((mx + 63) & ~63) + 4;
        const int bytes = (SM_ROWS * a.lds + RST * 64 * BPAD) * (int)sizeof(double);
        trsm_right_kernel<<<(unsigned)tiles, TNT, bytes, s>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

// Left-side X = L^{-1} B / L^{-T} B in place for n <= 320 (else RSC_TRSM_TOO_WIDE).
int rsc_trsm_left_fused(int trans, int count, const double *const *L, const int *n, const int *ldl,
                        const double *const *Dinv, double *const *B, const int *m, const int *ldb,
                        cudaStream_t s) {
    int maxn = 0;
    for (int i = 0; i < count; ++i) maxn = n[i] > maxn ? n[i] : maxn;
    if (maxn > TMAXN) return RSC_TRSM_TOO_WIDE;
    static thread_local TrsmLArgs a;
    static bool attr = false;
    const int maxbytes = (((TMAXN + 63) & ~63) * (LCW + 4) + 2 * LSTAGE) * (int)sizeof(double);
    if (!attr) {
        cudaFuncSetAttribute(trsm_left_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxbytes);
        cudaFuncSetAttribute(trsm_left_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, maxbytes);
        attr = true;
    }
    for (int c0 = 0; c0 < count;) {
        a.count = 0;
        long long tiles = 0;
        int mx = 0;
        for (; c0 < count && a.count < MAXT; ++c0) {
            if (m[c0] <= 0 || n[c0] <= 0) continue;
            const int c = a.count++;
            a.L[c] = L[c0];
            a.Dinv[c] = Dinv[c0];
            a.B[c] = B[c0];
            a.n[c] = n[c0];
            a.m[c] = m[c0];
            a.ldl[c] = ldl[c0];
            a.ldb[c] = ldb[c0];
            a.tile_begin[c] = tiles;
            tiles += (m[c0] + LCW - 1) / LCW;
            mx = n[c0] > mx ? n[c0] : mx;
        }
        if (!a.count) continue;
        a.tile_begin[a.count] = tiles;
        a.lds = LCW + 4;
        const int bytes = (((mx + 63) & ~63) * a.lds + 2 * LSTAGE) * (int)sizeof(double);
        if (trans) trsm_left_kernel<1><<<(unsigned)tiles, TNT, bytes, s>>>(a);
        else trsm_left_kernel<0><<<(unsigned)tiles, TNT, bytes, s>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}
