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
#include <cooperative_groups.h>
#include <cstdlib>

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

// One launch can mix problems of different modes and scales (a whole phase of a
// level of the apply): mode and alpha are per problem.
//
// mode bit 0: transpose; bit 1: M is lower triangular (read c <= r only);
// bit 2: assign instead of atomic accumulate (transpose 0 only: one segment owns a
// row); bit 3: M is upper triangular (transpose 0 only: read c >= r only); bit 4:
// plain read-modify-write accumulate (the CTA is the only writer: subtree tasks).
//
// transpose 0: a row is owned by a segment of `lpr` lanes (8 / 16 / 32 by width), so
//   narrow panels (the low-rank factors, k ~ 20-60 columns) still keep every lane
//   busy; each lane keeps four independent loads in flight.
// transpose 1: a CTA owns a 64-row slab x up to 256 columns; columns narrower than
//   the CTA are covered by several row subgroups whose partial sums meet in shared
//   memory before one atomic per column.
constexpr int GMAXP = 224;
constexpr int SLAB = 64;     // rows per CTA, transpose 1
constexpr int CTILE = 256;   // columns per CTA, transpose 1

struct GemvProb {
    const double *M;
    const double *x;
    double *y;
    const int *xidx;
    const int *yidx;
    double alpha;
    long long blk_begin;        // first block of this problem (within its launch / phase)
    int rows, cols, ld;
    int mode, lpr;              // lanes per row (transpose 0) / column tile width (transpose 1)
};

struct GemvArgs {
    int count;
    long long total;
    GemvProb p[GMAXP];
};

__device__ __forceinline__ double ldnc(const double *p) { return __ldg(p); }

// one CTA-block of work of problem d (block index lb within the problem)
__device__ __forceinline__ void gemv_block(const GemvProb &d, long long lb, double *xr, double *part) {
    const int mode = d.mode;
    const bool trans = mode & 1, lower = mode & 2, assign = mode & 4, upper = mode & 8;
    const int rows = d.rows, cols = d.cols, ld = d.ld;
    const double alpha = d.alpha;
    const double *M = d.M;
    const double *x = d.x;
    double *y = d.y;
    const int *xi = d.xidx;
    const int *yi = d.yidx;
    const int t = threadIdx.x;
    if (!trans) {
        const int lpr = d.lpr;                    // 8, 16 or 32
        const int seg = t / lpr, sub = t % lpr;   // T / lpr segments per CTA
        const int nseg = T / lpr;
        const int r = (int)lb * nseg + seg;
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (r < rows) {
            const double *Mr = M + (long long)r * ld;
            const int cend = lower ? min(cols, r + 1) : cols;
            int c = (upper ? r : 0) + sub;
            const int step = 4 * lpr;
            if (xi) {
                for (; c + 3 * lpr < cend; c += step) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + lpr), m2 = ldnc(Mr + c + 2 * lpr),
                                 m3 = ldnc(Mr + c + 3 * lpr);
                    s0 += m0 * x[__ldg(xi + c)];
                    s1 += m1 * x[__ldg(xi + c + lpr)];
                    s2 += m2 * x[__ldg(xi + c + 2 * lpr)];
                    s3 += m3 * x[__ldg(xi + c + 3 * lpr)];
                }
                for (; c < cend; c += lpr) s0 += ldnc(Mr + c) * x[__ldg(xi + c)];
            } else {
                for (; c + 3 * lpr < cend; c += step) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + lpr), m2 = ldnc(Mr + c + 2 * lpr),
                                 m3 = ldnc(Mr + c + 3 * lpr);
                    s0 += m0 * x[c];
                    s1 += m1 * x[c + lpr];
                    s2 += m2 * x[c + 2 * lpr];
                    s3 += m3 * x[c + 3 * lpr];
                }
                for (; c < cend; c += lpr) s0 += ldnc(Mr + c) * x[c];
            }
        }
        double s = (s0 + s1) + (s2 + s3);
        for (int o = lpr >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (r < rows && sub == 0) {
            double *dst = y + (yi ? __ldg(yi + r) : r);
            if (assign) *dst = alpha * s;
            else if (mode & 16) *dst += alpha * s;  // exclusive owner (subtree task)
            else atomicAdd(dst, alpha * s);
        }
    } else {
        const int cw = d.lpr;                     // column tile width: 32 .. 256 (power of 2)
        const int ntile = (cols + CTILE - 1) / CTILE;
        const int slab = (int)(lb / ntile), tile = (int)(lb % ntile);
        const int r0 = slab * SLAB, r1 = min(rows, r0 + SLAB);
        for (int r = r0 + t; r < r1; r += T) xr[r - r0] = x[xi ? __ldg(xi + r) : r];
        __syncthreads();
        const int nsub = T / cw;                  // row subgroups
        const int sub = t / cw, c = tile * CTILE + (t % cw);
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (c < cols) {
            int r = r0 + sub;
            if (lower && r < c) r += ((c - r + nsub - 1) / nsub) * nsub;  // rows >= c only
            const double *Mc = M + (long long)r * ld + c;
            const long long st = (long long)nsub * ld;
            for (; r + 3 * nsub < r1; r += 4 * nsub, Mc += 4 * st) {
                const double m0 = ldnc(Mc), m1 = ldnc(Mc + st), m2 = ldnc(Mc + 2 * st), m3 = ldnc(Mc + 3 * st);
                s0 += m0 * xr[r - r0];
                s1 += m1 * xr[r + nsub - r0];
                s2 += m2 * xr[r + 2 * nsub - r0];
                s3 += m3 * xr[r + 3 * nsub - r0];
            }
            for (; r < r1; r += nsub, Mc += st) s0 += ldnc(Mc) * xr[r - r0];
        }
        part[t] = (s0 + s1) + (s2 + s3);
        __syncthreads();
        if (sub == 0 && c < cols) {
            double s = part[t];
            for (int q = 1; q < nsub; ++q) s += part[t + q * cw];
            double *dst = y + (yi ? __ldg(yi + c) : c);
            if (mode & 16) *dst += alpha * s;  // exclusive owner (subtree task)
            else atomicAdd(dst, alpha * s);
        }
    }
}

__device__ __forceinline__ int find_prob(const GemvProb *p, int lo, int hi, long long blk) {
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p[mid].blk_begin <= blk) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(T) gemv_kernel(const __grid_constant__ GemvArgs a) {
    __shared__ double xr[SLAB];
    __shared__ double part[T];
    const long long blk = blockIdx.x;
    const int p = find_prob(a.p, 0, a.count - 1, blk);
    // programmatic dependent launch: the apply's phases are chains of these launches;
    // let the next phase's CTAs be scheduled now, and wait here until the previous
    // phase (whose outputs are this phase's inputs) has completed and flushed
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    gemv_block(a.p[p], blk - a.p[p].blk_begin, xr, part);
}

// The same block for phases with more problems than one parameter block holds: the
// descriptors live in device memory (static after factorization, uploaded once) with a
// block -> problem map, so a whole phase is ONE launch instead of ceil(count / GMAXP)
// back-to-back launches (config[4]'s interior-coupling phases have 4546 problems: 21
// launches of ~19 us, each paying its own ramp and tail).  The descriptor does not
// depend on the previous phase, so it is fetched before the dependency wait.
__global__ void __launch_bounds__(T) gemv_dev_kernel(const GemvProb *__restrict__ P, const int *__restrict__ b2p) {
    __shared__ double xr[SLAB];
    __shared__ double part[T];
    const long long blk = blockIdx.x;
    const GemvProb d = P[__ldg(b2p + blk)];
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    gemv_block(d, blk - d.blk_begin, xr, part);
}

// Subtree tasks: one CTA runs the whole op list of one nested-dissection subtree
// (its interior blocks and small separators, bottom-up for the forward sweep,
// top-down for the backward one).  A unit's update sources all lie in its own
// subtree, so a task depends on nothing outside it; inside, the ops run in order
// with a CTA barrier between them (the CTA owns every row of its subtree, bit 4),
// and only couplings into ancestor rows outside the subtree use FP64 atomics.
// This replaces the ~800 latency-bound level phases of the small units with one
// launch per sweep.  Op descriptors come from rsc_gemv_describe over all tasks'
// ops plus one empty sentinel (block counts = successive blk_begin differences).
__global__ void __launch_bounds__(T) apply_tasks_kernel(const GemvProb *__restrict__ ops,
                                                         const int *__restrict__ task_ptr) {
    __shared__ double xr[SLAB];
    __shared__ double part[T];
    const int o0 = __ldg(task_ptr + blockIdx.x), o1 = __ldg(task_ptr + blockIdx.x + 1);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int o = o0; o < o1; ++o) {
        const GemvProb d = ops[o];
        const long long nb = ops[o + 1].blk_begin - d.blk_begin;  // ops end with a sentinel
        for (long long lb = 0; lb < nb; ++lb) gemv_block(d, lb, xr, part);
        __syncthreads();  // the next op reads this op's results
    }
}

// Cluster tasks: one thread-block cluster of C CTAs per task (the Alg. 4 op list of
// one diagonal block tree, diagblocks.py:192-273).  CTA q of the cluster runs blocks
// q, q + C, ... of each op, and a cluster barrier (release / acquire at cluster
// scope) separates consecutive ops -- a tree's dependent chain of leaf solves and
// couplings costs one cluster barrier per op instead of one dependent kernel launch
// per wave.  Ops whose blocks share outputs across CTAs (column sums) keep their
// atomic epilogue; row-partitioned ops are exclusive per block.
__global__ void __launch_bounds__(T) apply_cluster_tasks_kernel(const GemvProb *__restrict__ ops,
                                                                 const int *__restrict__ task_ptr, int C) {
    __shared__ double xr[SLAB];
    __shared__ double part[T];
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int task = blockIdx.x / C, q = (int)cl.block_rank();
    const int o0 = __ldg(task_ptr + task), o1 = __ldg(task_ptr + task + 1);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int o = o0; o < o1; ++o) {
        const GemvProb d = ops[o];
        const long long nb = ops[o + 1].blk_begin - d.blk_begin;  // ops end with a sentinel
        for (long long lb = q; lb < nb; lb += C) {
            gemv_block(d, lb, xr, part);
            __syncthreads();  // xr / part reuse by the next block
        }
        cl.sync();  // the next op reads this op's results
    }
}

inline int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}

// problem descriptor + its block count
inline long long describe(GemvProb &d, const double *M, int rows, int cols, int ld, const double *x, const int *xi,
                          double *y, const int *yi, int mode, double alpha) {
    d.M = M; d.x = x; d.y = y; d.xidx = xi; d.yidx = yi;
    d.rows = rows; d.cols = cols; d.ld = ld; d.mode = mode; d.alpha = alpha;
    if (mode & 1) {
        d.lpr = cols >= CTILE ? CTILE : (pow2ceil(cols) < 32 ? 32 : pow2ceil(cols));
        return (long long)((rows + SLAB - 1) / SLAB) * ((cols + CTILE - 1) / CTILE);
    }
    d.lpr = cols <= 64 ? 8 : (cols <= 256 ? 16 : 32);  // (lpr 32 from 65 columns measured slower)
    const int nseg = T / d.lpr;
    return (rows + nseg - 1) / nseg;
}

int gemv_launch(int count, const double *const *M, const int *rows, const int *cols, const int *ldm,
                const double *const *x, const int *const *xidx, double *const *y, const int *const *yidx,
                const int *modes, int mode_all, const double *alphas, double alpha_all, cudaStream_t s) {
    static thread_local GemvArgs a;
    int i = 0;
    while (i < count) {
        a.count = 0;
        long long blocks = 0;
        while (i < count && a.count < GMAXP) {
            if (rows[i] <= 0 || cols[i] <= 0) { ++i; continue; }
            GemvProb &d = a.p[a.count++];
            d.blk_begin = blocks;
            blocks += describe(d, M[i], rows[i], cols[i], ldm[i], x[i], xidx ? xidx[i] : nullptr, y[i],
                               yidx ? yidx[i] : nullptr, modes ? modes[i] : mode_all, alphas ? alphas[i] : alpha_all);
            ++i;
        }
        if (a.count == 0) continue;
        a.total = blocks;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        // RSC_APPLY_NO_PDL: plain stream order (profiling only: with PDL a launch's
        // recorded duration includes its wait for the previous phase)
        static const bool no_pdl = getenv("RSC_APPLY_NO_PDL") != nullptr;
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
        cfg.gridDim = dim3((unsigned)blocks);
        cfg.blockDim = dim3(T);
        cfg.stream = s;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, gemv_kernel, a);
        rsc_count_launch();
        if (e != cudaSuccess) return (int)e;
    }
    return 0;
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
    return gemv_launch(count, M, rows, cols, ldm, x, xidx, y, yidx, nullptr, mode, nullptr, alpha,
                       (cudaStream_t)stream);
}

extern "C" int rsc_gemv_desc_bytes(void) { return (int)sizeof(GemvProb); }

extern "C" int rsc_gemv_describe(int count, const double *const *M, const int *rows, const int *cols,
                                 const int *ldm, const double *const *x, const int *const *xidx,
                                 double *const *y, const int *const *yidx, const int *modes,
                                 const double *alphas, void *desc, long long *blocks) {
    if (count < 0) return -1;
    if (count > 0 && (!M || !rows || !cols || !ldm || !x || !y || !modes || !alphas || !desc || !blocks)) return -2;
    GemvProb *d = static_cast<GemvProb *>(desc);
    long long total = 0;
    for (int i = 0; i < count; ++i) {
        d[i] = GemvProb{};
        d[i].blk_begin = total;
        if (rows[i] <= 0 || cols[i] <= 0) { blocks[i] = 0; continue; }
        blocks[i] = describe(d[i], M[i], rows[i], cols[i], ldm[i], x[i], xidx ? xidx[i] : nullptr, y[i],
                             yidx ? yidx[i] : nullptr, modes[i], alphas[i]);
        d[i].blk_begin = total;
        total += blocks[i];
    }
    return 0;
}

extern "C" int rsc_gemv_multi_dev(const void *desc, const int *blk2prob, long long total_blocks, void *stream) {
    if (total_blocks < 0) return -1;
    if (total_blocks == 0) return 0;
    if (!desc || !blk2prob || total_blocks > 0x7fffffffLL) return -2;
    static const bool no_pdl = getenv("RSC_APPLY_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.gridDim = dim3((unsigned)total_blocks);
    cfg.blockDim = dim3(T);
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, gemv_dev_kernel, static_cast<const GemvProb *>(desc), blk2prob);
    rsc_count_launch();
    return e == cudaSuccess ? 0 : (int)e;
}

extern "C" int rsc_apply_tasks(const void *ops, const int *task_ptr_dev, int ntasks, void *stream) {
    if (ntasks < 0) return -3;
    if (ntasks == 0) return 0;
    if (!ops || !task_ptr_dev) return -1;
    static const bool no_pdl = getenv("RSC_APPLY_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.gridDim = dim3((unsigned)ntasks);
    cfg.blockDim = dim3(T);
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, apply_tasks_kernel, static_cast<const GemvProb *>(ops),
                                             task_ptr_dev);
    rsc_count_launch();
    return e == cudaSuccess ? 0 : (int)e;
}

extern "C" int rsc_apply_cluster_tasks(const void *ops, const int *task_ptr_dev, int ntasks, int C, void *stream) {
    if (ntasks < 0 || C < 1 || C > 8) return -3;
    if (ntasks == 0) return 0;
    if (!ops || !task_ptr_dev) return -1;
    static const bool no_pdl = getenv("RSC_APPLY_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = no_pdl ? 0 : 1;
    cfg.gridDim = dim3((unsigned)ntasks * C);
    cfg.blockDim = dim3(T);
    cfg.stream = (cudaStream_t)stream;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, apply_cluster_tasks_kernel, static_cast<const GemvProb *>(ops),
                                             task_ptr_dev, C);
    rsc_count_launch();
    return e == cudaSuccess ? 0 : (int)e;
}

extern "C" int rsc_gemv_multi(int count, const double *const *M, const int *rows, const int *cols,
                              const int *ldm, const double *const *x, const int *const *xidx,
                              double *const *y, const int *const *yidx, const int *modes,
                              const double *alphas, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!M || !rows || !cols || !ldm || !x || !y || !modes || !alphas) return -2;
    return gemv_launch(count, M, rows, cols, ldm, x, xidx, y, yidx, modes, 0, alphas, 0.0, (cudaStream_t)stream);
}


// ---------------------------------------------------------------------------
// Batched identity / transpose for the apply program's explicit inverses (one
// launch each instead of two torch kernels per triangle): refresh after every
// refactorization re-derives Linv = L^{-1} (TRSM against I) and LinvT.
namespace {
constexpr int BMAX = 1024;
struct SqArgs {
    int count;
    const double *src[BMAX];
    double *dst[BMAX];
    int n[BMAX], lds[BMAX], ldd[BMAX];
};

__global__ void __launch_bounds__(256) eye_kernel(const __grid_constant__ SqArgs a) {
    const int b = blockIdx.x;
    const int n = a.n[b], ld = a.ldd[b];
    double *D = a.dst[b];
    for (long long e = threadIdx.x; e < (long long)n * n; e += 256) {
        const int i = (int)(e / n), j = (int)(e - (long long)i * n);
        D[(long long)i * ld + j] = (i == j) ? 1.0 : 0.0;
    }
}

// dst = src^T through 32x32 shared-memory tiles (coalesced both ways)
__global__ void __launch_bounds__(256) transpose_kernel(const __grid_constant__ SqArgs a) {
    __shared__ double tile[32][33];
    const int b = blockIdx.x;
    const int n = a.n[b], lds = a.lds[b], ldd = a.ldd[b];
    const double *S = a.src[b];
    double *D = a.dst[b];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int i0 = 0; i0 < n; i0 += 32)
        for (int j0 = 0; j0 < n; j0 += 32) {
            for (int q = ty; q < 32; q += 8) {
                const int i = i0 + q, j = j0 + tx;
                tile[q][tx] = (i < n && j < n) ? S[(long long)i * lds + j] : 0.0;
            }
            __syncthreads();
            for (int q = ty; q < 32; q += 8) {
                const int i = j0 + q, j = i0 + tx;  // D[i][j] = S[j][i]
                if (i < n && j < n) D[(long long)i * ldd + j] = tile[tx][q];
            }
            __syncthreads();
        }
}

int sq_launch(int mode, int count, const double *const *src, double *const *dst, const int *n, const int *lds,
              const int *ldd, cudaStream_t s) {
    static thread_local SqArgs a;
    for (int c0 = 0; c0 < count; c0 += BMAX) {
        const int cnt = count - c0 < BMAX ? count - c0 : BMAX;
        a.count = cnt;
        for (int i = 0; i < cnt; ++i) {
            a.src[i] = src ? src[c0 + i] : nullptr;
            a.dst[i] = dst[c0 + i];
            a.n[i] = n[c0 + i];
            a.lds[i] = lds ? lds[c0 + i] : 0;
            a.ldd[i] = ldd[c0 + i];
        }
        if (mode == 0) eye_kernel<<<cnt, 256, 0, s>>>(a);
        else transpose_kernel<<<cnt, 256, 0, s>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}
}  // namespace

extern "C" int rsc_identity_batched(int count, double *const *dst, const int *n, const int *ldd, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!dst || !n || !ldd) return -2;
    return sq_launch(0, count, nullptr, dst, n, nullptr, ldd, (cudaStream_t)stream);
}

extern "C" int rsc_transpose_batched(int count, const double *const *src, double *const *dst, const int *n,
                                     const int *lds, const int *ldd, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!src || !dst || !n || !lds || !ldd) return -2;
    return sq_launch(1, count, src, dst, n, lds, ldd, (cudaStream_t)stream);
}
