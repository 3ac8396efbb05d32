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
#ifndef GEMV_RPB
#define GEMV_RPB 4
#endif
#ifndef GEMV_MINB
#define GEMV_MINB 5  // CTAs per SM of the phase kernels (51 registers: a few spilled words; measured 6% faster
                     // applies than 4 CTAs at 62 registers -- the phases are bound by loads in flight)
#endif
constexpr int RPB = GEMV_RPB;  // rows per segment, transpose 0, full aligned rows
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
    int nblk, grp;              // dataflow program: blocks of the op, blocks per item
};

struct GemvArgs {
    int count;
    long long total;
    GemvProb p[GMAXP];
};

__device__ __forceinline__ double ldnc(const double *p) { return __ldg(p); }

// x reads: through L1 (read-only path) for phases separated by kernel boundaries;
// L2 only (ld.global.cg) inside the dataflow kernel, where x was written by other
// CTAs of the same launch
template <bool CG>
__device__ __forceinline__ double ldx(const double *p) {
    if constexpr (CG) return __ldcg(p);
    else return *p;
}

// one CTA-block of work of problem d (block index lb within the problem)
template <bool CG = false>
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
        if ((mode & 32) && !lower && !upper) {
            // full rows, 16-byte aligned: a segment owns RPB consecutive rows and walks
            // them together (one x pair feeds RPB double2 loads), so a CTA moves RPB times
            // the bytes of the one-row path per launch slot and keeps 2 RPB loads per
            // lane in flight
            const int rb = ((int)lb * nseg + seg) * RPB;
            double acc[RPB];
#pragma unroll
            for (int q = 0; q < RPB; ++q) acc[q] = 0.0;
            if (rb < rows) {
                const int nr = min(RPB, rows - rb);
                const double2 *M2[RPB];
#pragma unroll
                for (int q = 0; q < RPB; ++q)
                    M2[q] = reinterpret_cast<const double2 *>(M + (long long)(rb + (q < nr ? q : 0)) * ld);
                const int pend = cols >> 1;
#pragma unroll 2
                for (int p = sub; p < pend; p += lpr) {
                    const int c = 2 * p;
                    const double x0 = ldx<CG>(x + (xi ? __ldg(xi + c) : c));
                    const double x1 = ldx<CG>(x + (xi ? __ldg(xi + c + 1) : c + 1));
#pragma unroll
                    for (int q = 0; q < RPB; ++q) {
                        const double2 mv = __ldg(M2[q] + p);
                        acc[q] = fma(mv.y, x1, fma(mv.x, x0, acc[q]));
                    }
                }
                if ((cols & 1) && sub == lpr - 1) {
                    const int c = cols - 1;
                    const double xv = ldx<CG>(x + (xi ? __ldg(xi + c) : c));
#pragma unroll
                    for (int q = 0; q < RPB; ++q)
                        acc[q] = fma(ldnc(reinterpret_cast<const double *>(M2[q]) + c), xv, acc[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < RPB; ++q)
                for (int o = lpr >> 1; o > 0; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
            if (rb < rows && sub == 0) {
                const int nr = min(RPB, rows - rb);
#pragma unroll
                for (int q = 0; q < RPB; ++q) {
                    if (q >= nr) break;
                    double *dst = y + (yi ? __ldg(yi + rb + q) : rb + q);
                    if (assign) *dst = alpha * acc[q];
                    else if (mode & 16) *dst += alpha * acc[q];
                    else atomicAdd(dst, alpha * acc[q]);
                }
            }
            return;
        }
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        if (r < rows && (mode & 32)) {
            // rows 16-byte aligned: double2 loads of column pairs (2p, 2p+1), four pairs in
            // flight per lane; a lone first / last column is done by one lane
            const double *Mr = M + (long long)r * ld;
            const double2 *M2 = reinterpret_cast<const double2 *>(Mr);
            const int cend = lower ? min(cols, r + 1) : cols;
            int cb = upper ? r : 0;
            if ((cb & 1) && cb < cend) {
                if (sub == 0) s0 += ldnc(Mr + cb) * ldx<CG>(x + (xi ? __ldg(xi + cb) : cb));
                ++cb;
            }
            const int pend = cend >> 1;
            if ((cend & 1) && cend - 1 >= cb && sub == lpr - 1)
                s1 += ldnc(Mr + cend - 1) * ldx<CG>(x + (xi ? __ldg(xi + cend - 1) : cend - 1));
            int p = (cb >> 1) + sub;
            if (xi) {
                for (; p + 3 * lpr < pend; p += 4 * lpr) {
                    const double2 m0 = __ldg(M2 + p), m1 = __ldg(M2 + p + lpr), m2 = __ldg(M2 + p + 2 * lpr),
                                  m3 = __ldg(M2 + p + 3 * lpr);
                    const int c0 = 2 * p, c1 = 2 * (p + lpr), c2 = 2 * (p + 2 * lpr), c3 = 2 * (p + 3 * lpr);
                    s0 += m0.x * ldx<CG>(x + __ldg(xi + c0)) + m0.y * ldx<CG>(x + __ldg(xi + c0 + 1));
                    s1 += m1.x * ldx<CG>(x + __ldg(xi + c1)) + m1.y * ldx<CG>(x + __ldg(xi + c1 + 1));
                    s2 += m2.x * ldx<CG>(x + __ldg(xi + c2)) + m2.y * ldx<CG>(x + __ldg(xi + c2 + 1));
                    s3 += m3.x * ldx<CG>(x + __ldg(xi + c3)) + m3.y * ldx<CG>(x + __ldg(xi + c3 + 1));
                }
                for (; p < pend; p += lpr) {
                    const double2 m = __ldg(M2 + p);
                    s0 += m.x * ldx<CG>(x + __ldg(xi + 2 * p)) + m.y * ldx<CG>(x + __ldg(xi + 2 * p + 1));
                }
            } else {
                for (; p + 3 * lpr < pend; p += 4 * lpr) {
                    const double2 m0 = __ldg(M2 + p), m1 = __ldg(M2 + p + lpr), m2 = __ldg(M2 + p + 2 * lpr),
                                  m3 = __ldg(M2 + p + 3 * lpr);
                    const int c0 = 2 * p, c1 = 2 * (p + lpr), c2 = 2 * (p + 2 * lpr), c3 = 2 * (p + 3 * lpr);
                    s0 += m0.x * ldx<CG>(x + c0) + m0.y * ldx<CG>(x + c0 + 1);
                    s1 += m1.x * ldx<CG>(x + c1) + m1.y * ldx<CG>(x + c1 + 1);
                    s2 += m2.x * ldx<CG>(x + c2) + m2.y * ldx<CG>(x + c2 + 1);
                    s3 += m3.x * ldx<CG>(x + c3) + m3.y * ldx<CG>(x + c3 + 1);
                }
                for (; p < pend; p += lpr) {
                    const double2 m = __ldg(M2 + p);
                    s0 += m.x * ldx<CG>(x + 2 * p) + m.y * ldx<CG>(x + 2 * p + 1);
                }
            }
        } else if (r < rows) {
            const double *Mr = M + (long long)r * ld;
            const int cend = lower ? min(cols, r + 1) : cols;
            int c = (upper ? r : 0) + sub;
            const int step = 4 * lpr;
            if (xi) {
                for (; c + 3 * lpr < cend; c += step) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + lpr), m2 = ldnc(Mr + c + 2 * lpr),
                                 m3 = ldnc(Mr + c + 3 * lpr);
                    s0 += m0 * ldx<CG>(x + __ldg(xi + c));
                    s1 += m1 * ldx<CG>(x + __ldg(xi + c + lpr));
                    s2 += m2 * ldx<CG>(x + __ldg(xi + c + 2 * lpr));
                    s3 += m3 * ldx<CG>(x + __ldg(xi + c + 3 * lpr));
                }
                for (; c < cend; c += lpr) s0 += ldnc(Mr + c) * ldx<CG>(x + __ldg(xi + c));
            } else {
                for (; c + 3 * lpr < cend; c += step) {
                    const double m0 = ldnc(Mr + c), m1 = ldnc(Mr + c + lpr), m2 = ldnc(Mr + c + 2 * lpr),
                                 m3 = ldnc(Mr + c + 3 * lpr);
                    s0 += m0 * ldx<CG>(x + c);
                    s1 += m1 * ldx<CG>(x + c + lpr);
                    s2 += m2 * ldx<CG>(x + c + 2 * lpr);
                    s3 += m3 * ldx<CG>(x + c + 3 * lpr);
                }
                for (; c < cend; c += lpr) s0 += ldnc(Mr + c) * ldx<CG>(x + c);
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
        for (int r = r0 + t; r < r1; r += T) xr[r - r0] = ldx<CG>(x + (xi ? __ldg(xi + r) : r));
        __syncthreads();
        if ((mode & 32) && !lower) {
            // column pairs: a thread owns columns (c, c+1), double2 loads down its rows
            const int cwp = cw >> 1;              // pair-threads per row group (16 .. 128)
            const int nsub = T / cwp;
            const int sub = t / cwp, c = tile * CTILE + 2 * (t % cwp);
            double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, b3 = 0.0;
            if (c + 1 < cols) {
                int r = r0 + sub;
                const double *Mc = M + (long long)r * ld + c;
                const long long st = (long long)nsub * ld;
                for (; r + 3 * nsub < r1; r += 4 * nsub, Mc += 4 * st) {
                    const double2 m0 = __ldg(reinterpret_cast<const double2 *>(Mc)),
                                  m1 = __ldg(reinterpret_cast<const double2 *>(Mc + st)),
                                  m2 = __ldg(reinterpret_cast<const double2 *>(Mc + 2 * st)),
                                  m3 = __ldg(reinterpret_cast<const double2 *>(Mc + 3 * st));
                    const double x0 = xr[r - r0], x1 = xr[r + nsub - r0], x2 = xr[r + 2 * nsub - r0],
                                 x3 = xr[r + 3 * nsub - r0];
                    a0 += m0.x * x0; b0 += m0.y * x0;
                    a1 += m1.x * x1; b1 += m1.y * x1;
                    a2 += m2.x * x2; b2 += m2.y * x2;
                    a3 += m3.x * x3; b3 += m3.y * x3;
                }
                for (; r < r1; r += nsub, Mc += st) {
                    const double2 m = __ldg(reinterpret_cast<const double2 *>(Mc));
                    a0 += m.x * xr[r - r0];
                    b0 += m.y * xr[r - r0];
                }
            } else if (c < cols) {
                for (int r = r0 + sub; r < r1; r += nsub) a0 += ldnc(M + (long long)r * ld + c) * xr[r - r0];
            }
            part[2 * t] = (a0 + a1) + (a2 + a3);
            part[2 * t + 1] = (b0 + b1) + (b2 + b3);
            __syncthreads();
            if (sub == 0 && c < cols) {
                double sa = part[2 * t], sb = part[2 * t + 1];
                for (int q = 1; q < nsub; ++q) {
                    sa += part[2 * (t + q * cwp)];
                    sb += part[2 * (t + q * cwp) + 1];
                }
                double *da = y + (yi ? __ldg(yi + c) : c);
                if (mode & 16) *da += alpha * sa;
                else atomicAdd(da, alpha * sa);
                if (c + 1 < cols) {
                    double *db = y + (yi ? __ldg(yi + c + 1) : c + 1);
                    if (mode & 16) *db += alpha * sb;
                    else atomicAdd(db, alpha * sb);
                }
            }
            return;
        }
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

// L2 prefetch of the matrix bytes that block lb of problem d reads (128-byte lines).
// The factor's matrices are static during an apply, so the phase kernels issue this
// BEFORE the programmatic-dependency wait: the DRAM fetch of a phase's matrices
// overlaps the tail of the previous phase (the phases are chains of dependent
// launches, most of them under one wave), and every line of a block is requested at
// once instead of eight loads per lane at a time.  A hint only: results are unchanged.
#ifndef GEMV_PREFETCH
#define GEMV_PREFETCH 1
#endif
#ifndef GEMV_TASK_PREFETCH
#define GEMV_TASK_PREFETCH 0  // one op ahead inside the subtree tasks: measured 3% slower (3.71 vs 3.60 ms)
#endif
__device__ __forceinline__ void prefetch_block(const GemvProb &d, long long lb) {
    const int mode = d.mode;
    const bool trans = mode & 1, lower = mode & 2, upper = mode & 8;
    int r0, r1, c0, c1;
    if (!trans) {
        const int per = (T / d.lpr) * (((mode & 32) && !lower && !upper) ? RPB : 1);  // rows per block
        r0 = (int)lb * per;
        r1 = min(d.rows, r0 + per);
        c0 = 0;
        c1 = d.cols;
    } else {
        const int ntile = (d.cols + CTILE - 1) / CTILE;
        r0 = (int)(lb / ntile) * SLAB;
        r1 = min(d.rows, r0 + SLAB);
        c0 = (int)(lb % ntile) * CTILE;
        c1 = min(d.cols, c0 + CTILE);
    }
    if (r1 <= r0 || c1 <= c0) return;
    const int lines = ((c1 - c0) * 8 + 127) / 128 + 1;  // per row, upper bound
    const int n = (r1 - r0) * lines;
    for (int i = threadIdx.x; i < n; i += T) {
        const int r = r0 + i / lines, l = i % lines;
        const int a = upper ? max(c0, r) : c0, b = lower ? min(c1, r + 1) : c1;  // columns row r reads
        if (b <= a) continue;
        const double *row = d.M + (long long)r * d.ld;
        const size_t lo = reinterpret_cast<size_t>(row + a) & ~size_t(127);
        const size_t hi = reinterpret_cast<size_t>(row + b - 1);
        const size_t q = lo + 128 * (size_t)l;
        if (q <= hi) asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
    }
}

__global__ void __launch_bounds__(T, GEMV_MINB) gemv_kernel(const __grid_constant__ GemvArgs a) {
    __shared__ double xr[SLAB];
    __shared__ double part[2 * T];
    const long long blk = blockIdx.x;
    const int p = find_prob(a.p, 0, a.count - 1, blk);
    // programmatic dependent launch: the apply's phases are chains of these launches;
    // let the next phase's CTAs be scheduled now, and wait here until the previous
    // phase (whose outputs are this phase's inputs) has completed and flushed
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (GEMV_PREFETCH) prefetch_block(a.p[p], blk - a.p[p].blk_begin);
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    gemv_block(a.p[p], blk - a.p[p].blk_begin, xr, part);
}

// The same block for phases with more problems than one parameter block holds: the
// descriptors live in device memory (static after factorization, uploaded once) with a
// block -> problem map, so a whole phase is ONE launch instead of ceil(count / GMAXP)
// back-to-back launches (config[4]'s interior-coupling phases have 4546 problems: 21
// launches of ~19 us, each paying its own ramp and tail).  The descriptor does not
// depend on the previous phase, so it is fetched before the dependency wait.
__global__ void __launch_bounds__(T, GEMV_MINB) gemv_dev_kernel(const GemvProb *__restrict__ P, const int *__restrict__ b2p) {
    __shared__ double xr[SLAB];
    __shared__ double part[2 * T];
    const long long blk = blockIdx.x;
    const GemvProb d = P[__ldg(b2p + blk)];
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (GEMV_PREFETCH) prefetch_block(d, blk - d.blk_begin);
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
    __shared__ double part[2 * T];
    const int o0 = __ldg(task_ptr + blockIdx.x), o1 = __ldg(task_ptr + blockIdx.x + 1);
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#if GEMV_TASK_PREFETCH
    // the task's first op before the dependency wait, then always one op ahead
    // (the ops of a task run one after the other, each a short dependent chain)
    if (o0 < o1) {
        const GemvProb d = ops[o0];
        const long long nb = ops[o0 + 1].blk_begin - d.blk_begin;
        for (long long lb = 0; lb < nb; ++lb) prefetch_block(d, lb);
    }
#endif
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    for (int o = o0; o < o1; ++o) {
        const GemvProb d = ops[o];
        const long long nb = ops[o + 1].blk_begin - d.blk_begin;  // ops end with a sentinel
#if GEMV_TASK_PREFETCH
        if (o + 1 < o1) {
            const GemvProb e = ops[o + 1];
            const long long ne = ops[o + 2].blk_begin - e.blk_begin;
            for (long long lb = 0; lb < ne; ++lb) prefetch_block(e, lb);
        }
#endif
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
    __shared__ double part[2 * T];
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

// The whole apply (both sweeps) as ONE persistent dataflow launch.  Items = the
// blocks of every op, in a topological order of the op graph (rsc_flow_deps); CTAs
// take items from a global counter in that order, wait until the item's op has
// received all its predecessors' completion signals, run the block, and the block
// that completes an op signals the op's successors.  Deadlock-free without any
// co-residency assumption: an item waits only on ops earlier in the order, whose
// items were all taken by CTAs that are already running.  The level phases' ~1000
// dependent launches (5-7 us of ramp, tail and launch latency each on config[4])
// become flag waits on the ops that actually feed an op, and independent subtrees'
// chains overlap instead of meeting at every level barrier.
//
// state: [0] item counter, [1, 1+nops) finished blocks per op, [1+nops, 1+2 nops)
// completion signals received per op -- zeroed before every launch.
__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ int atom_add_acqrel(int *p, int v) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void red_add_release(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long v;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
    return v;
}

// trace (diagnostics, rsc_apply_flow_trace): per item the %globaltimer at take, after
// the dependency wait and at completion, and the SM
#ifndef FLOW_PREFETCH
#define FLOW_PREFETCH 1
#endif
// L2 prefetch of the matrix region of blocks [lb0, lb1) of op d (128-byte lines)
__device__ __forceinline__ void prefetch_item(const GemvProb &d, int lb0, int lb1) {
    if (d.rows <= 0 || d.cols <= 0) return;
    const int t = threadIdx.x;
    int r0, r1, c0, c1;
    if (!(d.mode & 1)) {
        const int nseg = (T / d.lpr) * (((d.mode & 32) && !(d.mode & (2 | 8))) ? RPB : 1);  // rows per block
        r0 = lb0 * nseg;
        r1 = min(d.rows, lb1 * nseg);
        c0 = 0;
        c1 = d.cols;
    } else {  // blocks = (slab, column tile), tile fastest: cover the slabs' full width
        const int ntile = (d.cols + CTILE - 1) / CTILE;
        r0 = (lb0 / ntile) * SLAB;
        r1 = min(d.rows, ((lb1 - 1) / ntile + 1) * SLAB);
        c0 = 0;
        c1 = d.cols;
    }
    const long long first = (long long)(reinterpret_cast<size_t>(d.M + c0) >> 7);
    const int lines = (int)(((reinterpret_cast<size_t>(d.M + c1 - 1)) >> 7) - first + 1);
    const int n = (r1 - r0) * lines;
    for (int i = t; i < n; i += T) {
        const int r = r0 + i / lines, l = i % lines;
        const char *a = reinterpret_cast<const char *>(d.M + (long long)r * d.ld + c0);
        a = reinterpret_cast<const char *>((reinterpret_cast<size_t>(a) & ~size_t(127)) + 128 * (size_t)l);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
}

template <bool TRACE>
__global__ void __launch_bounds__(T) apply_flow_kernel(const GemvProb *__restrict__ ops,
                                                        const int *__restrict__ item_op,
                                                        const int *__restrict__ need,
                                                        const int *__restrict__ succ_ptr,
                                                        const int *__restrict__ succ, int *state, int nops,
                                                        int total, unsigned long long *trace) {
    __shared__ double xr[SLAB];
    __shared__ double part[2 * T];
    __shared__ int s_item[2], s_last;
    int *head = state, *done = state + 1, *ready = state + 1 + nops;
    const int t = threadIdx.x;
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (t == 0) s_item[0] = atomicAdd(head, 1);
    __syncthreads();
    int item = s_item[0], buf = 0;
    while (item < total) {
        unsigned long long t_take = 0, t_go = 0;
        if (TRACE && t == 0) t_take = gtimer();
        // take the next item now: the counter's round trip overlaps this item's work
        if (t == 0) s_item[buf ^ 1] = atomicAdd(head, 1);
        const int o = __ldg(item_op + item);
        const GemvProb d = ops[o];
        const int it = item - (int)d.blk_begin;
        const int lb0 = it * d.grp, lb1 = min(lb0 + d.grp, d.nblk);
        // the matrix tile does not depend on the predecessors: start pulling it into
        // L2 now, so that after the wait only the vector loads see memory latency
        if (FLOW_PREFETCH) prefetch_item(d, lb0, lb1);
        if (t == 0) {
            const int nd = __ldg(need + o);
            if (nd > 0)
                while (ld_acquire(ready + o) < nd) __nanosleep(32);
            if (TRACE) t_go = gtimer();
        }
        __syncthreads();
        for (int lb = lb0; lb < lb1; ++lb) gemv_block<true>(d, lb, xr, part);
        __syncthreads();
        if (t == 0) {
            // release this CTA's writes (ordered before by the barrier) and count the item;
            // the op's last item acquires every other item's writes before signalling
            const int nitems = (d.nblk + d.grp - 1) / d.grp;
            s_last = (nitems == 1) || (atom_add_acqrel(done + o, 1) == nitems - 1);
            if (TRACE) {
                unsigned smid;
                asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
                trace[4 * (long long)item] = t_take;
                trace[4 * (long long)item + 1] = t_go;
                trace[4 * (long long)item + 2] = gtimer();
                trace[4 * (long long)item + 3] = smid;
            }
        }
        __syncthreads();
        if (s_last) {
            const int e0 = __ldg(succ_ptr + o), e1 = __ldg(succ_ptr + o + 1);
            if (e1 > e0) {
                if (t == 0) __threadfence();
                __syncthreads();
                for (int e = e0 + t; e < e1; e += T) red_add_release(ready + __ldg(succ + e), 1);
            }
        }
        buf ^= 1;
        item = s_item[buf];
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
    // bit 5: every row starts 16-byte aligned (double2 loads)
    static const bool scalar_only = getenv("RSC_GEMV_SCALAR") != nullptr;  // A/B switch
    const bool vec = (reinterpret_cast<size_t>(M) % 16 == 0) && (ld % 2 == 0) && !scalar_only;
    mode = (mode & ~32) | (vec ? 32 : 0);
    d.rows = rows; d.cols = cols; d.ld = ld; d.mode = mode; d.alpha = alpha;
    if (mode & 1) {
        d.lpr = cols >= CTILE ? CTILE : (pow2ceil(cols) < 32 ? 32 : pow2ceil(cols));
        return (long long)((rows + SLAB - 1) / SLAB) * ((cols + CTILE - 1) / CTILE);
    }
    d.lpr = cols <= 64 ? 8 : (cols <= 256 ? 16 : 32);  // (lpr 32 from 65 columns measured slower)
    const int nseg = T / d.lpr;
    if (vec && !(mode & (2 | 8))) return (rows + nseg * RPB - 1) / (nseg * RPB);  // RPB rows per segment
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

inline long long flow_item_bytes() {
    static const long long b = getenv("RSC_FLOW_ITEM_KB") ? atoll(getenv("RSC_FLOW_ITEM_KB")) * 1024 : 32 * 1024;
    return b;
}

// Descriptors of the dataflow program: like rsc_gemv_describe, but every op gets at
// least one item (an op whose rank dropped to 0 still completes and signals), the
// items are numbered globally in op order (blk_begin), the plain-accumulate bit is
// dropped (every accumulation is an L2 atomic: other CTAs may target the same rows),
// and item_op (if not null) receives the item -> op map.  Returns the item count.
extern "C" long long rsc_flow_describe(int count, const double *const *M, const int *rows, const int *cols,
                                       const int *ldm, const double *const *x, const int *const *xidx,
                                       double *const *y, const int *const *yidx, const int *modes,
                                       const double *alphas, void *desc, int *item_op) {
    if (count < 0) return -1;
    if (count > 0 && (!M || !rows || !cols || !ldm || !x || !y || !modes || !alphas || !desc)) return -2;
    GemvProb *d = static_cast<GemvProb *>(desc);
    long long total = 0;
    for (int i = 0; i < count; ++i) {
        d[i] = GemvProb{};
        long long nb = 0;
        const int mode = modes[i] & ~16;
        if (rows[i] > 0 && cols[i] > 0) {
            const long long nblk = describe(d[i], M[i], rows[i], cols[i], ldm[i], x[i], xidx ? xidx[i] : nullptr,
                                            y[i], yidx ? yidx[i] : nullptr, mode, alphas[i]);
            // blocks per item: about FLOW_ITEM_BYTES of matrix per item (the per-item
            // queue / wait / signal round trips are amortized over it)
            const long long bb = (mode & 1) ? (long long)SLAB * (cols[i] < CTILE ? cols[i] : CTILE) * 8
                                            : (long long)(T / d[i].lpr) * cols[i] * 8;
            long long g = flow_item_bytes() / (bb > 0 ? bb : 1);
            g = g < 1 ? 1 : (g > nblk ? nblk : g);
            d[i].nblk = (int)nblk;
            d[i].grp = (int)g;
            nb = (nblk + g - 1) / g;
        } else {  // an empty op (rank 0): one no-op item so that it still signals
            d[i].M = M[i]; d[i].x = x[i]; d[i].y = y[i];
            d[i].rows = 0; d[i].cols = 0; d[i].ld = 1; d[i].mode = 0; d[i].lpr = 32;  // no rows: no writes
            d[i].nblk = 1; d[i].grp = 1;
            d[i].alpha = alphas[i];
            nb = 1;
        }
        d[i].blk_begin = total;
        if (item_op)
            for (long long b = 0; b < nb; ++b) item_op[total + b] = i;
        total += nb;
    }
    return total;
}

int flow_launch(const void *ops, const int *item_op, const int *need, const int *succ_ptr, const int *succ,
                int *state, int nops, int total, unsigned long long *trace, cudaStream_t s);

extern "C" int rsc_apply_flow_trace(const void *ops, const int *item_op, const int *need, const int *succ_ptr,
                                    const int *succ, int *state, int nops, int total, void *trace, void *stream) {
    if (!trace) return -2;
    return flow_launch(ops, item_op, need, succ_ptr, succ, state, nops, total,
                       static_cast<unsigned long long *>(trace), (cudaStream_t)stream);
}

extern "C" int rsc_apply_flow(const void *ops, const int *item_op, const int *need, const int *succ_ptr,
                              const int *succ, int *state, int nops, int total, void *stream) {
    return flow_launch(ops, item_op, need, succ_ptr, succ, state, nops, total, nullptr, (cudaStream_t)stream);
}

int flow_launch(const void *ops, const int *item_op, const int *need, const int *succ_ptr, const int *succ,
                int *state, int nops, int total, unsigned long long *trace, cudaStream_t s) {
    if (nops < 0 || total < 0) return -1;
    if (total == 0) return 0;
    if (!ops || !item_op || !need || !succ_ptr || !succ || !state) return -2;
    static int grid = 0;
    if (!grid) {
        int dev = 0, nsm = 0, occ = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, apply_flow_kernel<false>, T, 0);
        grid = nsm * (occ > 0 ? occ : 1);
    }
    cudaError_t e = cudaMemsetAsync(state, 0, sizeof(int) * (1 + 2 * (size_t)nops), s);
    if (e != cudaSuccess) return (int)e;
    const int g = grid < total ? grid : total;
    if (trace)
        apply_flow_kernel<true><<<g, T, 0, s>>>(static_cast<const GemvProb *>(ops), item_op, need, succ_ptr, succ,
                                                 state, nops, total, trace);
    else
        apply_flow_kernel<false><<<g, T, 0, s>>>(static_cast<const GemvProb *>(ops), item_op, need, succ_ptr, succ,
                                                  state, nops, total, nullptr);
    rsc_count_launch();
    e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
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

// Batched rectangular copy (trans 0: dst = src) or transpose (trans 1: dst = src^T,
// src rows x cols) for the diagonal trees' flattened inverses (apply.py: copies of
// V / U and of the dense couplings before the tree solves).  Row tiles of every
// matrix are dealt over gridDim.y.
namespace {
constexpr int RMAX = 768;
struct RectArgs {
    int count, trans;
    const double *src[RMAX];
    double *dst[RMAX];
    int rows[RMAX], cols[RMAX], lds[RMAX], ldd[RMAX];
};

__global__ void __launch_bounds__(256) rect_copy_kernel(const __grid_constant__ RectArgs a) {
    __shared__ double tile[32][33];
    const int b = blockIdx.x;
    const int rows = a.rows[b], cols = a.cols[b], lds = a.lds[b], ldd = a.ldd[b];
    const double *S = a.src[b];
    double *D = a.dst[b];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int i0 = 32 * blockIdx.y; i0 < rows; i0 += 32 * gridDim.y)
        for (int j0 = 0; j0 < cols; j0 += 32) {
            if (!a.trans) {
                for (int q = ty; q < 32; q += 8) {
                    const int i = i0 + q, j = j0 + tx;
                    if (i < rows && j < cols) D[(long long)i * ldd + j] = S[(long long)i * lds + j];
                }
                continue;
            }
            for (int q = ty; q < 32; q += 8) {
                const int i = i0 + q, j = j0 + tx;
                tile[q][tx] = (i < rows && j < cols) ? S[(long long)i * lds + j] : 0.0;
            }
            __syncthreads();
            for (int q = ty; q < 32; q += 8) {
                const int i = j0 + q, j = i0 + tx;  // D[i][j] = S[j][i]
                if (i < cols && j < rows) D[(long long)i * ldd + j] = tile[tx][q];
            }
            __syncthreads();
        }
}
}  // namespace

extern "C" int rsc_copy2d_batched(int count, const double *const *src, double *const *dst, const int *rows,
                                  const int *cols, const int *lds, const int *ldd, int trans, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!src || !dst || !rows || !cols || !lds || !ldd) return -2;
    static thread_local RectArgs a;
    for (int c0 = 0; c0 < count; c0 += RMAX) {
        const int cnt = count - c0 < RMAX ? count - c0 : RMAX;
        a.count = cnt;
        a.trans = trans ? 1 : 0;
        int maxr = 1;
        for (int i = 0; i < cnt; ++i) {
            a.src[i] = src[c0 + i];
            a.dst[i] = dst[c0 + i];
            a.rows[i] = rows[c0 + i];
            a.cols[i] = cols[c0 + i];
            a.lds[i] = lds[c0 + i];
            a.ldd[i] = ldd[c0 + i];
            maxr = a.rows[i] > maxr ? a.rows[i] : maxr;
        }
        int gy = (maxr + 255) / 256;  // ~8 row tiles per CTA of the tallest matrix
        gy = gy < 1 ? 1 : (gy > 64 ? 64 : gy);
        rect_copy_kernel<<<dim3(cnt, gy), 256, 0, (cudaStream_t)stream>>>(a);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

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
