// Multi-matrix cooperative column-pivoted Householder QR.
//
// Same arithmetic contract as qrcp_kernel (LAPACK dlaqp2 pivoting, dlarfg
// reflectors, partial-norm downdating with the sqrt(eps) recomputation test,
// dorg2r for the kept columns; reference kernels.py:67-82), for sketches that do
// not fit one SM and for running many such QRs at once.
//
// Every matrix of a launch gets a GROUP of CTAs; CTA b of a group owns physical
// columns [b*cpc, (b+1)*cpc) and keeps them in shared memory for the whole
// factorization.  Pivoting never moves data: every CTA keeps the same
// position->column permutation and applies LAPACK's swap sequence to it
// redundantly, so "first position of the largest partial norm" is reproduced
// exactly.  Per column: the owner of the pivot column forms and publishes the
// reflector -> group barrier -> every CTA updates its own columns and downdates
// their norms -> group barrier.  Group barriers are release/acquire counters
// (one per matrix), so the QRs of a whole ND level run concurrently; the launch is
// cooperative, which guarantees every CTA of every group is co-resident.
//
// Q is formed afterwards (qr_form_q_kernel): column j of Q is H_0 ... H_j e_j
// applied right-to-left (dorg2r order), one warp per column.
#include <cooperative_groups.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cstdlib>
#include <vector>
#include "common.cuh"

namespace {

constexpr int CT = 256;   // threads per CTA (8 warps): cluster QRCP, Q formation
constexpr int MCT = 512;  // threads per CTA of the cooperative QRCP (16 warps: the owned-column updates and
                          // block reductions of a column step spread over twice the warps)
constexpr int MAXM = 96;
constexpr double EPS = 2.220446049250313e-16;
constexpr double TOL3Z = 1.0536712127723509e-08;
constexpr size_t SMEM_BUDGET = 200 * 1024;

struct MatDesc {
    const double *G;
    double *Q;
    double *W;  // per-matrix workspace: cols (ldw*k) | vn1 | vn2 | tau | diagR | vbuf(m) | perm(k ints)
    int *rank;
    int m, k, ldg, ldq, ldw, cpc, nblk, blk0;
    int vsm;    // global-column variant: the reflector is staged in shared memory
};

struct MArgs {
    int count;
    unsigned *bar;  // one zeroed counter per matrix
    MatDesc d[MAXM];
};

struct Ws {
    double *cols, *vn1, *vn2, *tau, *diagR, *vbuf;
    int *perm;
    double *cand_v;    // per-CTA pivot candidate of the next step: largest vn1 ...
    int *cand_p;       // ... its position ...
    int *cand_pc;      // ... and its physical column (-1: none); all three double-buffered by step parity
    double *cand_col;  // the candidate column itself (rows >= the step), [parity][CTA][ldw]
    int cq2;           // CTAs per parity slot of cand_col
};

constexpr int CQ_MAX = 256;  // >= CTAs of one matrix group (<= SM count)
constexpr int QB_WY = 64;    // = QB, the compact-WY block of the Q formation below

// start (in doubles) of the candidate region, after the factorization workspace and
// the WY region of the Q formation (rsc_qrcp_coop_doubles)
__host__ __device__ inline long long coop_cand_base(int m, int k) {
    const long long ldw = m | 1;
    const long long kmin = m < k ? m : k;
    return ldw * k + 4LL * k + m + k + 2 * CQ_MAX + 64 + (long long)m * kmin + QB_WY * kmin +
           2LL * QB_WY * QB_WY + 64;
}

__device__ __forceinline__ Ws carve(const MatDesc &d) {
    Ws w;
    w.cols = d.W;
    w.vn1 = d.W + (long long)d.ldw * d.k;
    w.vn2 = w.vn1 + d.k;
    w.tau = w.vn2 + d.k;
    w.diagR = w.tau + d.k;
    w.vbuf = w.diagR + d.k;
    w.perm = reinterpret_cast<int *>(w.vbuf + d.m);
    double *ext = d.W + coop_cand_base(d.m, d.k);
    w.cand_v = ext;
    w.cand_p = reinterpret_cast<int *>(ext + 2 * CQ_MAX);
    w.cand_pc = w.cand_p + 2 * CQ_MAX;
    w.cand_col = ext + 4 * CQ_MAX;
    w.cq2 = d.k < CQ_MAX ? d.k : CQ_MAX;
    return w;
}

__device__ __forceinline__ void group_barrier(unsigned *ctr, int nblk, unsigned &epoch) {
    __syncthreads();
    if (nblk > 1) {
        if (threadIdx.x == 0) {
            // release-increment (orders this CTA's prior writes, which bar.sync made
            // visible to this thread, before the arrival) instead of a full
            // __threadfence + atomicAdd; acquire-poll for the last arrival
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(ctr) : "memory");
            const unsigned target = (epoch + 1) * (unsigned)nblk;
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
            } while (v < target);
        }
        __syncthreads();
    }
    ++epoch;
}

// This CTA's pivot candidate for step i: the largest vn1 among its owned columns
// still at positions >= i (first position on ties; NaN never wins), published to
// slot `par` of cand_v / cand_p / cand_pc.  The next pivot search then reads one
// candidate per CTA instead of walking all k norms through L2.  With pub_col the
// candidate column's rows [i, m) are published too (cand_col), so every CTA can form
// the next reflector itself when this candidate wins -- no second group barrier per
// column step.
__device__ __forceinline__ void publish_candidate(const Ws &w, const double *vn1, const int *posof, int c0, int c1,
                                                  int i, int lb, double *red, int *redp, int par, const double *cols,
                                                  int ldw, int m, bool pub_col) {
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    double best = -1.0;
    int bp = 0x7fffffff, bph = -1;
    for (int phys = c0 + t; phys < c1; phys += MCT) {
        const int ps = posof[phys];
        if (ps < i) continue;
        const double vv = vn1[phys];
        if (vv > best || (vv == best && ps < bp)) { best = vv; bp = ps; bph = phys; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int oh = __shfl_xor_sync(0xffffffffu, bph, o);
        if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; bph = oh; }
    }
    __shared__ int s_bph;
    if (lane == 0) { red[warp] = best; redp[warp] = bp; redp[16 + warp] = bph; }
    __syncthreads();
    if (t == 0) {
        for (int q = 1; q < MCT / 32; ++q)
            if (red[q] > best || (red[q] == best && redp[q] < bp)) { best = red[q]; bp = redp[q]; bph = redp[16 + q]; }
        w.cand_v[par * CQ_MAX + lb] = best;
        w.cand_p[par * CQ_MAX + lb] = bp;
        w.cand_pc[par * CQ_MAX + lb] = (best >= 0.0) ? bph : -1;
        s_bph = (best >= 0.0) ? bph : -1;
    }
    if (pub_col) {
        __syncthreads();
        const int ph = s_bph;
        if (ph >= 0) {
            const double *src = cols + (long long)(ph - c0) * ldw;
            double *dst = w.cand_col + ((long long)par * w.cq2 + lb) * ldw;
            for (int r = i + t; r < m; r += MCT) dst[r] = src[r];
        }
    }
}

// CB block sums at once (one pass through shared memory); results broadcast.
// red must hold >= CB * CT/32 doubles.
template <int CB>
__device__ __forceinline__ void block_sum_n(double (&x)[CB], double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int NW = MCT / 32;
#pragma unroll
    for (int c = 0; c < CB; ++c) x[c] = warp_sum(x[c]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int c = 0; c < CB; ++c) red[c * NW + warp] = x[c];
    __syncthreads();
#pragma unroll
    for (int c = 0; c < CB; ++c) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) t += red[c * NW + q];  // same order in every thread
        x[c] = t;
    }
}

// Householder step i on this CTA's global-memory columns [c0, c1) (mqrcp_kernel,
// !SMEM): apply H_i^T = I - tau v v^T (v[i] = 1 implicit, v[i+1..m) in `vs`) to the
// columns still unchosen, then the dlaqp2 norm downdate with the sqrt(eps)
// recomputation test.  CB columns per pass; every sum is a fixed-order block sum.
__device__ __forceinline__ void coop_update(double *vn1, double *vn2, double *cols, const double *vs, bool vsm,
                                            const int *posof, int c0, int c1, int i, int m, int ldw, double tau,
                                            double *red) {
    constexpr int CB = 4;
    __shared__ int s_redo[CB];
    const int t = threadIdx.x;
    for (int jb = c0; jb < c1; jb += CB) {
        bool on[CB];
        double *cj[CB];
        bool any = false;
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            const int phys = jb + c;
            on[c] = phys < c1 && posof[phys] > i;  // posof is replicated: uniform in the CTA
            cj[c] = cols + (long long)(on[c] ? phys - c0 : 0) * ldw;
            any |= on[c];
        }
        if (!any) continue;
        double f[CB], cji0[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) cji0[c] = on[c] ? cj[c][i] : 0.0;  // before thread 0 rewrites row i
        if (tau != 0.0) {
            double x[CB];
#pragma unroll
            for (int c = 0; c < CB; ++c) x[c] = 0.0;
#pragma unroll 4
            for (int r = i + 1 + t; r < m; r += MCT) {
                const double vr = vsm ? vs[r] : __ldcg(vs + r);
#pragma unroll
                for (int c = 0; c < CB; ++c)
                    if (on[c]) x[c] = fma(vr, cj[c][r], x[c]);
            }
            block_sum_n<CB>(x, red);
#pragma unroll
            for (int c = 0; c < CB; ++c) f[c] = on[c] ? tau * (x[c] + cji0[c]) : 0.0;
#pragma unroll 4
            for (int r = i + 1 + t; r < m; r += MCT) {
                const double vr = vsm ? vs[r] : __ldcg(vs + r);
#pragma unroll
                for (int c = 0; c < CB; ++c)
                    if (on[c]) cj[c][r] -= f[c] * vr;
            }
        }
        if (t == 0) {
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                s_redo[c] = 0;
                if (!on[c]) continue;
                double cji = cji0[c];
                if (tau != 0.0) {
                    cji -= f[c];
                    cj[c][i] = cji;
                }
                const int phys = jb + c;
                const double v1 = vn1[phys];
                if (v1 == 0.0) continue;
                double temp = fabs(cji) / v1;
                temp = 1.0 - temp * temp;
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = v1 / vn2[phys];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= TOL3Z) s_redo[c] = 1;
                else vn1[phys] = v1 * sqrt(temp);
            }
        }
        __syncthreads();  // the updated rows of this pass and the recompute flags
        bool redo[CB], anyr = false;
#pragma unroll
        for (int c = 0; c < CB; ++c) { redo[c] = s_redo[c] != 0; anyr |= redo[c]; }
        if (anyr) {
            double x[CB];
#pragma unroll
            for (int c = 0; c < CB; ++c) x[c] = 0.0;
#pragma unroll 4
            for (int r = i + 1 + t; r < m; r += MCT) {
#pragma unroll
                for (int c = 0; c < CB; ++c)
                    if (redo[c]) x[c] = fma(cj[c][r], cj[c][r], x[c]);
            }
            block_sum_n<CB>(x, red);
            if (t == 0)
#pragma unroll
                for (int c = 0; c < CB; ++c)
                    if (redo[c]) {
                        const double x2 = (i + 1 < m) ? sqrt(x[c]) : 0.0;
                        vn1[jb + c] = x2;
                        vn2[jb + c] = x2;
                    }
        }
        __syncthreads();  // s_redo / red reused by the next pass
    }
}

// Global-memory columns come in two builds: 128 registers / one CTA per SM (fastest
// for a single sketch: 29.3 ms for 6048x987) and 64 registers / two CTAs per SM, so
// that two groups (the two 6048x987 top-separator sketches of config[4]) are
// co-resident instead of running one after the other (52.6 vs 58.3 ms for the pair,
// 80.5 vs 95.3 ms for three 9000x700; a single sketch would take 41.7 ms).  The host
// picks by the number of global-memory sketches left in the batch.  Bit-identical.
template <bool SMEM, int MINB>
__global__ void __launch_bounds__(MCT, MINB) mqrcp_kernel(const __grid_constant__ MArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64]  /* block_sum_n: CB x MCT/32 */;
    __shared__ int redp[32];
    __shared__ int piv_s;
    // locate this CTA's matrix
    int g = 0;
    while (g + 1 < a.count && (int)blockIdx.x >= a.d[g + 1].blk0) ++g;
    const MatDesc &d = a.d[g];
    const Ws w = carve(d);
    unsigned *bar = a.bar + g;
    const int m = d.m, k = d.k, ldw = d.ldw, cpc = d.cpc, nblk = d.nblk;
    const int lb = blockIdx.x - d.blk0;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = MCT / 32;
    const int c0 = lb * cpc, c1 = min(k, c0 + cpc);
    double *cols = SMEM ? sm : w.cols + (long long)c0 * ldw;
    const bool vsm = !SMEM && d.vsm;
    double *v = SMEM ? sm + (long long)cpc * ldw : (vsm ? sm : nullptr);
    int *pos2phys = reinterpret_cast<int *>(SMEM ? v + m : (vsm ? sm + m : sm));
    int *posof = pos2phys + k;
    // partial column norms of the owned columns in shared memory, indexed by the
    // physical column (the pivot search and the downdates never leave the SM)
    double *vn1 = reinterpret_cast<double *>(posof + k) - c0;
    double *vn2 = vn1 + cpc;
    unsigned epoch = 0;

    for (long long e = t; e < (long long)m * (c1 - c0); e += MCT) {
        const int r = (int)(e / (c1 - c0)), j = (int)(e % (c1 - c0));
        cols[(long long)j * ldw + r] = d.G[(long long)r * d.ldg + c0 + j];
    }
    for (int j = t; j < k; j += MCT) { pos2phys[j] = j; posof[j] = j; }
    __syncthreads();
    for (int j = warp; j < c1 - c0; j += nw) {
        const double *cj = cols + (long long)j * ldw;
        double s = 0.0;
        for (int r = lane; r < m; r += 32) s += cj[r] * cj[r];
        s = sqrt(warp_sum(s));
        if (lane == 0) { vn1[c0 + j] = s; vn2[c0 + j] = s; }
    }
    __syncthreads();
    // one group barrier per column step when the reflector can be staged in shared
    // memory: every CTA forms it from the published winning candidate column
    // (shared-memory columns publish a copy of their candidate column; global-memory
    // columns are read in place, and the owner writes the scaled reflector back into
    // its column only after the next barrier, when every CTA has read it)
    const bool onebar = nblk > 1 && (SMEM || vsm);
    __shared__ int fast_s;
    publish_candidate(w, vn1, posof, c0, c1, 0, lb, red, redp, 0, cols, ldw, m, onebar && SMEM);
    group_barrier(bar, nblk, epoch);

    const int kmin = m < k ? m : k;
    int pend_c = -1, pend_i = 0;  // deferred reflector write-back (global columns)
    double pend_beta = 0.0;
    for (int i = 0; i < kmin; ++i) {
        const int par = i & 1;
        if (!SMEM && pend_c >= 0) {  // v still holds step pend_i's reflector
            double *ci = cols + (long long)(pend_c - c0) * ldw;
            for (int r = pend_i + 1 + t; r < m; r += MCT) ci[r] = v[r];
            if (t == 0) ci[pend_i] = pend_beta;
            pend_c = -1;
            __syncthreads();
        }
        // 1. pivot: first position j >= i with the largest vn1 (identical in every CTA),
        // reduced over the group's per-CTA candidates
        if (warp == 0) {
            double best = -1.0;
            int bp = k, bpc = -1;  // bpc: the column the winning CTA published
            for (int b = lane; b < nblk; b += 32) {
                const double vv = __ldcg(w.cand_v + par * CQ_MAX + b);
                const int pp = __ldcg(w.cand_p + par * CQ_MAX + b);
                const int pcv = __ldcg(w.cand_pc + par * CQ_MAX + b);
                if (vv > best || (vv == best && pp < bp)) { best = vv; bp = pp; bpc = pcv; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bpc, o);
                if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; bpc = oc; }
            }
            if (lane == 0) {
                if (bp >= k) bp = i;  // NaN norms (failed upstream pivot): keep the order
                const int ci = pos2phys[i], cp = pos2phys[bp];
                pos2phys[i] = cp; pos2phys[bp] = ci;
                posof[cp] = i; posof[ci] = bp;
                piv_s = cp;
                // the owner published exactly this column as its candidate (else: the
                // NaN fallback above -- take the two-barrier path for this step)
                fast_s = onebar && bpc == cp;
            }
        }
        __syncthreads();
        const int pc = piv_s;
        const bool fast = fast_s != 0;
        double tau;
        if (fast) {
            // 2'. every CTA forms the reflector (dlarfg) from the published column, in
            // the same order the owner would: identical tau / beta / v everywhere
            const bool own = pc >= c0 && pc < c1;
            const double *src = own ? cols + (long long)(pc - c0) * ldw
                                : SMEM ? w.cand_col + ((long long)par * w.cq2 + pc / cpc) * ldw
                                       : w.cols + (long long)pc * ldw;
#pragma unroll 4
            for (int r = i + t; r < m; r += MCT) v[r] = own ? src[r] : __ldcg(src + r);
            __syncthreads();
            double part = 0.0;
            for (int r = i + 1 + t; r < m; r += MCT) part += v[r] * v[r];
            const double xnorm = sqrt(block_sum(part, red));
            const double alpha = v[i];
            double beta = alpha, scal = 0.0;
            tau = 0.0;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            double *ci = (own && SMEM) ? cols + (long long)(pc - c0) * ldw : nullptr;
            for (int r = i + 1 + t; r < m; r += MCT) {
                const double x = (xnorm != 0.0) ? v[r] * scal : v[r];
                v[r] = x;
                if (ci) ci[r] = x;
            }
            if (own && t == 0) {
                if (ci) ci[i] = beta;
                w.tau[i] = tau;
                w.diagR[i] = beta;
            }
            if (own && !SMEM) { pend_c = pc; pend_i = i; pend_beta = beta; }
            __syncthreads();
        } else {
            // 2. the owner of the pivot column forms and publishes the reflector (dlarfg)
            if (pc >= c0 && pc < c1) {
                double *ci = cols + (long long)(pc - c0) * ldw;
                double part = 0.0;
                for (int r = i + 1 + t; r < m; r += MCT) part += ci[r] * ci[r];
                const double xnorm = sqrt(block_sum(part, red));
                const double alpha = ci[i];
                double tau0 = 0.0, beta = alpha, scal = 0.0;
                if (xnorm != 0.0) {
                    beta = -copysign(hypot(alpha, xnorm), alpha);
                    tau0 = (beta - alpha) / beta;
                    scal = 1.0 / (alpha - beta);
                }
                __syncthreads();
                for (int r = i + 1 + t; r < m; r += MCT) {
                    const double x = (xnorm != 0.0) ? ci[r] * scal : ci[r];
                    ci[r] = x;
                    if (nblk > 1) w.vbuf[r] = x;
                }
                if (t == 0) {
                    ci[i] = beta;
                    w.tau[i] = tau0;
                    w.diagR[i] = beta;
                }
            }
            group_barrier(bar, nblk, epoch);
            tau = __ldcg(w.tau + i);
            if (nblk > 1 && (SMEM || vsm)) {
                for (int r = i + 1 + t; r < m; r += MCT) v[r] = __ldcg(w.vbuf + r);
                __syncthreads();
            }
        }
        // 3. apply H_i^T to the unchosen owned columns, downdate their norms
        if (!SMEM && nblk > 1) {
            // global-memory columns: the whole CTA works on its columns together
            // (rows spread over all threads, CB columns per pass, block reductions),
            // so every step keeps ~MCT x CB independent L2 loads in flight instead of
            // one warp walking one column serially through L2
            coop_update(vn1, vn2, cols, vsm ? v : w.vbuf, vsm, posof, c0, c1, i, m, ldw, tau, red);
        } else {
        const double *vsrc = (nblk == 1) ? cols + (long long)(pc - c0) * ldw  // the reflector lives in this CTA
                                         : v;
        for (int j = warp; j < c1 - c0; j += nw) {
            const int phys = c0 + j;
            if (posof[phys] <= i) continue;
            double *cj = cols + (long long)j * ldw;
            if (tau != 0.0) {
                double s = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) s += vsrc[r] * cj[r];
                s = warp_sum(s) + cj[i];
                const double f = tau * s;
                for (int r = i + 1 + lane; r < m; r += 32) cj[r] -= f * vsrc[r];
                __syncwarp();
                if (lane == 0) cj[i] -= f;
                __syncwarp();
            }
            const double v1 = vn1[phys];
            if (v1 != 0.0) {
                double temp = fabs(cj[i]) / v1;
                temp = 1.0 - temp * temp;
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = v1 / vn2[phys];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= TOL3Z) {
                    double s = 0.0;
                    for (int r = i + 1 + lane; r < m; r += 32) s += cj[r] * cj[r];
                    s = (i + 1 < m) ? sqrt(warp_sum(s)) : 0.0;
                    if (lane == 0) { vn1[phys] = s; vn2[phys] = s; }
                } else if (lane == 0) {
                    vn1[phys] = v1 * sqrt(temp);
                }
            }
            __syncwarp();
        }
        }
        if (i + 1 < kmin) {
            __syncthreads();
            publish_candidate(w, vn1, posof, c0, c1, i + 1, lb, red, redp, par ^ 1, cols, ldw, m, onebar && SMEM);
        }
        group_barrier(bar, nblk, epoch);
    }
    if (!SMEM && pend_c >= 0) {  // the last deferred reflector
        double *ci = cols + (long long)(pend_c - c0) * ldw;
        for (int r = pend_i + 1 + t; r < m; r += MCT) ci[r] = v[r];
        if (t == 0) ci[pend_i] = pend_beta;
        __syncthreads();
    }
    // spill the owned columns (reflectors) for the Q kernel; publish the permutation
    if (SMEM)
        for (long long e = t; e < (long long)ldw * (c1 - c0); e += MCT) w.cols[(long long)c0 * ldw + e] = cols[e];
    if (lb == 0)
        for (int j = t; j < k; j += MCT) w.perm[j] = pos2phys[j];
}


// ---- thread-block-cluster QRCP ------------------------------------------------
// The same algorithm for sketches that fit the shared memory of one cluster (<= 16
// CTAs): CTA b of the cluster owns physical columns [b*cpc, (b+1)*cpc) as in
// mqrcp_kernel, but the per-matrix state lives in every CTA's shared memory and
// moves through distributed shared memory: the owner of the pivot column PUSHES the
// reflector, tau and beta into every CTA's buffers, every CTA pushes the downdated
// norms of its columns into every replica, and the two synchronisations per column
// are hardware cluster barriers (release/acquire) instead of global-memory counters
// -- the pivot search then reads only local shared memory.
constexpr int QC_MAXC = 8;  // 16-CTA clusters measured slower than the cooperative kernel

struct QcArgs {
    int count;
    int C;
    MatDesc d[MAXM];
};

inline size_t cluster_smem(int m, int k, int cpc) {
    return (size_t)cpc * (size_t)(m | 1) * 8 + (size_t)m * 8 + 4 * (size_t)k * 8 + 2 * sizeof(int) * (size_t)k + 16;
}

__device__ unsigned long long qc_phase_cycles[32];  // RSC_QR_TIMING diagnostics

// Update of this warp's owned, still unchosen columns for Householder step i
// (apply H_i^T, dlaqp2 downdate, push the norms into every replica).  CB columns
// are processed interleaved; with RPL > 0 (m <= 32 RPL) rows are unrolled and the
// reflector sits in registers.
template <int RPL, int CB, class Cl>
__device__ __forceinline__ void qc_update(Cl &cl, int C, int i, int m, int k, int ldw, int lb, int nloc,
                                          double *cols, const double *v, double tau_i, double *vn1,
                                          double *vn2, const int *posof, int warp, int lane, int nw) {
    constexpr int R = RPL > 0 ? RPL : 1;
    double vr[R];
    if (RPL > 0) {
#pragma unroll
        for (int q = 0; q < R; ++q) {
            const int r = lane + 32 * q;
            vr[q] = (r > i && r < m) ? v[r] : 0.0;
        }
    }
    for (int jl0 = warp; jl0 < nloc; jl0 += CB * nw) {
        int phys[CB];
        bool on[CB];
        double *cj[CB];
        double x[CB][R], cji[CB], w[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            const int jl = jl0 + c * nw;
            phys[c] = lb + C * jl;
            on[c] = jl < nloc && phys[c] < k && posof[phys[c]] > i;
            cj[c] = cols + (long long)(on[c] ? jl : 0) * ldw;
            cji[c] = on[c] ? cj[c][i] : 0.0;
            w[c] = 0.0;
            if (RPL > 0) {
#pragma unroll
                for (int q = 0; q < R; ++q) {
                    const int r = lane + 32 * q;
                    x[c][q] = (on[c] && r < m) ? cj[c][r] : 0.0;
                }
            }
        }
        if (tau_i != 0.0) {
            if (RPL > 0) {
#pragma unroll
                for (int c = 0; c < CB; ++c)
#pragma unroll
                    for (int q = 0; q < R; ++q) w[c] = fma(vr[q], x[c][q], w[c]);
            } else {
#pragma unroll
                for (int c = 0; c < CB; ++c)
                    if (on[c])
                        for (int r = i + 1 + lane; r < m; r += 32) w[c] += v[r] * cj[c][r];
            }
            warp_sum4(w);
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                if (!on[c]) continue;
                const double f = tau_i * (w[c] + cji[c]);
                if (RPL > 0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int r = lane + 32 * q;
                        if (r > i && r < m) {
                            x[c][q] = fma(-f, vr[q], x[c][q]);
                            cj[c][r] = x[c][q];
                        }
                    }
                } else {
                    for (int r = i + 1 + lane; r < m; r += 32) cj[c][r] -= f * v[r];
                }
                cji[c] -= f;
                if (lane == 0) cj[c][i] = cji[c];
            }
        }
        bool redo[CB], any_redo = false;
        double nv1[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            redo[c] = false;
            nv1[c] = -1.0;
            if (!on[c]) continue;
            const double v1 = vn1[phys[c]];
            if (v1 == 0.0) continue;
            double temp = fabs(cji[c]) / v1;
            temp = 1.0 - temp * temp;
            temp = temp < 0.0 ? 0.0 : temp;
            const double ratio = v1 / vn2[phys[c]];
            const double temp2 = temp * ratio * ratio;
            if (temp2 <= TOL3Z) redo[c] = any_redo = true;
            else nv1[c] = v1 * sqrt(temp);
        }
        if (any_redo) {  // uniform across the warp
            __syncwarp();
            double nv[CB];
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                nv[c] = 0.0;
                if (!redo[c]) continue;
                if (RPL > 0) {
#pragma unroll
                    for (int q = 0; q < R; ++q) {
                        const int r = lane + 32 * q;
                        if (r > i && r < m) nv[c] = fma(x[c][q], x[c][q], nv[c]);
                    }
                } else {
                    for (int r = i + 1 + lane; r < m; r += 32) nv[c] += cj[c][r] * cj[c][r];
                }
            }
            warp_sum4(nv);
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                if (!redo[c]) continue;
                const double x2 = (i + 1 < m) ? sqrt(nv[c]) : 0.0;
                if (lane < C) {
                    cl.map_shared_rank(vn1, lane)[phys[c]] = x2;
                    cl.map_shared_rank(vn2, lane)[phys[c]] = x2;
                }
            }
        }
#pragma unroll
        for (int c = 0; c < CB; ++c)
            if (nv1[c] >= 0.0 && lane < C) cl.map_shared_rank(vn1, lane)[phys[c]] = nv1[c];
        __syncwarp();
    }
}

// RPL > 0: m <= 32 RPL (rows unrolled); 0: any m.  Columns are dealt cyclically to
// the CTAs of the cluster (physical column j -> CTA j mod C), so the pivoting, which
// retires columns in data order, keeps the CTAs' remaining work balanced.
template <bool TIMING, int RPL>
__global__ void __launch_bounds__(CT) qrcp_cluster_kernel(const __grid_constant__ QcArgs a) {
    namespace cg = cooperative_groups;
    long long tp = TIMING ? clock64() : 0;
    auto mark = [&](int ph) {
        if (TIMING && threadIdx.x == 0 && blockIdx.x == 0) {
            const long long now = clock64();
            atomicAdd(&qc_phase_cycles[ph], (unsigned long long)(now - tp));
            tp = now;
        }
    };
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[32];
    __shared__ int piv_s;
    const int C = a.C;
    const int g = blockIdx.x / C;
    const int lb = (int)cl.block_rank();
    const MatDesc &d = a.d[g];
    const Ws w = carve(d);
    const int m = d.m, k = d.k, ldw = d.ldw, cpc = d.cpc;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = CT / 32;
    const int nloc = (k - lb + C - 1) / C;  // owned columns: lb, lb + C, ...
    double *cols = sm;
    double *v = cols + (size_t)cpc * ldw;
    double *vn1 = v + m, *vn2 = vn1 + k, *tau = vn2 + k, *diagR = tau + k;
    int *pos2phys = reinterpret_cast<int *>(diagR + k);
    int *posof = pos2phys + k;

    for (long long e = t; e < (long long)m * nloc; e += CT) {
        const int r = (int)(e / nloc), jl = (int)(e % nloc);
        cols[(long long)jl * ldw + r] = d.G[(long long)r * d.ldg + lb + C * jl];
    }
    for (int j = t; j < k; j += CT) { pos2phys[j] = j; posof[j] = j; }
    cl.sync();  // every CTA of the cluster is running before any DSMEM store
    for (int jl = warp; jl < nloc; jl += nw) {
        const double *cj = cols + (long long)jl * ldw;
        double s = 0.0;
        for (int r = lane; r < m; r += 32) s += cj[r] * cj[r];
        s = sqrt(warp_sum(s));
        if (lane < C) {
            cl.map_shared_rank(vn1, lane)[lb + C * jl] = s;
            cl.map_shared_rank(vn2, lane)[lb + C * jl] = s;
        }
    }
    cl.sync();

    const int kmin = m < k ? m : k;
    for (int i = 0; i < kmin; ++i) {
        // 1. pivot from the local replica of the norms (identical in every CTA)
        if (warp == 0) {
            double best = -1.0;
            int bp = k;
            for (int j = i + lane; j < k; j += 32) {
                const double vv = vn1[pos2phys[j]];
                if (vv > best) { best = vv; bp = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
            }
            if (lane == 0) {
                if (bp >= k) bp = i;  // NaN norms (failed upstream pivot): keep the order
                const int ci = pos2phys[i], cp = pos2phys[bp];
                pos2phys[i] = cp; pos2phys[bp] = ci;
                posof[cp] = i; posof[ci] = bp;
                piv_s = cp;
            }
        }
        __syncthreads();
        mark(0);
        const int pc = piv_s;
        // 2. the owner forms the reflector (dlarfg) and pushes it to every CTA
        if (pc % C == lb) {
            double *ci = cols + (long long)(pc / C) * ldw;
            double part = 0.0;
            for (int r = i + 1 + t; r < m; r += CT) part += ci[r] * ci[r];
            const double xnorm = sqrt(block_sum(part, red));
            const double alpha = ci[i];
            double tau_i = 0.0, beta = alpha, scal = 0.0;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau_i = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
            }
            __syncthreads();
            for (int r = i + 1 + t; r < m; r += CT) {
                const double x = (xnorm != 0.0) ? ci[r] * scal : ci[r];
                ci[r] = x;
                for (int q = 0; q < C; ++q) cl.map_shared_rank(v, q)[r] = x;
            }
            if (t < C) {
                cl.map_shared_rank(tau, t)[i] = tau_i;
                cl.map_shared_rank(diagR, t)[i] = beta;
            }
            if (t == 0) ci[i] = beta;
        }
        mark(1);
        cl.sync();
        mark(2);
        // 3. apply H_i^T to the unchosen owned columns, downdate and push their norms
        const long long tw0 = TIMING ? clock64() : 0;
        qc_update<RPL, 4>(cl, C, i, m, k, ldw, lb, nloc, cols, v, tau[i], vn1, vn2, posof, warp, lane, nw);
        if (TIMING && lane == 0 && blockIdx.x < 2)
            atomicAdd(&qc_phase_cycles[8 + 8 * blockIdx.x + warp], (unsigned long long)(clock64() - tw0));
        mark(3);
        cl.sync();
        mark(4);
    }
    // spill the reflector columns, the permutation, tau and R's diagonal to the
    // workspace the Q formation reads
    for (long long e = t; e < (long long)ldw * nloc; e += CT) {
        const int jl = (int)(e / ldw), r = (int)(e % ldw);
        w.cols[(long long)(lb + C * jl) * ldw + r] = cols[e];
    }
    if (lb == 0) {
        for (int j = t; j < k; j += CT) {
            w.perm[j] = pos2phys[j];
            w.vn1[j] = vn1[j];
            w.vn2[j] = vn2[j];
        }
        for (int j = t; j < kmin; j += CT) {
            w.tau[j] = tau[j];
            w.diagR[j] = diagR[j];
        }
    }
}

struct QDesc {
    double *W;
    double *Q;
    int *rank;
    int m, k, ldw, ldq, blk0, nblk, wpc;
};

struct QArgs {
    int count;
    QDesc d[MAXM];
};

// Q[:, j] = H_0 ... H_j e_j for j < rank; one warp per output column (in smem);
// also publishes the kept rank (kernels.py:78-81)
__global__ void __launch_bounds__(CT) mq_form_q_kernel(const __grid_constant__ QArgs a) {
    extern __shared__ __align__(16) double qcol[];
    int g = 0;
    while (g + 1 < a.count && (int)blockIdx.x >= a.d[g + 1].blk0) ++g;
    const QDesc &d = a.d[g];
    const int m = d.m, k = d.k, ldw = d.ldw;
    const double *W = d.W;
    const double *vn1 = W + (long long)ldw * k;
    const double *tau = vn1 + 2 * k;
    const double *diagR = tau + k;
    const int *perm = reinterpret_cast<const int *>(diagR + k + m);
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
        if (blockIdx.x == d.blk0) *d.rank = r;
    }
    __syncthreads();
    const int rank = rank_s;
    if (warp >= d.wpc) return;
    const int j = (blockIdx.x - d.blk0) * d.wpc + warp;
    if (j >= rank) return;
    double *q = qcol + (long long)warp * m;
    for (int r = lane; r < m; r += 32) q[r] = (r == j) ? 1.0 : 0.0;
    __syncwarp();
    for (int i = j; i >= 0; --i) {
        const double *vi = W + (long long)perm[i] * ldw;  // v_i[i] = 1 implicitly
        const double ti = tau[i];
        double s = 0.0;
        for (int r = i + 1 + lane; r < m; r += 32) s += vi[r] * q[r];
        s = warp_sum(s) + q[i];
        const double f = ti * s;
        __syncwarp();
        for (int r = i + 1 + lane; r < m; r += 32) q[r] -= f * vi[r];
        if (lane == 0) q[i] -= f;
        __syncwarp();
    }
    for (int r = lane; r < m; r += 32) d.Q[(long long)r * d.ldq + j] = q[r];
}

// ---- blocked (compact-WY) Q formation, dorgqr-style, on DMMA GEMMs ----------
// Q = H_0 ... H_{k-1} [I; 0] = B_0 (B_1 ( ... B_last [I;0])), B_b = I - V_b T_b V_b^T
// over blocks of QB reflectors; V_b is the explicit unit-lower reflector block and
// T_b the dlarft triangle.  Applying every reflector (not only the first `rank`)
// leaves Q[:, :rank] exactly unchanged (reflector i acts on rows >= i, where the
// first columns are still zero).
constexpr int QB = 64;

struct VBuild {
    int count;
    const double *W[MAXM];
    const int *perm[MAXM];
    double *V[MAXM];
    double *Q[MAXM];
    int m[MAXM], kmin[MAXM], ldw[MAXM], ldq[MAXM];
};

// V[r, i] = (r < i ? 0 : r == i ? 1 : W[perm[i]][r]);  Q[r, i] = (r == i)
// 32x32 tiles through shared memory (coalesced column-major read, row-major write)
__global__ void build_vq_kernel(const __grid_constant__ VBuild a) {
    __shared__ double tile[32][33];
    const int g = blockIdx.z;
    const int m = a.m[g], km = a.kmin[g];
    const int r0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    if (r0 >= m || i0 >= km) return;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    for (int q = ty; q < 32; q += 8) {
        const int i = i0 + q, r = r0 + tx;
        double v = 0.0;
        if (i < km && r < m) v = (r < i) ? 0.0 : (r == i ? 1.0 : a.W[g][(long long)a.perm[g][i] * a.ldw[g] + r]);
        tile[q][tx] = v;
    }
    __syncthreads();
    for (int q = ty; q < 32; q += 8) {
        const int r = r0 + q, i = i0 + tx;
        if (r < m && i < km) {
            a.V[g][(long long)r * km + i] = tile[tx][q];
            a.Q[g][(long long)r * a.ldq[g] + i] = (r == i) ? 1.0 : 0.0;
        }
    }
}

struct TArgs {
    int count, nbk;           // matrices, blocks per matrix (CTA = matrix * nbk + block)
    const double *G[MAXM];    // Gram of every block (nbk x QB x QB, ld QB)
    const double *tau[MAXM];
    double *T[MAXM];          // nbk x QB x QB, ld QB
    int kmin[MAXM];
};

// dlarft (forward, columnwise) for one QB = 64 block: the T of I - V T V^T.
// Blocked: the four 16-column diagonal blocks run the column recurrence
// T[0:i, i] = -tau_i T[0:i, 0:i] G[0:i, i] concurrently (one warp each), then the
// off-diagonal blocks are joined pairwise, T12 = -T11 (G12 T22) (the product of two
// compact-WY blocks: (I - V1 T11 V1^T)(I - V2 T22 V2^T)), 16 -> 32 -> 64.
// G = V^T V (QB x QB).  One shared array holds T in its upper triangle and G's
// strict upper triangle transposed into its strict lower triangle (M[y][x] = G[x][y],
// x < y); one CTA of 256 threads per matrix.
__global__ void __launch_bounds__(256) larft_kernel(const __grid_constant__ TArgs a) {
    __shared__ double M[QB][QB + 1];
    __shared__ double X[QB * QB / 4];  // G12 T22 of the pairs being joined
    const int g = blockIdx.x / a.nbk, bb = blockIdx.x % a.nbk;
    const int j0 = bb * QB;
    const int nb = min(QB, a.kmin[g] - j0);
    if (nb <= 0) return;
    double *T = a.T[g] + (long long)bb * QB * QB;
    const double *G = a.G[g] + (long long)bb * QB * QB;
    const double *tau = a.tau[g] + j0;
    const int t = threadIdx.x;
    for (int e = t; e < QB * QB; e += blockDim.x) {
        const int r = e / QB, c = e % QB;
        M[r][c] = (r > c && r < nb) ? G[c * QB + r] : 0.0;
    }
    __syncthreads();
    // 1. diagonal 16-blocks, one warp each (lane = row within the block)
    constexpr int L = 16;
    {
        const int blk = t >> 5, r = t & 31;
        const int b0 = blk * L;
        if (blk < QB / L)
            for (int i = 0; i < L; ++i) {
                const int ci = b0 + i;
                if (ci < nb) {
                    if (r < i) {
                        double s = 0.0;
                        for (int l = r; l < i; ++l) s += M[b0 + r][b0 + l] * M[ci][b0 + l];
                        M[b0 + r][ci] = -tau[ci] * s;
                    }
                    if (r == i) M[ci][ci] = tau[ci];
                }
                __syncwarp();
            }
    }
    __syncthreads();
    // 2. join: block size h = 16, then 32; pair p has T11 at b0 = 2hp, T22 at b1 = b0 + h
    for (int h = L; h < QB; h *= 2) {
        const int work = (QB / (2 * h)) * h * h;
        for (int e = t; e < work; e += blockDim.x) {  // X = G12 T22
            const int pr = e / (h * h), r = (e / h) % h, c = e % h;
            const int b0 = pr * 2 * h, b1 = b0 + h;
            double s = 0.0;
            for (int l = 0; l <= c; ++l) s += M[b1 + l][b0 + r] * M[b1 + l][b1 + c];
            X[e] = s;
        }
        __syncthreads();
        for (int e = t; e < work; e += blockDim.x) {  // T12 = -T11 X
            const int pr = e / (h * h), r = (e / h) % h, c = e % h;
            const int b0 = pr * 2 * h, b1 = b0 + h;
            const double *Xp = X + pr * h * h;
            double s = 0.0;
            for (int l = r; l < h; ++l) s += M[b0 + r][b0 + l] * Xp[l * h + c];
            M[b0 + r][b1 + c] = -s;
        }
        __syncthreads();
    }
    for (int e = t; e < QB * QB; e += blockDim.x) {
        const int r = e / QB, c = e % QB;
        T[e] = (r <= c && c < nb) ? M[r][c] : 0.0;
    }
}

struct RankArgs {
    int count;
    const double *diagR[MAXM];
    int *rank[MAXM];
    int m[MAXM], k[MAXM];
};

__global__ void rank_kernel(const __grid_constant__ RankArgs a) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= a.count) return;
    const int m = a.m[g], k = a.k[g];
    const double *d = a.diagR[g];
    const double d0 = fabs(d[0]);
    const int kmin = m < k ? m : k;
    int r = 0;
    if (d0 != 0.0) {
        const double cut = (double)(m > k ? m : k) * EPS * d0;
        for (int i = 0; i < kmin; ++i)
            if (fabs(d[i]) > cut) ++r;
    }
    *a.rank[g] = r;
}

inline size_t smem_for(int m, int k, int cpc) {
    const size_t ldw = (size_t)(m | 1);
    return (size_t)cpc * ldw * 8 + (size_t)m * 8 + sizeof(int) * 2 * (size_t)k + 16 * (size_t)cpc;
}

}  // namespace

// workspace doubles of one matrix
long long rsc_qrcp_coop_doubles(int m, int k) {
    const long long ldw = m | 1;
    const long long kmin = m < k ? m : k;
    // factorization | explicit V (m x kmin) | W_b (QB x kmin) | Gram, T (QB x QB each)
    static_assert(QB == QB_WY, "candidate region offset assumes the WY block size");
    (void)kmin;
    // ... then the double-buffered pivot candidates and candidate columns
    // ... and the Gram and T triangles of every 64-reflector block (Q formation)
    const long long nbk = (kmin + QB - 1) / QB;
    return coop_cand_base(m, k) + 4LL * CQ_MAX + 2LL * (k < CQ_MAX ? k : CQ_MAX) * ldw + 2LL * nbk * QB * QB;
}

// per-block Gram / T region of a matrix's workspace (rsc_qrcp_coop_doubles)
static inline double *gt_base(double *W, int m, int k) {
    const long long ldw = m | 1;
    return W + coop_cand_base(m, k) + 4LL * CQ_MAX + 2LL * (k < CQ_MAX ? k : CQ_MAX) * ldw;
}

static inline double *wy_base(double *W, int m, int k) {
    const long long ldw = m | 1;
    return W + ldw * k + 4LL * k + m + k + 2 * CQ_MAX + 64;
}

int rsc_gemm_grouped(int transA, int transB, const rsc_gemm_problem *problems, int count, void *stream);

static inline rsc_gemm_problem gp(const double *A, int lda, const double *B, int ldb, double *C, int ldc, int M,
                                  int N, int K, double alpha, double beta) {
    rsc_gemm_problem p{};
    p.A = A; p.B = B; p.C = C; p.lda = lda; p.ldb = ldb; p.ldc = ldc;
    p.M = M; p.N = N; p.K = K; p.alpha = alpha; p.beta = beta; p.batch = 1;
    return p;
}

// Q for the matrices of one launch group: ranks, explicit V, then per block b (from
// the last): Gram = V_b^T V_b, T_b (dlarft), W = V_b^T Q_b, W = T_b W, Q_b -= V_b W.
static int form_q_blocked(int cnt, const MatDesc *ds, cudaStream_t s) {
    static thread_local RankArgs ra;
    static thread_local VBuild vb;
    static thread_local TArgs ta;
    ra.count = cnt;
    vb.count = cnt;
    int maxm = 1, maxk = 1;
    for (int c = 0; c < cnt; ++c) {
        const MatDesc &d = ds[c];
        const Ws w = {d.W, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        (void)w;
        double *diagR = d.W + (long long)d.ldw * d.k + 3LL * d.k;
        double *vbuf = diagR + d.k;
        const int *perm = reinterpret_cast<const int *>(vbuf + d.m);
        const int kmin = d.m < d.k ? d.m : d.k;
        ra.diagR[c] = diagR; ra.rank[c] = d.rank; ra.m[c] = d.m; ra.k[c] = d.k;
        vb.W[c] = d.W; vb.perm[c] = perm; vb.V[c] = wy_base(d.W, d.m, d.k); vb.Q[c] = d.Q;
        vb.m[c] = d.m; vb.kmin[c] = kmin; vb.ldw[c] = d.ldw; vb.ldq[c] = d.ldq;
        maxm = d.m > maxm ? d.m : maxm;
        maxk = kmin > maxk ? kmin : maxk;
    }
    rank_kernel<<<(cnt + 127) / 128, 128, 0, s>>>(ra);
    RSC_CHECK_LAUNCH();
    dim3 grid((maxm + 31) / 32, (maxk + 31) / 32, cnt);
    build_vq_kernel<<<grid, 256, 0, s>>>(vb);
    RSC_CHECK_LAUNCH();
    const int nblocks = (maxk + QB - 1) / QB;
    // Gram V_b^T V_b of every block of every matrix in ONE grouped launch (V is final
    // before the Q formation starts), then every block's T in ONE dlarft launch; only
    // the Q updates (W = V_b^T Q_b, W = T_b W, Q_b -= V_b W) stay a sequence over the
    // blocks, last to first.  The long K (= rows) of the two V^T products is cut into
    // KS-row slabs summed by the ordered accumulation, so each output tile gets
    // rows / KS CTAs and a short k-loop.
    constexpr int KS = 128;
    std::vector<rsc_gemm_problem> pg, pw, pt, pq;
    ta.count = cnt;
    ta.nbk = nblocks;
    for (int c = 0; c < cnt; ++c) {
        const MatDesc &d = ds[c];
        const int km = vb.kmin[c];
        double *V = vb.V[c];
        double *GT = gt_base(d.W, d.m, d.k);
        const int nbk = (km + QB - 1) / QB;
        double *Gall = GT, *Tall = GT + (long long)nbk * QB * QB;
        ta.G[c] = Gall; ta.T[c] = Tall; ta.kmin[c] = km;
        ta.tau[c] = d.W + (long long)d.ldw * d.k + 2LL * d.k;
        cudaMemsetAsync(Gall, 0, sizeof(double) * (size_t)nbk * QB * QB, s);
        for (int b = 0; b < nbk; ++b) {
            const int j0 = b * QB, nb = km - j0 < QB ? km - j0 : QB, rows = d.m - j0;
            const double *Vb = V + (long long)j0 * km + j0;
            for (int k0 = 0; k0 < rows; k0 += KS) {
                const int kk = rows - k0 < KS ? rows - k0 : KS;
                const double *Vk = Vb + (long long)k0 * km;
                rsc_gemm_problem a = gp(Vk, km, Vk, km, Gall + (long long)b * QB * QB, QB, nb, nb, kk, 1.0, 1.0);
                a.atomic = 1;
                pg.push_back(a);
            }
        }
    }
    if (!pg.empty()) {
        int rc = rsc_gemm_grouped(1, 0, pg.data(), (int)pg.size(), s);
        if (rc) return rc;
        larft_kernel<<<cnt * nblocks, 256, 0, s>>>(ta);
        RSC_CHECK_LAUNCH();
    }
    for (int b = nblocks - 1; b >= 0; --b) {
        pw.clear(); pt.clear(); pq.clear();
        const int j0 = b * QB;
        for (int c = 0; c < cnt; ++c) {
            const MatDesc &d = ds[c];
            const int km = vb.kmin[c];
            if (j0 >= km) continue;
            double *V = vb.V[c];
            double *Wb = V + (long long)d.m * km;
            const double *Tm = ta.T[c] + (long long)b * QB * QB;
            const int nb = km - j0 < QB ? km - j0 : QB;
            const int rows = d.m - j0, cols = km - j0;
            const double *Vb = V + (long long)j0 * km + j0;
            double *Qb = d.Q + (long long)j0 * d.ldq + j0;
            cudaMemsetAsync(Wb, 0, sizeof(double) * (size_t)QB * km, s);
            for (int k0 = 0; k0 < rows; k0 += KS) {
                const int kk = rows - k0 < KS ? rows - k0 : KS;
                const double *Vk = Vb + (long long)k0 * km;
                rsc_gemm_problem w = gp(Vk, km, Qb + (long long)k0 * d.ldq, d.ldq, Wb, km, nb, cols, kk, 1.0, 1.0);
                w.atomic = 1;                                                              // W = V^T Q (TA)
                pw.push_back(w);
            }
            pt.push_back(gp(Tm, QB, Wb, km, Wb, km, nb, cols, nb, 1.0, 0.0));           // W = T W (in place)
            pq.push_back(gp(Vb, km, Wb, km, Qb, d.ldq, rows, cols, nb, -1.0, 1.0));    // Q -= V W
        }
        if (pw.empty()) continue;
        int rc;
        if ((rc = rsc_gemm_grouped(1, 0, pw.data(), (int)pw.size(), s))) return rc;
        if ((rc = rsc_gemm_grouped(0, 0, pt.data(), (int)pt.size(), s))) return rc;
        if ((rc = rsc_gemm_grouped(0, 0, pq.data(), (int)pq.size(), s))) return rc;
    }
    return 0;
}

// Factor `n` matrices (indices into the arrays) concurrently.  work_off[i] is the
// byte offset of matrix i's workspace in `work`; bar has >= n zeroable counters.
int rsc_qrcp_multi(int n, const int *ids, double *const *G, const int *m, const int *k, const int *ldg,
                   double *const *Q, const int *ldq, int *rank_dev, char *work, const long long *work_off,
                   unsigned *bar, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    nsm = std::min(nsm, CQ_MAX);  // a group never has more CTAs than pivot-candidate slots
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(mqrcp_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BUDGET + 8192);
        cudaFuncSetAttribute(mqrcp_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BUDGET + 8192);
        cudaFuncSetAttribute(mqrcp_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BUDGET + 8192);
        cudaFuncSetAttribute(mq_form_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BUDGET);
        attr = true;
    }
    // per-matrix plan: fewest CTAs whose owned columns fit shared memory
    struct P { int i, cpc, nblk; bool smem; size_t sm; };
    std::vector<P> plans;
    for (int t = 0; t < n; ++t) {
        const int i = ids[t];
        if (m[i] <= 0 || k[i] <= 0) continue;
        const size_t fixed = (size_t)m[i] * 8 + sizeof(int) * 2 * (size_t)k[i];
        const size_t per_col = (size_t)(m[i] | 1) * 8 + 16;  // column + its two partial norms
        int cpc = fixed < SMEM_BUDGET ? (int)((SMEM_BUDGET - fixed) / per_col) : 0;
        if (cpc >= 1) {
            cpc = std::min(cpc, k[i]);
            const int nblk = (k[i] + cpc - 1) / cpc;
            if (nblk <= nsm) {
                plans.push_back({i, cpc, nblk, true, smem_for(m[i], k[i], cpc)});
                continue;
            }
        }
        cpc = (k[i] + nsm - 1) / nsm;  // global-memory columns, one group over all SMs
        // the reflector is staged in shared memory when it fits (vsm)
        const size_t base = sizeof(int) * 2 * (size_t)k[i] + 16 * (size_t)cpc;
        const size_t gsm = (size_t)m[i] * 8 + base;
        plans.push_back({i, cpc, (k[i] + cpc - 1) / cpc, false, gsm <= SMEM_BUDGET ? gsm : base});
    }
    // sketches that fit one thread-block cluster: cluster kernel (DSMEM + hardware
    // cluster barriers); the rest stays on the cooperative kernel
    {
        static bool cattr = false;
        if (!cattr) {
            for (void *f : {(void *)qrcp_cluster_kernel<false, 0>, (void *)qrcp_cluster_kernel<true, 0>,
                            (void *)qrcp_cluster_kernel<false, 8>, (void *)qrcp_cluster_kernel<true, 8>,
                            (void *)qrcp_cluster_kernel<false, 16>, (void *)qrcp_cluster_kernel<true, 16>}) {
                cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
                cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            }
            cattr = true;
        }
        static thread_local QcArgs qc;
        std::vector<std::pair<int, int>> cl_list;  // (C, plan index)
        std::vector<size_t> cl_sm(plans.size(), 0);
        std::vector<char> done(plans.size(), 0);
        if (!getenv("RSC_QR_NOCLUSTER")) {
            // smallest cluster whose shared memory holds the sketch, widened so the
            // batch's clusters cover the SMs (fewer owned columns per CTA)
            std::vector<int> cmin(plans.size(), 0);
            int neligible = 0;
            for (size_t pi = 0; pi < plans.size(); ++pi) {
                const int i = plans[pi].i;
                for (int C = 2; C <= QC_MAXC && C <= k[i]; ++C)
                    if (cluster_smem(m[i], k[i], (k[i] + C - 1) / C) <= 220 * 1024) { cmin[pi] = C; break; }
                if (cmin[pi]) ++neligible;
            }
            // (widening the clusters to cover all SMs measured slower: more DSMEM
            // pushes and cluster-barrier participants per column)
            const int cwide = 0;
            (void)neligible;
            for (size_t pi = 0; pi < plans.size(); ++pi) {
                if (!cmin[pi]) continue;
                const int i = plans[pi].i;
                const int chi = std::max(cmin[pi], std::min(cwide, k[i] / 4));
                for (int C = chi; C >= cmin[pi]; --C) {
                    const int cpc = (k[i] + C - 1) / C;
                    const size_t smb = cluster_smem(m[i], k[i], cpc);
                    cudaLaunchConfig_t cfg = {};
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    cfg.gridDim = dim3(C);
                    cfg.blockDim = dim3(CT);
                    cfg.dynamicSmemBytes = smb;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    // occupancy queries cost tens of microseconds of host time: memoized
                    // per (cluster size, shared memory bytes)
                    static std::map<std::pair<int, size_t>, int> occ_cl;
                    static std::mutex occ_mu;
                    int ncl = 0;
                    {
                        std::lock_guard<std::mutex> lk(occ_mu);
                        auto it = occ_cl.find({C, smb});
                        if (it != occ_cl.end()) {
                            ncl = it->second;
                        } else {
                            if (cudaOccupancyMaxActiveClusters(&ncl, (void *)qrcp_cluster_kernel<false, 0>, &cfg) !=
                                cudaSuccess) {
                                cudaGetLastError();
                                ncl = 0;
                            }
                            occ_cl[{C, smb}] = ncl;
                        }
                    }
                    if (ncl < 1) continue;
                    cl_list.push_back({C, (int)pi});
                    cl_sm[pi] = smb;
                    done[pi] = 1;
                    break;
                }
            }
        }
        std::sort(cl_list.begin(), cl_list.end());
        size_t pos = 0;
        while (pos < cl_list.size()) {
            const int C = cl_list[pos].first;
            int cnt = 0;
            size_t smb = 0;
            while (pos < cl_list.size() && cl_list[pos].first == C && cnt < MAXM) {
                const P &p = plans[cl_list[pos].second];
                const int i = p.i;
                MatDesc &d = qc.d[cnt];
                d.G = G[i]; d.Q = Q[i];
                d.W = reinterpret_cast<double *>(work + work_off[i]);
                d.rank = rank_dev + i;
                d.m = m[i]; d.k = k[i]; d.ldg = ldg[i]; d.ldq = ldq[i]; d.ldw = m[i] | 1;
                d.cpc = (k[i] + C - 1) / C; d.nblk = C; d.blk0 = cnt * C;
                smb = std::max(smb, cl_sm[cl_list[pos].second]);
                ++cnt;
                ++pos;
            }
            qc.count = cnt;
            qc.C = C;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(cnt * C);
            cfg.blockDim = dim3(CT);
            cfg.dynamicSmemBytes = smb;
            cfg.stream = s;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            static const bool timing = getenv("RSC_QR_TIMING") != nullptr;
            int maxm = 0;
            for (int c = 0; c < cnt; ++c) maxm = std::max(maxm, qc.d[c].m);
            cudaError_t e;
            if (maxm <= 256)
                e = timing ? cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<true, 8>, qc)
                           : cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<false, 8>, qc);
            else if (maxm <= 512)
                e = timing ? cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<true, 16>, qc)
                           : cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<false, 16>, qc);
            else
                e = timing ? cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<true, 0>, qc)
                           : cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel<false, 0>, qc);
            rsc_count_launch();
            if (e != cudaSuccess) return (int)e;
            const int rc = form_q_blocked(cnt, qc.d, s);
            if (rc) return rc;
        }
        std::vector<P> rest;
        for (size_t pi = 0; pi < plans.size(); ++pi)
            if (!done[pi]) rest.push_back(plans[pi]);
        plans.swap(rest);
    }
    cudaMemsetAsync(bar, 0, sizeof(unsigned) * (size_t)std::max(n, 1), s);
    static thread_local MArgs ma;
    static thread_local QArgs qa;
    for (int pass = 0; pass < 2; ++pass) {
        const bool smem = pass == 0;
        size_t pos = 0;
        std::vector<P> sel;
        for (auto &p : plans)
            if (p.smem == smem) sel.push_back(p);
        while (pos < sel.size()) {
            // pack groups while they fit co-resident
            size_t sm = 0;
            int blocks = 0, cnt = 0;
            size_t start = pos;
            // global-memory columns: the two-CTAs-per-SM build when at least two sketches are left
            const bool pair = !smem && sel.size() - pos >= 2;
            void *kfn = smem ? (void *)mqrcp_kernel<true, 1>
                             : pair ? (void *)mqrcp_kernel<false, 2> : (void *)mqrcp_kernel<false, 1>;
            const int kid = smem ? 1 : pair ? 2 : 0;
            while (pos < sel.size() && cnt < MAXM) {
                const size_t sm2 = std::max(sm, sel[pos].sm);
                static std::map<std::pair<int, size_t>, int> occ_b;
                static std::mutex occ_bmu;
                int per_sm = 0;
                {
                    std::lock_guard<std::mutex> lk(occ_bmu);
                    auto it = occ_b.find({kid, sm2});
                    if (it != occ_b.end()) {
                        per_sm = it->second;
                    } else {
                        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, MCT, sm2);
                        occ_b[{kid, sm2}] = per_sm;
                    }
                }
                if (per_sm < 1) return 77;
                if (cnt > 0 && blocks + sel[pos].nblk > nsm * per_sm) break;
                sm = sm2;
                blocks += sel[pos].nblk;
                ++cnt;
                ++pos;
            }
            ma.count = cnt;
            ma.bar = bar;
            int b0 = 0;
            for (int c = 0; c < cnt; ++c) {
                const P &p = sel[start + c];
                const int i = p.i;
                MatDesc &d = ma.d[c];
                d.G = G[i]; d.Q = Q[i];
                d.W = reinterpret_cast<double *>(work + work_off[i]);
                d.rank = rank_dev + i;
                d.m = m[i]; d.k = k[i]; d.ldg = ldg[i]; d.ldq = ldq[i]; d.ldw = m[i] | 1;
                d.cpc = p.cpc; d.nblk = p.nblk; d.blk0 = b0;
                d.vsm = !smem && p.sm > sizeof(int) * 2 * (size_t)k[i] + 16 * (size_t)p.cpc;
                b0 += p.nblk;
            }
            // distinct barrier counter per matrix of this launch
            ma.bar = bar + start + (smem ? 0 : 0);
            void *args[] = {&ma};
            cudaError_t e = cudaLaunchCooperativeKernel(kfn, dim3(b0), dim3(MCT), args, sm, s);
            rsc_count_launch();
            if (e != cudaSuccess) return (int)e;
            // Q formation (blocked compact-WY on DMMA GEMMs) for the same matrices
            {
                const int rc = form_q_blocked(cnt, ma.d, s);
                if (rc) return rc;
            }
        }
        // second pass uses fresh counters beyond the first pass's
        if (pass == 0) {
            bar += sel.size();
        }
    }
    return 0;
}

extern "C" int rsc_qr_phase_cycles(unsigned long long *out8, int reset) {
    cudaError_t e = cudaMemcpyFromSymbol(out8, qc_phase_cycles, 32 * sizeof(unsigned long long));
    if (reset) {
        unsigned long long z[32] = {};
        cudaMemcpyToSymbol(qc_phase_cycles, z, sizeof(z));
    }
    return (int)e;
}
