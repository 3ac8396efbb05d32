// Batched column-pivoted Householder QR (LAPACK dgeqp3/dlaqp2 semantics) with the
// reference rank cutoff and explicit Q (dorg2r) for the kept columns.
//
// Reference: kernels.py:67-82 orthonormalize ->
//   Q, R, _ = scipy.linalg.qr(G, mode="economic", pivoting=True)
//   rank = #{ |R_ii| > max(m,k) * eps * |R_00| };  return Q[:, :rank]
// The kept count is decided by |R_ii| sitting as close as 1% to the cutoff, so the
// pivot rule (first index of the largest partial norm), the Householder convention
// (dlarfg: beta = -sign(alpha) * ||x||) and the partial-norm downdating with the
// sqrt(eps) recomputation threshold (dlaqp2) are reproduced, in FP64 throughout.
// Q[:, :rank] only depends on the first `rank` reflectors (H_i e_j = e_j for i > j),
// so dorg2r is run on those only.
//
// One CTA per matrix.  The sketch is transposed into a column-major tile so every
// Householder step is warp-per-column with coalesced, conflict-free access; the tile
// lives in shared memory when it fits (cfg1: 256 x 58) and otherwise in a global
// (L2-resident) workspace.
#include <vector>
#include "common.cuh"

namespace {

constexpr int QR_THREADS = 512;
constexpr int QR_MAXK = 1024;
constexpr int MAXB = 600;  // one launch covers a whole config[1] batch (single partial wave)
constexpr double EPS = 2.220446049250313e-16;        // np.finfo(float64).eps
constexpr double TOL3Z = 1.0536712127723509e-08;     // sqrt(dlamch('E')) = sqrt(2^-53)

struct QrArgs {
    int count;
    double *G[MAXB];
    double *Q[MAXB];
    long long woff[MAXB];
    int m[MAXB], k[MAXB], ldg[MAXB], ldq[MAXB];
    int base;
};

__device__ __forceinline__ double col_norm2(const double *c, int r0, int m, int lane) {
    double s = 0.0;
    for (int r = r0 + lane; r < m; r += 32) s += c[r] * c[r];
    return warp_sum(s);
}

// One CTA per matrix.  Pivoting is a permutation (pos2phys / posof) instead of
// column swaps, and each Householder step is two phases separated by a single CTA
// barrier: (1) warp 0 picks the pivot (first position of the largest partial norm),
// forms the reflector on that column and publishes tau; (2) every warp applies it to
// its own unchosen columns and downdates their norms.  dorg2r runs on the first
// `rank` positions with the same indirection.
template <bool SMEM, int RPL>
__global__ void __launch_bounds__(QR_THREADS) qrcp_kernel(const __grid_constant__ QrArgs args,
                                                           double *work, int *rank_out) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ int piv_s, rank_s;

    const int b = blockIdx.x;
    const int m = args.m[b], k = args.k[b];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5, nw = QR_THREADS / 32;
    const int ldw = m | 1;  // odd column stride: conflict-free transposed load
    double *W = SMEM ? dyn : work + args.woff[b];
    double *vn1 = SMEM ? dyn + (long long)ldw * k : dyn;
    double *vn2 = vn1 + k, *tau = vn2 + k, *diagR = tau + k;
    int *pos2phys = reinterpret_cast<int *>(diagR + k);
    int *posof = pos2phys + k;
    const double *G = args.G[b];
    const int ldg = args.ldg[b];

    if (m == 0 || k == 0) {
        if (t == 0) rank_out[args.base + b] = 0;
        return;
    }
    for (long long e = t; e < (long long)m * k; e += QR_THREADS) {
        const int i = (int)(e / k), j = (int)(e % k);
        W[(long long)j * ldw + i] = G[(long long)i * ldg + j];
    }
    for (int j = t; j < k; j += QR_THREADS) { pos2phys[j] = j; posof[j] = j; }
    __syncthreads();
    for (int j = warp; j < k; j += nw) {
        const double nrm = sqrt(col_norm2(W + (long long)j * ldw, 0, m, lane));
        if (lane == 0) { vn1[j] = nrm; vn2[j] = nrm; }
    }
    __syncthreads();

    const int kmin = m < k ? m : k;
    for (int i = 0; i < kmin; ++i) {
        if (warp == 0) {
            // pivot: first position of the largest partial norm (idamax over positions)
            double best = -1.0;
            int bp = k;
            for (int j = i + lane; j < k; j += 32) {
                const double v = vn1[pos2phys[j]];
                if (v > best) { best = v; bp = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ob = __shfl_xor_sync(0xffffffffu, best, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
            }
            if (bp >= k) bp = i;  // NaN norms (failed upstream pivot): keep the order
            const int pc = pos2phys[bp];
            __syncwarp();
            if (lane == 0) {
                const int ci = pos2phys[i];
                pos2phys[i] = pc; pos2phys[bp] = ci;
                posof[pc] = i; posof[ci] = bp;
                piv_s = pc;
            }
            // reflector on the pivot column (dlarfg)
            double *cp = W + (long long)pc * ldw;
            const double xnorm = sqrt(col_norm2(cp, i + 1, m, lane));
            const double alpha = cp[i];
            double tau_i = 0.0, beta = alpha, scal = 0.0;
            if (xnorm != 0.0) {
                beta = -copysign(hypot(alpha, xnorm), alpha);
                tau_i = (beta - alpha) / beta;
                scal = 1.0 / (alpha - beta);
                for (int r = i + 1 + lane; r < m; r += 32) cp[r] *= scal;
            }
            __syncwarp();
            if (lane == 0) { cp[i] = beta; tau[i] = tau_i; diagR[i] = beta; }
        }
        __syncthreads();
        const int pc = piv_s;
        const double *ci = W + (long long)pc * ldw;
        const double tau_i = tau[i];
        // apply H^T to the unchosen columns (positions > i, round-robin over warps for
        // balance) and downdate their norms
        if constexpr (RPL > 0) {
            // m <= 32 RPL: the reflector is held in registers for every column of the
            // step, rows unrolled at compile time (same per-lane summation order)
            double vr[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int r = lane + 32 * q;
                vr[q] = (r > i && r < m) ? ci[r] : 0.0;
            }
            // four columns of the warp at a time, interleaved: their loads, dot
            // products, butterflies and downdates overlap instead of running back to back
            constexpr int CB = 4;
            for (int jp0 = i + 1 + warp; jp0 < k; jp0 += CB * nw) {
                int jj[CB];
                bool on[CB];
                double *cj[CB];
                double x[CB][RPL], cji[CB], w[CB];
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    const int jp = jp0 + c * nw;
                    on[c] = jp < k;
                    jj[c] = on[c] ? pos2phys[jp] : 0;
                    cj[c] = W + (long long)jj[c] * ldw;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) {
                        const int r = lane + 32 * q;
                        x[c][q] = (on[c] && r < m) ? cj[c][r] : 0.0;
                    }
                    cji[c] = on[c] ? cj[c][i] : 0.0;
                    w[c] = 0.0;
                }
                if (tau_i != 0.0) {
#pragma unroll
                    for (int c = 0; c < CB; ++c)
#pragma unroll
                        for (int q = 0; q < RPL; ++q) w[c] = fma(vr[q], x[c][q], w[c]);
                    warp_sum4(w);
#pragma unroll
                    for (int c = 0; c < CB; ++c) {
                        if (!on[c]) continue;
                        const double f = tau_i * (w[c] + cji[c]);
#pragma unroll
                        for (int q = 0; q < RPL; ++q) {
                            const int r = lane + 32 * q;
                            if (r > i && r < m) {
                                x[c][q] = fma(-f, vr[q], x[c][q]);
                                cj[c][r] = x[c][q];
                            }
                        }
                        cji[c] -= f;
                        if (lane == 0) cj[c][i] = cji[c];
                    }
                }
                bool redo[CB], any_redo = false;
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    redo[c] = false;
                    if (!on[c]) continue;
                    const double v1 = vn1[jj[c]];
                    if (v1 == 0.0) continue;
                    double temp = fabs(cji[c]) / v1;
                    temp = 1.0 - temp * temp;
                    temp = temp < 0.0 ? 0.0 : temp;
                    const double ratio = v1 / vn2[jj[c]];
                    const double temp2 = temp * ratio * ratio;
                    if (temp2 <= TOL3Z) {
                        redo[c] = any_redo = true;
                    } else if (lane == 0) {
                        vn1[jj[c]] = v1 * sqrt(temp);
                    }
                }
                if (any_redo) {  // uniform: every lane evaluated the same values
                    double nv[CB];
#pragma unroll
                    for (int c = 0; c < CB; ++c) {
                        nv[c] = 0.0;
#pragma unroll
                        for (int q = 0; q < RPL; ++q) {
                            const int r = lane + 32 * q;
                            if (r > i && r < m) nv[c] = fma(x[c][q], x[c][q], nv[c]);
                        }
                    }
                    warp_sum4(nv);
#pragma unroll
                    for (int c = 0; c < CB; ++c) {
                        if (!redo[c]) continue;
                        const double x2 = (i + 1 < m) ? sqrt(nv[c]) : 0.0;
                        if (lane == 0) { vn1[jj[c]] = x2; vn2[jj[c]] = x2; }
                    }
                }
                __syncwarp();
            }
        } else {
        for (int jp = i + 1 + warp; jp < k; jp += nw) {
            const int j = pos2phys[jp];
            double *cj = W + (long long)j * ldw;
            if (tau_i != 0.0) {
                double w = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) w += ci[r] * cj[r];
                w = warp_sum(w) + cj[i];
                const double f = tau_i * w;
                for (int r = i + 1 + lane; r < m; r += 32) cj[r] -= f * ci[r];
                __syncwarp();
                if (lane == 0) cj[i] -= f;
                __syncwarp();
            }
            const double v1 = vn1[j];
            if (v1 != 0.0) {
                double temp = fabs(cj[i]) / v1;
                temp = 1.0 - temp * temp;
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = v1 / vn2[j];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= TOL3Z) {
                    double nv = 0.0;
                    if (i + 1 < m) nv = sqrt(col_norm2(cj, i + 1, m, lane));
                    if (lane == 0) { vn1[j] = nv; vn2[j] = nv; }
                } else if (lane == 0) {
                    vn1[j] = v1 * sqrt(temp);
                }
            }
            __syncwarp();
        }
        }
        __syncthreads();
    }

    // rank decision (kernels.py:78-81)
    if (t == 0) {
        const double d0 = fabs(diagR[0]);
        int r = 0;
        if (d0 != 0.0) {
            const double cut = (double)(m > k ? m : k) * EPS * d0;
            for (int i = 0; i < kmin; ++i)
                if (fabs(diagR[i]) > cut) ++r;
        }
        rank_s = r;
        rank_out[args.base + b] = r;
    }
    __syncthreads();
    const int rank = rank_s;

    double *Q = args.Q[b];
    const int ldq = args.ldq[b];
    if constexpr (RPL > 0) {
        // Q column j = H_0 H_1 ... H_j e_j (what dorg2r forms for column j, in the same
        // reflector order), one warp per column, no CTA barriers: the reflectors stay
        // in the tile, read-only
        for (int j = warp; j < rank; j += nw) {
            double qv[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q) qv[q] = (lane + 32 * q == j) ? 1.0 : 0.0;
            for (int i = j; i >= 0; --i) {
                const double *vi = W + (long long)pos2phys[i] * ldw;
                const double ti = tau[i];
                double vr[RPL], d = 0.0;
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int r = lane + 32 * q;
                    vr[q] = (r > i && r < m) ? vi[r] : (r == i ? 1.0 : 0.0);
                    d = fma(vr[q], qv[q], d);
                }
                d = ti * warp_sum(d);
#pragma unroll
                for (int q = 0; q < RPL; ++q) qv[q] = fma(-d, vr[q], qv[q]);
            }
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int r = lane + 32 * q;
                if (r < m) Q[(long long)r * ldq + j] = qv[q];
            }
        }
        return;
    }
    // dorg2r on positions 0..rank-1 (storage of position i = physical pos2phys[i])
    for (int i = rank - 1; i >= 0; --i) {
        double *ci = W + (long long)pos2phys[i] * ldw;
        const double ti = tau[i];
        if (i < rank - 1) {
            for (int jp = i + 1 + warp; jp < rank; jp += nw) {
                double *cj = W + (long long)pos2phys[jp] * ldw;
                double w = 0.0;
                for (int r = i + 1 + lane; r < m; r += 32) w += ci[r] * cj[r];
                w = warp_sum(w) + cj[i];  // v_i[i] = 1
                const double f = ti * w;
                for (int r = i + 1 + lane; r < m; r += 32) cj[r] -= f * ci[r];
                __syncwarp();
                if (lane == 0) cj[i] -= f;
                __syncwarp();
            }
            __syncthreads();
        }
        for (int r = i + 1 + t; r < m; r += QR_THREADS) ci[r] *= -ti;
        for (int r = t; r < i; r += QR_THREADS) ci[r] = 0.0;
        if (t == 0) ci[i] = 1.0 - ti;
        __syncthreads();
    }
    for (long long e = t; e < (long long)m * rank; e += QR_THREADS) {
        const int r = (int)(e / rank), j = (int)(e % rank);
        Q[(long long)r * ldq + j] = W[(long long)pos2phys[j] * ldw + r];
    }
}

// ---------------------------------------------------------------------------
// Register-resident QRCP for small sketches (m <= 256, k <= 64, e.g. config[1]'s
// 256 x 58): the sketch lives in registers -- physical column j belongs to warp
// j % 16 (slot j / 16), lane l holds rows l, l+32, ..., l+224 -- so a Householder
// step touches only registers plus one 2 KB reflector broadcast through shared
// memory.  Every warp keeps a replicated copy of the position permutation (two
// entries per lane) and evaluates the pivot rule itself, so a step needs exactly two
// CTA barriers (dorg2r: one, with a double-buffered reflector).
//
// Row i of step i lives in register q = i / 32 of lane i % 32.  The steps are
// generated per register index QI (template), so every "row > i" mask and every
// extraction of row i is resolved at compile time except inside register QI: no
// runtime-indexed register selects (which made the first version instruction-bound).
// The sketch is loaded and Q stored through a shared-memory tile (coalesced global
// access), and Q's columns past the kept rank are written as zeros here.
constexpr int RQ_ROWS = 8;   // rows per lane  (m <= 256)
constexpr int RQ_SLOTS = 4;  // columns per warp (k <= 64)
constexpr int RQ_WARPS = 16;
constexpr int RQ_LDT = 65;   // staging tile stride in doubles (odd: conflict-free)
constexpr int RQ_SMEM = RQ_ROWS * 32 * RQ_LDT * 8;

__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

struct RegQr {
    double a[RQ_SLOTS][RQ_ROWS];
    int pos[RQ_SLOTS];  // position of my column, or k if unchosen
    int p0, p1;         // replicated permutation: positions lane and lane + 32
    int lane, warp, k;

    // pivot rule (first position of the largest partial norm), evaluated identically
    // by every warp; swaps positions i and the winner, returns the physical column
    __device__ __forceinline__ int pivot(int i, const double *vn1) {
        double best = -1.0;
        int bp = k;
        if (lane >= i && lane < k) { const double x = vn1[p0]; if (x > best) { best = x; bp = lane; } }
        if (lane + 32 >= i && lane + 32 < k) { const double x = vn1[p1]; if (x > best) { best = x; bp = lane + 32; } }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (ob > best || (ob == best && op < bp)) { best = ob; bp = op; }
        }
        if (bp >= k) bp = i;  // NaN norms (failed upstream pivot): keep the order
        const int pi = __shfl_sync(0xffffffffu, i < 32 ? p0 : p1, i & 31);
        const int pb = __shfl_sync(0xffffffffu, bp < 32 ? p0 : p1, bp & 31);
        if (lane == (i & 31)) { if (i < 32) p0 = pb; else p1 = pb; }
        if (lane == (bp & 31)) { if (bp < 32) p0 = pi; else p1 = pi; }
        return pb;
    }

    // dlarfg on rows i..m-1 of my slot-S column (the pivot); v gets rows > i
    template <int QI, int S>
    __device__ __forceinline__ void reflect(int i, int li, double *v, double *tau, double *diagR) {
        pos[S] = i;
        double part = 0.0;
#pragma unroll
        for (int q = QI; q < RQ_ROWS; ++q)
            if (q > QI || lane > li) part += a[S][q] * a[S][q];
        const double xnorm = sqrt(warp_sum(part));
        const double alpha = shfl(a[S][QI], li);
        double tau_i = 0.0, beta = alpha, scal = 1.0;
        if (xnorm != 0.0) {
            beta = -copysign(hypot(alpha, xnorm), alpha);
            tau_i = (beta - alpha) / beta;
            scal = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int q = QI; q < RQ_ROWS; ++q) {
            if (q > QI || lane > li) {
                if (xnorm != 0.0) a[S][q] *= scal;
                v[lane + 32 * q] = a[S][q];
            } else if (lane == li) {
                a[S][q] = beta;
            }
        }
        if (lane == 0) { tau[i] = tau_i; diagR[i] = beta; }
    }

    // H_i applied to my unchosen columns, then the dlaqp2 partial-norm downdate.  The
    // reflector carries its implicit 1 on row i, so one reduction gives v^T a
    // including row i, and row i of every column is updated in place by the lane
    // that holds it -- that lane also evaluates the downdate (no broadcast of row i).
    template <int QI>
    __device__ __forceinline__ void update(int i, int li, const double *v, double tau_i, double *vn1, double *vn2) {
        double vr[RQ_ROWS];
#pragma unroll
        for (int q = QI; q < RQ_ROWS; ++q)
            vr[q] = (q > QI || lane > li) ? v[lane + 32 * q] : ((q == QI && lane == li) ? 1.0 : 0.0);
        bool act[RQ_SLOTS];
#pragma unroll
        for (int s = 0; s < RQ_SLOTS; ++s) {
            const int j = warp + RQ_WARPS * s;
            act[s] = j < k && pos[s] >= k;
        }
        if (tau_i != 0.0) {
            double d[RQ_SLOTS];
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                d[s] = 0.0;
#pragma unroll
                for (int q = QI; q < RQ_ROWS; ++q) d[s] = fma(vr[q], a[s][q], d[s]);
            }
            warp_sum4(d);
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                if (!act[s]) continue;
                const double f = tau_i * d[s];
#pragma unroll
                for (int q = QI; q < RQ_ROWS; ++q) a[s][q] = fma(-f, vr[q], a[s][q]);
            }
        }
        // downdate on the lane holding row i; the recompute decision is broadcast
        unsigned redo_bits = 0;
        if (lane == li) {
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                const int j = warp + RQ_WARPS * s;
                if (!act[s]) continue;
                const double v1 = vn1[j];
                if (v1 == 0.0) continue;
                double temp = fabs(a[s][QI]) / v1;
                temp = 1.0 - temp * temp;
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = v1 / vn2[j];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= TOL3Z) redo_bits |= 1u << s;
                else vn1[j] = v1 * sqrt(temp);
            }
        }
        redo_bits = __shfl_sync(0xffffffffu, redo_bits, li);
        if (redo_bits) {
            double nv[RQ_SLOTS];
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                nv[s] = 0.0;
#pragma unroll
                for (int q = QI; q < RQ_ROWS; ++q)
                    if (q > QI || lane > li) nv[s] = fma(a[s][q], a[s][q], nv[s]);
            }
            warp_sum4(nv);
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                if (!((redo_bits >> s) & 1u)) continue;
                const double x = sqrt(nv[s]);  // rows > i exist: i + 1 < m is implied by zero padding
                if (lane == 0) { vn1[warp + RQ_WARPS * s] = x; vn2[warp + RQ_WARPS * s] = x; }
            }
        }
    }

    // Householder steps i0 <= i < i1 whose row lives in register QI
    template <int QI>
    __device__ __forceinline__ void factor_range(int i0, int i1, double *v, double *vn1, double *vn2,
                                                 double *tau, double *diagR) {
        for (int i = i0; i < i1; ++i) {
            const int li = i - 32 * QI;
            const int pc = pivot(i, vn1);
            if ((pc & (RQ_WARPS - 1)) == warp) {
                switch (pc / RQ_WARPS) {
                    case 0: reflect<QI, 0>(i, li, v, tau, diagR); break;
                    case 1: reflect<QI, 1>(i, li, v, tau, diagR); break;
                    case 2: reflect<QI, 2>(i, li, v, tau, diagR); break;
                    default: reflect<QI, 3>(i, li, v, tau, diagR); break;
                }
            }
            __syncthreads();
            update<QI>(i, li, v, tau[i], vn1, vn2);
            __syncthreads();
        }
    }

    // dorg2r steps i1-1 >= i >= i0 (rows in register QI); positions >= rank are idle
    template <int QI>
    __device__ __forceinline__ void form_range(int i0, int i1, int rank, double (*v)[RQ_ROWS * 32],
                                               const double *tau) {
        for (int i = i1 - 1; i >= i0; --i) {
            const int li = i - 32 * QI;
            double *vb = v[i & 1];
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                if (pos[s] != i) continue;
#pragma unroll
                for (int q = QI; q < RQ_ROWS; ++q)
                    if (q > QI || lane > li) vb[lane + 32 * q] = a[s][q];
            }
            __syncthreads();
            const double ti = tau[i];
            double vr[RQ_ROWS];
#pragma unroll
            for (int q = QI; q < RQ_ROWS; ++q) vr[q] = (q > QI || lane > li) ? vb[lane + 32 * q] : 0.0;
            double d[RQ_SLOTS], ai[RQ_SLOTS];
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                d[s] = 0.0;
#pragma unroll
                for (int q = QI; q < RQ_ROWS; ++q) d[s] += vr[q] * a[s][q];
                ai[s] = shfl(a[s][QI], li);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int s = 0; s < RQ_SLOTS; ++s) d[s] += __shfl_xor_sync(0xffffffffu, d[s], o);
#pragma unroll
            for (int s = 0; s < RQ_SLOTS; ++s) {
                if (pos[s] > i && pos[s] < rank) {
                    const double f = ti * (d[s] + ai[s]);
#pragma unroll
                    for (int q = QI; q < RQ_ROWS; ++q) a[s][q] -= f * vr[q];
                    if (lane == li) a[s][QI] -= f;
                } else if (pos[s] == i) {
#pragma unroll
                    for (int q = 0; q < RQ_ROWS; ++q) {
                        if (q < QI) a[s][q] = 0.0;
                        else if (q > QI) a[s][q] = -ti * vr[q];
                        else a[s][q] = lane > li ? -ti * vr[q] : (lane == li ? 1.0 - ti : 0.0);
                    }
                }
            }
        }
    }
};

__global__ void __launch_bounds__(RQ_WARPS * 32) qrcp_reg_kernel(const __grid_constant__ QrArgs args,
                                                                  int *rank_out) {
    extern __shared__ __align__(16) double tile[];  // [RQ_ROWS*32][RQ_LDT]
    __shared__ double v[2][RQ_ROWS * 32];
    __shared__ double vn1[64], vn2[64], tau[64], diagR[64];
    __shared__ int rank_s;
    const int b = blockIdx.x;
    const int m = args.m[b], k = args.k[b];
    const int t = threadIdx.x;
    RegQr st;
    st.lane = t & 31;
    st.warp = t >> 5;
    st.k = k;
    const int lane = st.lane, warp = st.warp;
    const double *G = args.G[b];
    const int ldg = args.ldg[b];
    // coalesced load of the row-major sketch into the tile, zero padded to 256 x 64
    for (int e = t; e < RQ_ROWS * 32 * 64; e += RQ_WARPS * 32) {
        const int r = e >> 6, j = e & 63;
        tile[r * RQ_LDT + j] = (r < m && j < k) ? G[(long long)r * ldg + j] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < RQ_SLOTS; ++s) {
        const int j = warp + RQ_WARPS * s;
        st.pos[s] = k;
        double nrm = 0.0;
#pragma unroll
        for (int q = 0; q < RQ_ROWS; ++q) {
            st.a[s][q] = tile[(lane + 32 * q) * RQ_LDT + j];
            nrm += st.a[s][q] * st.a[s][q];
        }
        nrm = sqrt(warp_sum(nrm));
        if (j < k && lane == 0) { vn1[j] = nrm; vn2[j] = nrm; }
    }
    st.p0 = lane;
    st.p1 = lane + 32;
    __syncthreads();
    const int kmin = m < k ? m : k;
    st.factor_range<0>(0, kmin < 32 ? kmin : 32, v[0], vn1, vn2, tau, diagR);
    st.factor_range<1>(32, kmin, v[0], vn1, vn2, tau, diagR);
    if (t == 0) {
        const double d0 = kmin > 0 ? fabs(diagR[0]) : 0.0;
        int r = 0;
        if (d0 != 0.0) {
            const double cut = (double)(m > k ? m : k) * EPS * d0;
            for (int i = 0; i < kmin; ++i)
                if (fabs(diagR[i]) > cut) ++r;
        }
        rank_s = r;
        rank_out[args.base + b] = r;
    }
    __syncthreads();
    const int rank = rank_s;
    // Q column j = H_0 ... H_j e_j (dorg2r's reflector order), formed per warp with no
    // CTA barriers: the reflectors go to the tile (column = position), every warp
    // builds its Q columns in registers, then they replace the reflectors in the tile
#pragma unroll
    for (int s = 0; s < RQ_SLOTS; ++s) {
        if (st.pos[s] >= rank) continue;
#pragma unroll
        for (int q = 0; q < RQ_ROWS; ++q) tile[(lane + 32 * q) * RQ_LDT + st.pos[s]] = st.a[s][q];
    }
    __syncthreads();
    double qv[RQ_SLOTS][RQ_ROWS];
#pragma unroll
    for (int c = 0; c < RQ_SLOTS; ++c) {
        const int j = warp + RQ_WARPS * c;
#pragma unroll
        for (int q = 0; q < RQ_ROWS; ++q) qv[c][q] = (lane + 32 * q == j) ? 1.0 : 0.0;
        if (j >= rank) continue;
        for (int i = j; i >= 0; --i) {
            const double ti = tau[i];
            double vr[RQ_ROWS], d = 0.0;
#pragma unroll
            for (int q = 0; q < RQ_ROWS; ++q) {
                const int r = lane + 32 * q;
                vr[q] = r > i ? tile[r * RQ_LDT + i] : (r == i ? 1.0 : 0.0);
                d = fma(vr[q], qv[c][q], d);
            }
            d = ti * warp_sum(d);
#pragma unroll
            for (int q = 0; q < RQ_ROWS; ++q) qv[c][q] = fma(-d, vr[q], qv[c][q]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < RQ_SLOTS; ++c) {
        const int j = warp + RQ_WARPS * c;
        if (j >= rank) continue;
#pragma unroll
        for (int q = 0; q < RQ_ROWS; ++q) tile[(lane + 32 * q) * RQ_LDT + j] = qv[c][q];
    }
    __syncthreads();
    double *Q = args.Q[b];
    const int ldq = args.ldq[b];
    for (int e = t; e < m * k; e += RQ_WARPS * 32) {
        const int r = e / k, j = e - r * k;
        Q[(long long)r * ldq + j] = j < rank ? tile[r * RQ_LDT + j] : 0.0;
    }
}

constexpr long long SMEM_BYTES_MAX = 220 * 1024;

// the one-CTA kernel keeps the sketch plus 4 FP64 + 2 int per-column arrays in smem
inline long long smem_bytes(int m, int k) { return (long long)(m | 1) * k * 8 + 40LL * k; }
inline bool fits_smem(int m, int k) { return smem_bytes(m, k) <= SMEM_BYTES_MAX; }

}  // namespace

// multi-CTA path for sketches that do not fit one SM (qr_coop.cu)
long long rsc_qrcp_coop_doubles(int m, int k);
int rsc_qrcp_multi(int n, const int *ids, double *const *G, const int *m, const int *k, const int *ldg,
                   double *const *Q, const int *ldq, int *rank_dev, char *work, const long long *work_off,
                   unsigned *bar, cudaStream_t s);

static inline long long coop_bytes(int m, int k) { return ((rsc_qrcp_coop_doubles(m, k) * 8 + 255) / 256) * 256; }

extern "C" long long rsc_qrcp_workspace_bytes(int count, const int *m, const int *k) {
    long long tot = ((4LL * count + 255) / 256) * 256;  // group-barrier counters
    for (int i = 0; i < count; ++i) {
        if (!fits_smem(m[i], k[i])) tot += coop_bytes(m[i], k[i]);
    }
    return tot < 256 ? 256 : tot;
}

// Q[:, rank:k] = 0 for every matrix (the factor keeps sketch-width panels whose
// trailing columns must contribute exact zeros; no host readback of the ranks)
__global__ void zero_tail_kernel(const __grid_constant__ QrArgs a, const int *rank_dev) {
    const int b = blockIdx.x;
    const int r0 = rank_dev[a.base + b], k = a.k[b], m = a.m[b], ldq = a.ldq[b];
    const int w = k - r0;
    if (w <= 0) return;
    double *Q = a.Q[b];
    for (long long e = threadIdx.x; e < (long long)m * w; e += blockDim.x) {
        const int r = (int)(e / w), j = r0 + (int)(e % w);
        Q[(long long)r * ldq + j] = 0.0;
    }
}

int qr_zero_tails(int count, const int *m, const int *k, double *const *Q, const int *ldq, int *rank_dev,
                  cudaStream_t s) {
    static thread_local QrArgs qa;
    for (int c0 = 0; c0 < count; c0 += MAXB) {
        const int cnt = count - c0 < MAXB ? count - c0 : MAXB;
        qa.count = cnt;
        qa.base = c0;
        for (int c = 0; c < cnt; ++c) {
            qa.Q[c] = Q[c0 + c];
            qa.m[c] = m[c0 + c];
            qa.k[c] = k[c0 + c];
            qa.ldq[c] = ldq[c0 + c];
        }
        zero_tail_kernel<<<cnt, 256, 0, s>>>(qa, rank_dev);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

extern "C" int rsc_qrcp_batched(int count, double *const *G, const int *m, const int *k,
                                const int *ldg, double *const *Q, const int *ldq, int *rank_dev,
                                void *work_dev, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!G || !m || !k || !ldg || !Q || !ldq || !rank_dev) return -2;
    cudaStream_t s = (cudaStream_t)stream;
    static bool attr_set = false;
    if (!attr_set) {
        cudaFuncSetAttribute(qrcp_kernel<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)SMEM_BYTES_MAX);
#define RSC_QR_ATTR(R) \
    cudaFuncSetAttribute(qrcp_kernel<true, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES_MAX);
        RSC_QR_ATTR(1) RSC_QR_ATTR(2) RSC_QR_ATTR(3) RSC_QR_ATTR(4)
        RSC_QR_ATTR(5) RSC_QR_ATTR(6) RSC_QR_ATTR(7) RSC_QR_ATTR(8)
#undef RSC_QR_ATTR
        cudaFuncSetAttribute(qrcp_reg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, RQ_SMEM);
        attr_set = true;
    }
    std::vector<int> tiny, small, big;
    for (int i = 0; i < count; ++i) {
        if (k[i] > QR_MAXK || m[i] < 0 || k[i] < 0) return -4;
        if (m[i] <= RQ_ROWS * 32 && k[i] <= RQ_SLOTS * RQ_WARPS) tiny.push_back(i);
        else if (fits_smem(m[i], k[i])) small.push_back(i);
        else big.push_back(i);
    }
    if (!big.empty() && !work_dev) return -10;
    static thread_local QrArgs qa;
    // the rank array is indexed by original position: launch per contiguous run so
    // `base` stays valid; simpler: one launch per matrix group with explicit mapping
    auto run = [&](const std::vector<int> &ids, bool smem) -> int {
        size_t pos = 0;
        long long woff = 0;
        while (pos < ids.size()) {
            // contiguous runs of original indices keep base+b addressing exact
            qa.count = 0;
            qa.base = ids[pos];
            long long maxsz = 0;
            while (pos < ids.size() && qa.count < MAXB && ids[pos] == qa.base + qa.count) {
                const int i = ids[pos++];
                const int c = qa.count++;
                qa.G[c] = G[i]; qa.Q[c] = Q[i];
                qa.m[c] = m[i]; qa.k[c] = k[i]; qa.ldg[c] = ldg[i]; qa.ldq[c] = ldq[i];
                const long long sz = (long long)(m[i] | 1) * k[i];
                const long long need = smem ? smem_bytes(m[i], k[i]) : 40LL * k[i];
                maxsz = need > maxsz ? need : maxsz;
                qa.woff[c] = smem ? 0 : woff / 8;
                if (!smem) woff += ((sz * 8 + 255) / 256) * 256;
            }
            if (smem) {
                int maxm = 0;
                for (int c = 0; c < qa.count; ++c) maxm = qa.m[c] > maxm ? qa.m[c] : maxm;
                const int rpl = (maxm + 31) / 32;
                switch (rpl) {
#define RSC_QR_CASE(R)                                                                           \
    case R:                                                                                      \
        qrcp_kernel<true, R><<<qa.count, QR_THREADS, (size_t)maxsz, s>>>(qa, nullptr, rank_dev); \
        break;
                    RSC_QR_CASE(1) RSC_QR_CASE(2) RSC_QR_CASE(3) RSC_QR_CASE(4)
                    RSC_QR_CASE(5) RSC_QR_CASE(6) RSC_QR_CASE(7) RSC_QR_CASE(8)
#undef RSC_QR_CASE
                    default:
                        qrcp_kernel<true, 0><<<qa.count, QR_THREADS, (size_t)maxsz, s>>>(qa, nullptr, rank_dev);
                }
            } else {
                qrcp_kernel<false, 0><<<qa.count, QR_THREADS, (size_t)maxsz, s>>>(qa, (double *)work_dev, rank_dev);
            }
            RSC_CHECK_LAUNCH();
        }
        return 0;
    };
    // register-resident kernel for the smallest sketches (contiguous runs keep `base`)
    {
        size_t pos = 0;
        while (pos < tiny.size()) {
            qa.count = 0;
            qa.base = tiny[pos];
            while (pos < tiny.size() && qa.count < MAXB && tiny[pos] == qa.base + qa.count) {
                const int i = tiny[pos++];
                const int c = qa.count++;
                qa.G[c] = G[i]; qa.Q[c] = Q[i];
                qa.m[c] = m[i]; qa.k[c] = k[i]; qa.ldg[c] = ldg[i]; qa.ldq[c] = ldq[i];
                qa.woff[c] = 0;
            }
            qrcp_reg_kernel<<<qa.count, RQ_WARPS * 32, RQ_SMEM, s>>>(qa, rank_dev);
            RSC_CHECK_LAUNCH();
        }
    }
    int rc = run(small, true);
    if (rc) return rc;
    // large sketches: all of them concurrently in cooperative multi-CTA groups;
    // workspace = barrier counters, then per-matrix slices in index order
    if (!big.empty()) {
        std::vector<long long> off(count, 0);
        long long o = ((4LL * count + 255) / 256) * 256;
        for (int i : big) {
            off[i] = o;
            o += coop_bytes(m[i], k[i]);
        }
        rc = rsc_qrcp_multi((int)big.size(), big.data(), G, m, k, ldg, Q, ldq, rank_dev, (char *)work_dev,
                            off.data(), (unsigned *)work_dev, s);
        if (rc) return rc;
    }
    if (tiny.size() == (size_t)count) return 0;  // the register kernel wrote its zero tails
    return qr_zero_tails(count, m, k, Q, ldq, rank_dev, s);
}
