// Device Gaussian sketches, bit-identical to the reference's host stream
//   np.random.Generator(np.random.PCG64(seed)).standard_normal((m, r))
// (reference kernels.py:85-92; factor.py:324-326 seeds each block).
//
// One stream per sketch.  numpy draws one 64-bit PCG64 output per normal in ~98.5%
// of cases (the ziggurat's quick accept) and 2 or more otherwise, so the position
// of the k-th normal in the raw stream is only known after a scan.  Three kernels:
//
//   1. rng_scan_kernel      one CTA per 4096-draw chunk: generate the chunk
//      (PCG64 jump-ahead to the chunk start), flag the "slow" positions (quick test
//      fails), and for each evaluate -- as if a try started there -- how many draws
//      the try consumes, whether it returns a value, and the value.  A try's outcome
//      depends only on the draws from its own position on, so this is exact.  The
//      chunk then walks its slow positions once assuming the first try starts at
//      the chunk start (true unless the previous chunk's last try spills over,
//      ~1.5% of chunks): all other positions are 1-draw tries that return.
//   2. rng_walk_kernel      one thread per stream: chains the chunks (entry offset,
//      output base); only a chunk entered at a non-zero offset is re-walked.
//   3. rng_emit_kernel      one CTA per chunk: per-position output flags, a block
//      scan, values staged in shared memory, one coalesced store.
//
// Both rare overflows (a chunk with > CAND_MAX slow positions; a stream that needs
// more draws than were scanned) fall back to an exact sequential generator on the
// walking thread, so the output never depends on luck.  Arithmetic follows numpy's
// random_standard_normal (numpy/random/src/distributions/distributions.c) op for
// op with explicit IEEE rounding; log1p is glibc's (log1p_fd.cuh); the tables are
// numpy's own bytes (gen_ziggurat.py).  The one libm call whose last bit is not
// reproduced is exp() in the wedge test, where a difference flips the accept only
// if both sides agree to within an ulp (~2^-52 per test).
#include <cstdint>
#include <vector>

#include "../../include/rsc_b200.h"
#include "build/ziggurat_tables.h"
#include "common.cuh"
#include "log1p_fd.cuh"

namespace {

typedef unsigned __int128 u128;

constexpr int CH = 4096;          // draws per chunk
constexpr int RT = 128;           // threads per chunk CTA
constexpr int PER = CH / RT;      // draws per thread (contiguous)
constexpr int CAND_MAX = 160;     // slow positions recorded per chunk (mean ~61)
constexpr int MAXS = 600;         // streams per launch group (kernel-parameter budget)

constexpr double ZIG_R = 3.6541528853610087963519472518;
constexpr double ZIG_INV_R = 0.27366123732975827203338247596;

struct RngStream {
    unsigned long long s_hi, s_lo, i_hi, i_lo;
    double *out;
    long long n;
};

struct RngArgs {
    int count;
    int nchunks;
    int cand_cap;                 // <= CAND_MAX; lowered only by the test hook
    int chunk_off[MAXS + 1];      // prefix of chunk counts per stream
    RngStream st[MAXS];
};

struct Cand {
    int pos;     // offset within the chunk
    int len;     // draws consumed by a try starting here
    int acc;     // try returns a value
    int tr;      // set by the walk: a real try start
    double val;
};

struct ChunkMeta {
    int ncand;   // -1: overflow (chunk emitted by the walk)
    int entry;   // first try start (offset), >= CH: nothing to emit
    long long base;
    int spec_count;  // values emitted when entered at offset 0
    int spec_exit;   // first try start past the chunk end - CH, same assumption
};

// jump tables c_jm / c_jg (build/ziggurat_tables.h): M^(2^k) and G_k = sum_{i < 2^k}
// M^i, so that k steps from s are M^k s + inc * G(k) -- stream independent,
// initialized with the module (no runtime upload, so every call is capture-safe)

__device__ __forceinline__ u128 mk(unsigned long long hi, unsigned long long lo) {
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ u128 pcg_mult() { return mk(0x2360ed051fc65da4ULL, 0x4385df649fccf645ULL); }

__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
    const unsigned long long x = (unsigned long long)(s >> 64) ^ (unsigned long long)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

// state after `delta` further steps
__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, unsigned long long delta) {
    for (int k = 0; delta; ++k, delta >>= 1)
        if (delta & 1) s = mk(c_jm[k][0], c_jm[k][1]) * s + inc * mk(c_jg[k][0], c_jg[k][1]);
    return s;
}

__device__ __forceinline__ double u01(unsigned long long d) {
    return __dmul_rn((double)(d >> 11), 1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double fi(int i) { return __longlong_as_double((long long)zig_fi_bits[i]); }

// quick path of one try: true if the draw returns immediately (value in *x);
// ki / wi point at the tables (shared-memory copies on the hot kernels: a
// per-lane table index through the constant cache would serialize)
__device__ __forceinline__ bool quick(unsigned long long d, const unsigned long long *ki,
                                      const unsigned long long *wi, double *x, int *idx_out,
                                      unsigned long long *rabs_out) {
    const int idx = (int)(d & 0xff);
    const unsigned long long r = d >> 8;
    const unsigned long long rabs = (r >> 1) & 0x000fffffffffffffULL;
    double v = __dmul_rn((double)rabs, __longlong_as_double((long long)wi[idx]));
    if (r & 1) v = -v;
    *x = v;
    *idx_out = idx;
    *rabs_out = rabs;
    return rabs < ki[idx];
}

// slow path of a try whose first draw failed the quick test; draws after it come
// from `next()`.  Returns (consumed draws incl. the first, accepted, value).
template <class Next>
__device__ __forceinline__ void slow_try(int idx, unsigned long long rabs, double x, Next next, int *len,
                                         int *acc, double *val) {
    if (idx == 0) {
        int used = 1;
        for (;;) {
            const double xx = __dmul_rn(-ZIG_INV_R, log1p_fdlibm(-u01(next())));
            const double yy = -log1p_fdlibm(-u01(next()));
            used += 2;
            if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
                const double v = __dadd_rn(ZIG_R, xx);
                *val = ((rabs >> 8) & 1) ? -v : v;
                *acc = 1;
                *len = used;
                return;
            }
        }
    }
    const double u = u01(next());
    const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(fi(idx - 1), fi(idx)), u), fi(idx));
    const double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
    *acc = lhs < rhs;
    *val = x;
    *len = 2;
}

__device__ __forceinline__ int find_stream(const RngArgs &a, int chunk) {
    int lo = 0, hi = a.count - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (a.chunk_off[mid] <= chunk) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ int block_excl_scan(int v, int *warp_tot, int *total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < RT / 32; ++i) {
        if (i < w) off += warp_tot[i];
        tot += warp_tot[i];
    }
    *total = tot;
    return off + incl - v;
}

// 8-byte smem slot of chunk position p: thread t owns p = 32t + j, so lanes with
// the same j would all hit one bank pair; xor-ing j with t spreads them
__device__ __forceinline__ int swz(int p) { return p ^ ((p >> 5) & 15); }

__device__ __forceinline__ void load_tables(unsigned long long *ki, unsigned long long *wi) {
    for (int i = threadIdx.x; i < 256; i += RT) {
        ki[i] = zig_ki[i];
        wi[i] = zig_wi_bits[i];
    }
}

__global__ void __launch_bounds__(RT) rng_scan_kernel(const __grid_constant__ RngArgs a, Cand *cands,
                                                      ChunkMeta *meta) {
    __shared__ unsigned long long dr[CH];
    __shared__ unsigned long long ki[256], wi[256];
    __shared__ Cand sc[CAND_MAX];
    __shared__ int warp_tot[RT / 32];
    const int chunk = blockIdx.x;
    const int s = find_stream(a, chunk);
    const long long c = chunk - a.chunk_off[s];
    const RngStream &S = a.st[s];
    const u128 s0 = mk(S.s_hi, S.s_lo), inc = mk(S.i_hi, S.i_lo), M = pcg_mult();
    const long long cs = c * CH;
    const int t0 = threadIdx.x * PER;
    load_tables(ki, wi);
    u128 st = pcg_advance(s0, inc, (unsigned long long)(cs + t0));
    __syncthreads();
    unsigned slow_mask = 0;
#pragma unroll 8
    for (int j = 0; j < PER; ++j) {
        st = st * M + inc;
        const unsigned long long d = pcg_out(st);
        dr[swz(t0 + j)] = d;
        if (((d >> 9) & 0x000fffffffffffffULL) >= ki[d & 0xff]) slow_mask |= 1u << j;  // quick test fails
    }
    int total;
    int slot = block_excl_scan(__popc(slow_mask), warp_tot, &total);  // also orders dr
    if (total > a.cand_cap) {
        if (threadIdx.x == 0) meta[chunk].ncand = -1;
        return;
    }
    while (slow_mask) {
        const int j = __ffs(slow_mask) - 1;
        slow_mask &= slow_mask - 1;
        const int pos = t0 + j;
        double x;
        int idx;
        unsigned long long rabs;
        quick(dr[swz(pos)], ki, wi, &x, &idx, &rabs);
        long long p = cs + pos + 1;  // absolute position of the next draw
        u128 far = 0;
        bool far_ok = false;
        auto next = [&]() -> unsigned long long {
            const long long q = p++;
            if (q < cs + CH) return dr[swz((int)(q - cs))];
            if (!far_ok) {
                far = pcg_advance(s0, inc, (unsigned long long)q);
                far_ok = true;
            }
            far = far * M + inc;
            return pcg_out(far);
        };
        Cand &cd = sc[slot++];
        cd.pos = pos;
        cd.tr = 0;
        slow_try(idx, rabs, x, next, &cd.len, &cd.acc, &cd.val);
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // walk assuming the chunk is entered at offset 0
        int cur = 0, outc = 0;
        for (int i = 0; i < total; ++i) {
            Cand &k = sc[i];
            if (k.pos < cur) continue;
            outc += k.pos - cur;
            k.tr = 1;
            outc += k.acc;
            cur = k.pos + k.len;
        }
        if (cur < CH) {
            outc += CH - cur;
            cur = CH;
        }
        ChunkMeta &m = meta[chunk];
        m.ncand = total;
        m.spec_count = outc;
        m.spec_exit = cur - CH;
    }
    __syncthreads();
    Cand *out = cands + (size_t)chunk * CAND_MAX;
    for (int i = threadIdx.x; i < total; i += RT) out[i] = sc[i];
}

// exact sequential generator from absolute position `cur` (a try start); emits into
// dst[*outc ..] while positions < limit and fewer than n values; returns next start
__device__ long long seq_fill(u128 s0, u128 inc, long long cur, long long limit, long long n, double *dst,
                              long long *outc) {
    const u128 M = pcg_mult();
    u128 st = pcg_advance(s0, inc, (unsigned long long)cur);
    long long p = cur, o = *outc;
    auto next = [&]() -> unsigned long long {
        st = st * M + inc;
        ++p;
        return pcg_out(st);
    };
    while (p < limit && o < n) {
        double x;
        int idx;
        unsigned long long rabs;
        if (quick(next(), zig_ki, zig_wi_bits, &x, &idx, &rabs)) {
            dst[o++] = x;
            continue;
        }
        int len, acc;
        double v;
        slow_try(idx, rabs, x, next, &len, &acc, &v);
        if (acc) dst[o++] = v;
    }
    *outc = o;
    return p;
}

// (count, exit) of chunk `cd` entered at offset `e` (0 < e < CH), marking try starts
__device__ void rewalk(Cand *cd, int ncand, int e, int *count, int *exit) {
    int cur = e, outc = 0;
    for (int i = 0; i < ncand; ++i) {
        const int q = cd[i].pos;
        if (q < cur) {
            cd[i].tr = 0;
            continue;
        }
        outc += q - cur;
        cd[i].tr = 1;
        outc += cd[i].acc;
        cur = q + cd[i].len;
    }
    if (cur < CH) {
        outc += CH - cur;
        cur = CH;
    }
    *count = outc;
    *exit = cur - CH;
}

// one warp per stream, 32 chunks per step: every lane assumes its chunk is entered
// where its left neighbour's current guess exits, re-walks if that is not offset 0,
// and the warp repeats until no entry changes (1-2 rounds in practice); then a warp
// scan of the counts gives the output bases.
__global__ void rng_walk_kernel(const __grid_constant__ RngArgs a, Cand *cands, ChunkMeta *meta) {
    const int s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (s >= a.count) return;
    const RngStream &S = a.st[s];
    const u128 s0 = mk(S.s_hi, S.s_lo), inc = mk(S.i_hi, S.i_lo);
    const long long n = S.n;
    const int c0 = a.chunk_off[s], c1 = a.chunk_off[s + 1];
    long long out = 0;  // values emitted by chunks before the current batch
    long long carry = 0;  // entry offset of the batch's first chunk
    for (int b = c0; b < c1; b += 32) {
        const int chunk = b + lane;
        const bool valid = chunk < c1;
        int ncand = 0, sc = 0, se = 0;
        if (valid) {
            ncand = meta[chunk].ncand;
            sc = meta[chunk].spec_count;
            se = meta[chunk].spec_exit;
        }
        if (__any_sync(0xffffffffu, valid && ncand < 0)) {
            // an overflowed chunk (never seen in practice): finish this batch serially
            if (lane == 0) {
                long long cur = (long long)(b - c0) * CH + carry;
                for (int ch = b; ch < c1 && ch < b + 32; ++ch) {
                    const long long cs = (long long)(ch - c0) * CH, ce = cs + CH;
                    ChunkMeta &m = meta[ch];
                    m.base = out;
                    if (out >= n || cur >= ce) {
                        m.entry = CH;
                        continue;
                    }
                    if (m.ncand < 0) {
                        m.entry = CH;
                        cur = seq_fill(s0, inc, cur, ce, n, S.out, &out);
                        continue;
                    }
                    m.entry = (int)(cur - cs);
                    int cnt = m.spec_count, ex = m.spec_exit;
                    if (cur != cs) rewalk(cands + (size_t)ch * CAND_MAX, m.ncand, m.entry, &cnt, &ex);
                    out += cnt;
                    cur = ce + ex;
                }
                carry = cur - (long long)(min(b + 32, c1) - c0) * CH;
            }
            out = __shfl_sync(0xffffffffu, out, 0);
            carry = __shfl_sync(0xffffffffu, carry, 0);
            continue;
        }
        long long entry = lane == 0 ? carry : 0;  // guess
        int cnt = sc, ex = se;
        bool dirty = false;  // try-start flags were rewritten by a re-walk
        for (;;) {
            if (valid) {
                if (entry >= CH) {
                    cnt = 0;
                    ex = (int)(entry - CH);
                } else if (entry > 0) {
                    rewalk(cands + (size_t)chunk * CAND_MAX, ncand, (int)entry, &cnt, &ex);
                    dirty = true;
                } else {
                    cnt = sc;
                    ex = se;
                }
            }
            long long left = __shfl_up_sync(0xffffffffu, (long long)ex, 1);
            const long long want = lane == 0 ? carry : left;
            const bool changed = valid && want != entry;
            if (!__any_sync(0xffffffffu, changed)) break;
            entry = want;
        }
        if (valid && dirty && entry == 0) rewalk(cands + (size_t)chunk * CAND_MAX, ncand, 0, &cnt, &ex);
        // output bases: warp scan of counts
        long long incl = valid ? cnt : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (valid) {
            ChunkMeta &m = meta[chunk];
            const long long base = out + incl - cnt;
            m.base = base;
            m.entry = (entry >= CH || base >= n) ? CH : (int)entry;
        }
        const int last = min(32, c1 - b) - 1;
        out += __shfl_sync(0xffffffffu, incl, last);
        carry = __shfl_sync(0xffffffffu, (long long)ex, last);
    }
    if (lane == 0 && out < n) {
        const long long cur = (long long)(c1 - c0) * CH + carry;
        seq_fill(s0, inc, cur, 0x7fffffffffffffffLL, n, S.out, &out);
    }
}

__global__ void __launch_bounds__(RT) rng_emit_kernel(const __grid_constant__ RngArgs a, const Cand *cands,
                                                      const ChunkMeta *meta) {
    __shared__ double vals[CH];
    __shared__ unsigned long long ki[256], wi[256];
    __shared__ unsigned omask[RT], cmask[RT];  // per owned 32-position word: emits / from a record
    __shared__ int tp[RT];
    __shared__ int warp_tot[RT / 32];
    const int chunk = blockIdx.x;
    const ChunkMeta m = meta[chunk];
    if (m.entry >= CH) return;
    const int s = find_stream(a, chunk);
    const RngStream &S = a.st[s];
    const long long c = chunk - a.chunk_off[s];
    const Cand *cd = cands + (size_t)chunk * CAND_MAX;
    const int t = threadIdx.x, t0 = t * PER;
    load_tables(ki, wi);
    omask[t] = m.entry <= t0 ? ~0u : (m.entry >= t0 + PER ? 0u : (~0u << (m.entry - t0)));
    cmask[t] = 0u;
    const u128 s0 = mk(S.s_hi, S.s_lo), inc = mk(S.i_hi, S.i_lo), M = pcg_mult();
    u128 st = pcg_advance(s0, inc, (unsigned long long)(c * CH + t0));
    __syncthreads();
    for (int i = t; i < m.ncand; i += RT) {
        const Cand k = cd[i];
        if (!k.tr) continue;
        if (k.acc) atomicOr(&cmask[k.pos >> 5], 1u << (k.pos & 31));
        else atomicAnd(&omask[k.pos >> 5], ~(1u << (k.pos & 31)));
        const int e = min(k.pos + k.len, CH);
        for (int q = k.pos + 1; q < e; ++q) atomicAnd(&omask[q >> 5], ~(1u << (q & 31)));
    }
    __syncthreads();
    const unsigned my = omask[t], mine_c = cmask[t];
    int total;
    const int off = block_excl_scan(__popc(my), warp_tot, &total);
    tp[t] = off;
    int o = off;
#pragma unroll 8
    for (int j = 0; j < PER; ++j) {
        st = st * M + inc;
        if ((my >> j) & 1) {
            if (!((mine_c >> j) & 1)) {
                double x;
                int idx;
                unsigned long long rabs;
                quick(pcg_out(st), ki, wi, &x, &idx, &rabs);
                vals[o] = x;
            }
            ++o;
        }
    }
    __syncthreads();
    for (int i = t; i < m.ncand; i += RT) {
        const Cand k = cd[i];
        if (!k.tr || !k.acc) continue;
        const int w = k.pos >> 5;
        vals[tp[w] + __popc(omask[w] & ((1u << (k.pos & 31)) - 1u))] = k.val;
    }
    __syncthreads();
    const long long lim = S.n - m.base;
    const int nw = (int)(total < lim ? total : (lim > 0 ? lim : 0));
    double *dst = S.out + m.base;
    for (int i = t; i < nw; i += RT) dst[i] = vals[i];
}

int g_cand_cap = CAND_MAX;   // test hook (rsc_normal_debug_limits)
int g_slack = 1;

long long chunks_for(long long n) {
    const long long draws = g_slack ? n + n / 32 + 256 : n / 2;
    return draws > 0 ? (draws + CH - 1) / CH : 1;
}

}  // namespace

extern "C" size_t rsc_normal_workspace_bytes(int count, const long long *n) {
    if (count <= 0 || !n) return 256;
    size_t best = 0;
    for (int g0 = 0; g0 < count; g0 += MAXS) {
        const int g1 = g0 + MAXS < count ? g0 + MAXS : count;
        long long ch = 0;
        for (int i = g0; i < g1; ++i) ch += n[i] > 0 ? chunks_for(n[i]) : 0;
        const size_t b = (size_t)ch * (CAND_MAX * sizeof(Cand) + sizeof(ChunkMeta));
        best = b > best ? b : best;
    }
    return best < 256 ? 256 : best;
}

extern "C" int rsc_normal_pcg64(int count, const unsigned long long *states, const long long *n,
                                double *const *out, void *work, size_t work_bytes, void *stream) {
    if (count < 0) return -1;
    if (count == 0) return 0;
    if (!states || !n || !out || !work) return -2;
    if (work_bytes < rsc_normal_workspace_bytes(count, n)) return -3;
    cudaStream_t sm = (cudaStream_t)stream;
    static thread_local RngArgs a;
    for (int g0 = 0; g0 < count; g0 += MAXS) {
        const int g1 = g0 + MAXS < count ? g0 + MAXS : count;
        a.count = 0;
        a.cand_cap = g_cand_cap;
        int ch = 0;
        for (int i = g0; i < g1; ++i) {
            if (n[i] < 0) return -4;
            if (n[i] == 0) continue;
            if (!out[i]) return -2;
            RngStream &S = a.st[a.count];
            S.s_hi = states[4 * (size_t)i];
            S.s_lo = states[4 * (size_t)i + 1];
            S.i_hi = states[4 * (size_t)i + 2];
            S.i_lo = states[4 * (size_t)i + 3];
            S.out = out[i];
            S.n = n[i];
            a.chunk_off[a.count++] = ch;
            ch += (int)chunks_for(n[i]);
        }
        if (!a.count) continue;
        a.chunk_off[a.count] = ch;
        a.nchunks = ch;
        Cand *cands = (Cand *)work;
        ChunkMeta *meta = (ChunkMeta *)((char *)work + (size_t)ch * CAND_MAX * sizeof(Cand));
        rng_scan_kernel<<<ch, RT, 0, sm>>>(a, cands, meta);
        RSC_CHECK_LAUNCH();
        rng_walk_kernel<<<(a.count + 3) / 4, 128, 0, sm>>>(a, cands, meta);
        RSC_CHECK_LAUNCH();
        rng_emit_kernel<<<ch, RT, 0, sm>>>(a, cands, meta);
        RSC_CHECK_LAUNCH();
    }
    return 0;
}

// Test hook: force the exact sequential fallbacks (cand_cap < CAND_MAX makes chunks
// overflow; slack = 0 scans only n/2 draws so every stream finishes sequentially).
extern "C" int rsc_normal_debug_limits(int cand_cap, int slack) {
    if (cand_cap < 0 || cand_cap > CAND_MAX) return -1;
    g_cand_cap = cand_cap;
    g_slack = slack ? 1 : 0;
    return 0;
}

extern "C" double rsc_log1p_fdlibm(double x) { return log1p_fdlibm(x); }
