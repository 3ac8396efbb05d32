// Host-side plan compiler kernels (plan.py NumericPlan): the descendant maps of
// every (update source, target supernode) pair and the window maps of every
// (diagonal-tree block, source) pair.  These are the index computations the
// reference redoes on every call (factor.py:389-398, 450-455, 477-482;
// diagblocks.py:231-262); here they run once per symbolic plan, on host threads.
// Every output is a pure function of the inputs (results are written by pair
// index, not by thread), so the threaded result is the sequential one.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <numeric>
#include <thread>
#include <vector>

#include "host_par.h"

namespace {

struct PairsOut {
    std::vector<long long> tgt, src, lo, hi, cpos, rpos;
    std::vector<int> idx;
};

struct TreeOut {
    std::vector<long long> tree, blk, src, clo, chi, rlo, rhi, coff, roff;
    std::vector<int> idx;
};

inline long long lbound(const long long *a, long long n, long long v) {
    return (long long)(std::lower_bound(a, a + n, v) - a);
}

}  // namespace

extern "C" {

// Pairs (target j, source s) for every source s and every target supernode j
// (is_target[j] != 0) that one of s's rows falls into; lo/hi = the run of s's
// rows inside C_j = [starts[j], starts[j+1]).  Grouped by target ascending, within
// a target by src_order ascending (factor.py:545-554,572 bucket order).  Index
// chunk per pair: cpos = rows[lo:hi] - c0 (hi-lo ints), then
// rpos = searchsorted(R_j, rows[hi:]) (nrows-hi ints); offsets relative to the
// chunk.  Returns a handle (fetch with rsc_plan_pairs_fetch) and the sizes.
void *rsc_plan_pairs(long long nsrc, const long long *src_ptr, const long long *src_rows,
                     const long long *src_order, long long M, const long long *starts,
                     const unsigned char *is_target, const long long *R_ptr, const long long *R_rows,
                     long long *npairs, long long *nidx) {
    auto *o = new PairsOut();
    const int T = rsc_host_threads();
    // pass 1: runs per source (counted, then filled in source order)
    std::vector<long long> cnt(nsrc + 1, 0);
    auto runs = [&](long long s, bool fill, long long base) {
        const long long *r = src_rows + src_ptr[s];
        const long long n = src_ptr[s + 1] - src_ptr[s];
        long long k = 0, p = 0;
        while (p < n) {
            const long long j = (long long)(std::upper_bound(starts, starts + M + 1, r[p]) - starts) - 1;
            const long long e = p + lbound(r + p, n - p, starts[j + 1]);
            if (is_target[j]) {
                if (fill) {
                    o->tgt[base + k] = j;
                    o->src[base + k] = s;
                    o->lo[base + k] = p;
                    o->hi[base + k] = e;
                }
                ++k;
            }
            p = e;
        }
        return k;
    };
    rsc_parallel_chunks(nsrc, T, [&](int, long long a, long long b) {
        for (long long s = a; s < b; ++s) cnt[s + 1] = runs(s, false, 0);
    });
    for (long long s = 0; s < nsrc; ++s) cnt[s + 1] += cnt[s];
    const long long np = cnt[nsrc];
    std::vector<long long> tgt(np), src(np), lo(np), hi(np);
    o->tgt.resize(np); o->src.resize(np); o->lo.resize(np); o->hi.resize(np);
    rsc_parallel_chunks(nsrc, T, [&](int, long long a, long long b) {
        for (long long s = a; s < b; ++s) runs(s, true, cnt[s]);
    });
    // group by target, then source order (stable: counting sort on the target of a
    // source-order sorted list)
    std::vector<long long> perm(np);
    std::iota(perm.begin(), perm.end(), 0LL);
    std::stable_sort(perm.begin(), perm.end(), [&](long long a, long long b) {
        if (o->tgt[a] != o->tgt[b]) return o->tgt[a] < o->tgt[b];
        return src_order[o->src[a]] < src_order[o->src[b]];
    });
    for (long long q = 0; q < np; ++q) {
        tgt[q] = o->tgt[perm[q]]; src[q] = o->src[perm[q]]; lo[q] = o->lo[perm[q]]; hi[q] = o->hi[perm[q]];
    }
    o->tgt.swap(tgt); o->src.swap(src); o->lo.swap(lo); o->hi.swap(hi);
    // pass 2: index chunk
    o->cpos.resize(np);
    o->rpos.resize(np);
    long long off = 0;
    for (long long q = 0; q < np; ++q) {
        const long long nr = src_ptr[o->src[q] + 1] - src_ptr[o->src[q]];
        o->cpos[q] = off;
        off += o->hi[q] - o->lo[q];
        o->rpos[q] = off;
        off += nr - o->hi[q];
    }
    o->idx.resize(off);
    rsc_parallel_chunks(np, T, [&](int, long long a, long long b) {
        for (long long q = a; q < b; ++q) {
            const long long s = o->src[q], j = o->tgt[q];
            const long long *r = src_rows + src_ptr[s];
            const long long nr = src_ptr[s + 1] - src_ptr[s];
            const long long c0 = starts[j];
            int *c = o->idx.data() + o->cpos[q];
            for (long long p = o->lo[q]; p < o->hi[q]; ++p) *c++ = (int)(r[p] - c0);
            const long long *R = R_rows + R_ptr[j];
            const long long nR = R_ptr[j + 1] - R_ptr[j];
            int *rp = o->idx.data() + o->rpos[q];
            long long at = 0;
            for (long long p = o->hi[q]; p < nr; ++p) {  // rows ascending: a moving lower bound
                at += lbound(R + at, nR - at, r[p]);
                *rp++ = (int)at;
            }
        }
    });
    *npairs = np;
    *nidx = off;
    return o;
}

int rsc_plan_pairs_fetch(void *h, long long *tgt, long long *src, long long *lo, long long *hi, long long *cpos,
                         long long *rpos, int *idx) {
    auto *o = static_cast<PairsOut *>(h);
    if (!o) return -1;
    std::copy(o->tgt.begin(), o->tgt.end(), tgt);
    std::copy(o->src.begin(), o->src.end(), src);
    std::copy(o->lo.begin(), o->lo.end(), lo);
    std::copy(o->hi.begin(), o->hi.end(), hi);
    std::copy(o->cpos.begin(), o->cpos.end(), cpos);
    std::copy(o->rpos.begin(), o->rpos.end(), rpos);
    std::copy(o->idx.begin(), o->idx.end(), idx);
    delete o;
    return 0;
}

// Window maps of diagonal trees: tree t has nb = blk_ptr[t+1]-blk_ptr[t] blocks
// with global spans spans[4*b..] = (row lo, row hi, col lo, col hi) and the pairs
// [pair_ptr[t], pair_ptr[t+1]) of its supernode (source ids in pair_src, reference
// order).  For every (block, pair) with non-empty column and row windows:
// clo/chi/rlo/rhi = searchsorted(rows_s, bounds) and the index chunk
// cidx = rows[clo:chi] - col lo, ridx = rows[rlo:rhi] - row lo.  Output grouped by
// (tree, block), pairs in order within a block.
void *rsc_plan_tree_maps(long long ntree, const long long *blk_ptr, const long long *spans, const long long *pair_ptr,
                         const long long *pair_src, const long long *src_ptr, const long long *src_rows,
                         long long *nmaps, long long *nidx) {
    auto *o = new TreeOut();
    const long long nblk = blk_ptr[ntree];
    // per block: its tree and the kept (pair, clo, chi, rlo, rhi)
    struct Hit { long long s, clo, chi, rlo, rhi; };
    std::vector<std::vector<Hit>> per(nblk);
    std::vector<long long> tree_of(nblk);
    for (long long t = 0; t < ntree; ++t)
        for (long long b = blk_ptr[t]; b < blk_ptr[t + 1]; ++b) tree_of[b] = t;
    rsc_parallel_chunks(nblk, rsc_host_threads(), [&](int, long long a, long long e) {
        for (long long b = a; b < e; ++b) {
            const long long t = tree_of[b];
            const long long r0 = spans[4 * b], r1 = spans[4 * b + 1], c0 = spans[4 * b + 2], c1 = spans[4 * b + 3];
            for (long long q = pair_ptr[t]; q < pair_ptr[t + 1]; ++q) {
                const long long s = pair_src[q];
                const long long *r = src_rows + src_ptr[s];
                const long long n = src_ptr[s + 1] - src_ptr[s];
                const long long clo = lbound(r, n, c0), chi = lbound(r, n, c1);
                if (clo >= chi) continue;
                const long long rlo = lbound(r, n, r0), rhi = lbound(r, n, r1);
                if (rlo >= rhi) continue;
                per[b].push_back({s, clo, chi, rlo, rhi});
            }
        }
    });
    long long nm = 0, ni = 0;
    for (long long b = 0; b < nblk; ++b) {
        nm += (long long)per[b].size();
        for (auto &h : per[b]) ni += (h.chi - h.clo) + (h.rhi - h.rlo);
    }
    o->tree.resize(nm); o->blk.resize(nm); o->src.resize(nm); o->clo.resize(nm); o->chi.resize(nm);
    o->rlo.resize(nm); o->rhi.resize(nm); o->coff.resize(nm); o->roff.resize(nm);
    o->idx.resize(ni);
    std::vector<long long> mbase(nblk + 1, 0), ibase(nblk + 1, 0);
    for (long long b = 0; b < nblk; ++b) {
        mbase[b + 1] = mbase[b] + (long long)per[b].size();
        long long k = 0;
        for (auto &h : per[b]) k += (h.chi - h.clo) + (h.rhi - h.rlo);
        ibase[b + 1] = ibase[b] + k;
    }
    rsc_parallel_chunks(nblk, rsc_host_threads(), [&](int, long long a, long long e) {
        for (long long b = a; b < e; ++b) {
            const long long r0 = spans[4 * b], c0 = spans[4 * b + 2];
            long long m = mbase[b], ip = ibase[b];
            for (auto &h : per[b]) {
                const long long *r = src_rows + src_ptr[h.s];
                o->tree[m] = tree_of[b]; o->blk[m] = b - blk_ptr[tree_of[b]]; o->src[m] = h.s;
                o->clo[m] = h.clo; o->chi[m] = h.chi; o->rlo[m] = h.rlo; o->rhi[m] = h.rhi;
                o->coff[m] = ip;
                for (long long p = h.clo; p < h.chi; ++p) o->idx[ip++] = (int)(r[p] - c0);
                o->roff[m] = ip;
                for (long long p = h.rlo; p < h.rhi; ++p) o->idx[ip++] = (int)(r[p] - r0);
                ++m;
            }
        }
    });
    *nmaps = nm;
    *nidx = ni;
    return o;
}

// out: 9 arrays of nmaps (tree, block, src, clo, chi, rlo, rhi, cidx_off, ridx_off)
// and the index chunk
int rsc_plan_tree_maps_fetch(void *h, long long *const *out, int *idx) {
    auto *o = static_cast<TreeOut *>(h);
    if (!o) return -1;
    const std::vector<long long> *v[9] = {&o->tree, &o->blk, &o->src, &o->clo, &o->chi,
                                          &o->rlo, &o->rhi, &o->coff, &o->roff};
    for (int i = 0; i < 9; ++i) std::copy(v[i]->begin(), v[i]->end(), out[i]);
    std::copy(o->idx.begin(), o->idx.end(), idx);
    delete o;
    return 0;
}

// 64-bit digest of a byte buffer: 1 MiB chunks hashed independently (multiply-
// xorshift over 8-byte words, tail bytes folded in) on host threads, chunk
// digests combined in order -- independent of the thread count.
unsigned long long rsc_hash64(const void *data, long long nbytes) {
    const unsigned char *p = static_cast<const unsigned char *>(data);
    const long long CH = 1 << 20;
    const long long nch = nbytes > 0 ? (nbytes + CH - 1) / CH : 0;
    std::vector<unsigned long long> dig(nch);
    auto mix = [](unsigned long long h) {
        h ^= h >> 33; h *= 0xff51afd7ed558ccdULL; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ULL; h ^= h >> 33;
        return h;
    };
    rsc_parallel_chunks(nch, rsc_host_threads(), [&](int, long long a, long long b) {
        for (long long c = a; c < b; ++c) {
            const long long lo = c * CH, hi = std::min(nbytes, lo + CH);
            unsigned long long h = 0x9e3779b97f4a7c15ULL ^ (unsigned long long)c;
            long long i = lo;
            for (; i + 8 <= hi; i += 8) {
                unsigned long long w;
                __builtin_memcpy(&w, p + i, 8);
                h = mix(h ^ w) + 0x9e3779b97f4a7c15ULL;
            }
            for (; i < hi; ++i) h = mix(h ^ p[i]);
            dig[c] = h;
        }
    });
    unsigned long long h = 0x2545f4914f6cdd1dULL ^ (unsigned long long)nbytes;
    for (long long c = 0; c < nch; ++c) h = mix(h ^ dig[c]) * 0x100000001b3ULL;
    return h;
}

}  // extern "C"
