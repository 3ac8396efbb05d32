// Host-side geometric bisection step of the nested-dissection ordering
// (reference ordering.py:182-192 boundary rule with the coordinate split the
// geometric method uses).  One call replaces the numpy sort / neighbour-gather /
// boundary test of symbolic.py's _Dissector.split_by_order; the recursion and the
// separator tree stay in Python.  Results are a pure function of the inputs
// (unique sort keys), so they are identical to the numpy formulation.
#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <vector>

extern "C" {

// verts[nv]: vertex ids.  xyz: n x dim row-major coordinates.  mark: n bytes of
// zero scratch (left zero on return).  out[nv] <- side1, separator, side2 (each
// ascending in position order, i.e. ascending when verts is); counts[3] <- sizes.
// Returns 0 on a split, 1 when one side would be empty (no split), <0 on bad args.
int rsc_nd_split_geometric(long long nv, const long long *verts, int dim, const double *xyz,
                           const long long *indptr, const long long *indices, unsigned char *mark,
                           long long *out, long long *counts) {
    if (nv < 0 || dim < 1) return -1;
    if (nv == 0) { counts[0] = counts[1] = counts[2] = 0; return 1; }
    // widest axis (first on ties): argmax over max - min
    int axis = 0;
    double best = -1.0;
    for (int d = 0; d < dim; ++d) {
        double lo = xyz[verts[0] * dim + d], hi = lo;
        for (long long i = 1; i < nv; ++i) {
            const double v = xyz[verts[i] * dim + d];
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        const double w = hi - lo;
        if (d == 0 || w > best) { best = w; axis = d; }
    }
    // positions sorted by (coordinate along axis, vertex id)
    std::vector<long long> ord(nv);
    for (long long i = 0; i < nv; ++i) ord[i] = i;
    std::sort(ord.begin(), ord.end(), [&](long long a, long long b) {
        const double xa = xyz[verts[a] * dim + axis], xb = xyz[verts[b] * dim + axis];
        if (xa < xb) return true;
        if (xb < xa) return false;
        return verts[a] < verts[b];
    });
    const long long half = (nv + 1) / 2;
    std::sort(ord.begin(), ord.begin() + half);
    std::sort(ord.begin() + half, ord.end());
    for (long long i = 0; i < half; ++i) mark[verts[ord[i]]] = 1;
    std::vector<long long> s2;
    s2.reserve(nv - half);
    long long k = half;
    for (long long i = 0; i < half; ++i) out[i] = verts[ord[i]];
    for (long long i = half; i < nv; ++i) {
        const long long v = verts[ord[i]];
        bool hit = false;
        for (long long p = indptr[v]; p < indptr[v + 1]; ++p)
            if (mark[indices[p]]) { hit = true; break; }
        if (hit) out[k++] = v;
        else s2.push_back(v);
    }
    for (long long i = 0; i < half; ++i) mark[verts[ord[i]]] = 0;
    counts[0] = half;
    counts[1] = k - half;
    counts[2] = (long long)s2.size();
    std::copy(s2.begin(), s2.end(), out + k);
    return (half == 0 || s2.empty()) ? 1 : 0;
}

}  // extern "C"

// Whole geometric nested dissection (ordering.py:277-368 with the geometric split
// above): the recursion of symbolic.py _Dissector.dissect in one call, subtrees on
// host threads.  A subtree over `verts` (ascending) owns order[base, base+nv): its
// left part, then its right part, then its separator -- positions depend only on
// the part sizes, so subtrees are independent.  Each split is O(nv): the half with
// the smallest (coordinate, vertex id) keys comes from nth_element (the keys are
// unique, so the set equals the sorted prefix the Python formulation takes) and is
// marked in a stamp array (a unique stamp per split, so concurrent subtrees never
// see each other's marks).
#include <atomic>
#include <thread>

namespace {

struct NdCtx {
    int dim;
    const double *xyz;
    const long long *indptr, *indices;
    long long leaf;
    long long *order;
    int *stamp;                    // n ints, last split stamp that marked the vertex
    std::atomic<int> next_stamp{0};
    std::atomic<long long> next_node{0};
    long long cap;
    long long *n_lo, *n_hi, *n_sub, *n_lev, *n_left, *n_right;
    std::atomic<int> err{0};
    int par_depth;
};

long long nd_node(NdCtx &c, long long lo, long long hi, long long sub, long long lev, long long l, long long r) {
    const long long id = c.next_node.fetch_add(1);
    if (id >= c.cap) { c.err.store(-3); return -1; }
    c.n_lo[id] = lo; c.n_hi[id] = hi; c.n_sub[id] = sub; c.n_lev[id] = lev; c.n_left[id] = l; c.n_right[id] = r;
    return id;
}

// split verts (ascending) into side1 / sep / side2 (each ascending); false = no split
bool nd_split(NdCtx &c, const std::vector<long long> &verts, std::vector<long long> &s1, std::vector<long long> &sep,
              std::vector<long long> &s2) {
    const long long nv = (long long)verts.size();
    const int dim = c.dim;
    const double *xyz = c.xyz;
    int axis = 0;
    double best = -1.0;
    for (int d = 0; d < dim; ++d) {
        double lo = xyz[verts[0] * dim + d], hi = lo;
        for (long long i = 1; i < nv; ++i) {
            const double v = xyz[verts[i] * dim + d];
            lo = v < lo ? v : lo;
            hi = v > hi ? v : hi;
        }
        const double w = hi - lo;
        if (d == 0 || w > best) { best = w; axis = d; }
    }
    const long long half = (nv + 1) / 2;
    if (half == 0 || half == nv) return false;
    std::vector<long long> ord(nv);
    for (long long i = 0; i < nv; ++i) ord[i] = i;
    auto less = [&](long long a, long long b) {
        const double xa = xyz[verts[a] * dim + axis], xb = xyz[verts[b] * dim + axis];
        if (xa < xb) return true;
        if (xb < xa) return false;
        return verts[a] < verts[b];
    };
    std::nth_element(ord.begin(), ord.begin() + half, ord.end(), less);
    std::vector<unsigned char> first(nv, 0);
    for (long long i = 0; i < half; ++i) first[ord[i]] = 1;
    const int st = c.next_stamp.fetch_add(1) + 1;
    s1.clear(); sep.clear(); s2.clear();
    s1.reserve(half);
    for (long long i = 0; i < nv; ++i)
        if (first[i]) {
            s1.push_back(verts[i]);
            __atomic_store_n(&c.stamp[verts[i]], st, __ATOMIC_RELAXED);
        }
    for (long long i = 0; i < nv; ++i) {
        if (first[i]) continue;
        const long long v = verts[i];
        bool hit = false;
        for (long long p = c.indptr[v]; p < c.indptr[v + 1]; ++p)
            if (__atomic_load_n(&c.stamp[c.indices[p]], __ATOMIC_RELAXED) == st) { hit = true; break; }
        (hit ? sep : s2).push_back(v);
    }
    return !s2.empty();
}

long long nd_dissect(NdCtx &c, std::vector<long long> verts, long long base, long long level, int depth) {
    const long long nv = (long long)verts.size();
    if (c.err.load()) return -1;
    std::vector<long long> s1, sep, s2;
    if (nv <= c.leaf || !nd_split(c, verts, s1, sep, s2)) {
        std::copy(verts.begin(), verts.end(), c.order + base);
        return nd_node(c, base, base + nv, base, level, -1, -1);
    }
    std::vector<long long>().swap(verts);
    const long long n1 = (long long)s1.size(), n2 = (long long)s2.size();
    long long left = -1, right = -1;
    if (depth < c.par_depth && n1 + n2 > 4096) {
        std::thread th([&] { left = nd_dissect(c, std::move(s1), base, level + 1, depth + 1); });
        right = nd_dissect(c, std::move(s2), base + n1, level + 1, depth + 1);
        th.join();
    } else {
        left = nd_dissect(c, std::move(s1), base, level + 1, depth + 1);
        right = nd_dissect(c, std::move(s2), base + n1, level + 1, depth + 1);
    }
    const long long lo = base + n1 + n2;
    std::copy(sep.begin(), sep.end(), c.order + lo);
    return nd_node(c, lo, lo + (long long)sep.size(), base, level, left, right);
}

}  // namespace

extern "C" {

// order[n] <- dissection order (order[pos] = vertex); node arrays (capacity cap):
// lo, hi, subtree_lo, level, left, right (-1 = leaf).  Returns the node count
// (root in *root) or < 0 (-1 bad args, -3 capacity).
long long rsc_nd_geometric(long long n, int dim, const double *xyz, const long long *indptr,
                           const long long *indices, long long leaf, long long *order, long long cap, long long *n_lo,
                           long long *n_hi, long long *n_sub, long long *n_lev, long long *n_left,
                           long long *n_right, long long *root) {
    if (n < 1 || dim < 1 || leaf < 1) return -1;
    NdCtx c;
    c.dim = dim; c.xyz = xyz; c.indptr = indptr; c.indices = indices; c.leaf = leaf; c.order = order;
    std::vector<int> stamp(n, 0);
    c.stamp = stamp.data();
    c.cap = cap;
    c.n_lo = n_lo; c.n_hi = n_hi; c.n_sub = n_sub; c.n_lev = n_lev; c.n_left = n_left; c.n_right = n_right;
    unsigned hw = std::thread::hardware_concurrency();
    const char *e = getenv("RSC_HOST_THREADS");
    int T = e ? atoi(e) : (int)(hw ? hw : 1);
    T = std::max(1, std::min(T, 64));
    int d = 0;
    while ((1 << d) < 2 * T) ++d;  // ~2 subtrees per thread at the fork frontier
    c.par_depth = T > 1 ? d : 0;
    std::vector<long long> all(n);
    for (long long i = 0; i < n; ++i) all[i] = i;
    *root = nd_dissect(c, std::move(all), 0, 0, 0);
    if (c.err.load()) return c.err.load();
    return c.next_node.load();
}

}  // extern "C"

// Batched sub-block extraction from a CSR matrix with sorted column indices
// (the A-block cuts of the numeric plan, plan.py NumericPlan): request q takes
// rows  sel[r_off[q] .. +r_n[q])  (or the range [r_lo[q], r_lo[q]+r_n[q]) when
// r_off[q] < 0) and the columns likewise (c_off / c_n / c_lo; a column list must be
// ascending), with block-local row and column numbers.  Outputs, concatenated in
// request order: rowptr (int32, r_n[q]+1 block-local entries per request), colidx
// (int32) and val[p] = (int)data[p] - 1 of each kept entry p (the matrix
// stores 1-based positions as its values).  Pass 1 (rowptr == nullptr) only writes
// nnz[q]; pass 2 fills everything.  Requests run on all host threads.
#include <thread>

namespace {

struct Win {
    const long long *indptr, *indices, *sel, *r_off, *r_n, *r_lo, *c_off, *c_n, *c_lo;
    const double *data;
    long long n;
};

// one request; colmap: n ints of zero scratch (column list -> local + 1), left zero
template <bool FILL>
long long cut_one(const Win &w, long long q, int *colmap, int *rowptr, int *colidx, int *val) {
    const bool clist = w.c_off[q] >= 0;
    if (clist)
        for (long long i = 0; i < w.c_n[q]; ++i) colmap[w.sel[w.c_off[q] + i]] = (int)(i + 1);
    long long cnt = 0;
    if (FILL) rowptr[0] = 0;
    for (long long i = 0; i < w.r_n[q]; ++i) {
        const long long row = w.r_off[q] < 0 ? w.r_lo[q] + i : w.sel[w.r_off[q] + i];
        long long b = w.indptr[row], e = w.indptr[row + 1];
        if (!clist) {
            const long long lo = w.c_lo[q], hi = lo + w.c_n[q];
            b = std::lower_bound(w.indices + b, w.indices + e, lo) - w.indices;
            e = std::lower_bound(w.indices + b, w.indices + e, hi) - w.indices;
            if (FILL)
                for (long long p = b; p < e; ++p) {
                    colidx[cnt + p - b] = (int)(w.indices[p] - lo);
                    val[cnt + p - b] = (int)w.data[p] - 1;
                }
            cnt += e - b;
        } else {
            for (long long p = b; p < e; ++p) {
                const int loc = colmap[w.indices[p]];
                if (!loc) continue;
                if (FILL) {
                    colidx[cnt] = loc - 1;
                    val[cnt] = (int)w.data[p] - 1;
                }
                ++cnt;
            }
        }
        if (FILL) rowptr[i + 1] = (int)cnt;
    }
    if (clist)
        for (long long i = 0; i < w.c_n[q]; ++i) colmap[w.sel[w.c_off[q] + i]] = 0;
    return cnt;
}

}  // namespace

extern "C" int rsc_csr_windows(long long nq, long long n, const long long *indptr, const long long *indices,
                               const double *data, const long long *sel, const long long *r_off,
                               const long long *r_n, const long long *r_lo, const long long *c_off,
                               const long long *c_n, const long long *c_lo, long long *nnz,
                               const long long *rp_off, const long long *nz_off, int *rowptr, int *colidx,
                               int *val) {
    if (nq < 0 || n < 0) return -1;
    const Win w{indptr, indices, sel, r_off, r_n, r_lo, c_off, c_n, c_lo, data, n};
    unsigned nt = std::thread::hardware_concurrency();
    nt = nt ? (nt > 32 ? 32 : nt) : 1;
    if (nq < 64) nt = 1;
    std::vector<std::thread> pool;
    auto work = [&](unsigned t) {
        std::vector<int> colmap(n, 0);
        for (long long q = t; q < nq; q += nt) {
            if (rowptr)
                cut_one<true>(w, q, colmap.data(), rowptr + rp_off[q], colidx + nz_off[q], val + nz_off[q]);
            else
                nnz[q] = cut_one<false>(w, q, colmap.data(), nullptr, nullptr, nullptr);
        }
    };
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto &th : pool) th.join();
    return 0;
}
