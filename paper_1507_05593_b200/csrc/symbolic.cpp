// Host-side symbolic analysis kernels (C++, no device code): elimination tree,
// postorder and Cholesky column counts of the permuted lower-CSC matrix.
// These are the sequential union-find sweeps of the symbolic phase
// (reference symbolic.py:44-151); their results are unique for a given pattern,
// so any correct algorithm is bit-exact with the reference.
#include <cstdint>
#include <algorithm>
#include <vector>

#include <atomic>
#include <thread>
#include "host_par.h"

extern "C" {

// parent[j] = min{ i > j : L(i,j) != 0 } or -1 (Liu's algorithm with path
// compression over the rows of the strict lower triangle).
int rsc_sym_etree(long long n, const long long *col_ptr, const long long *row_idx, long long *parent) {
    if (n < 0) return -1;
    if (!col_ptr || !row_idx || !parent) return -2;
    // transpose the strict lower triangle to row lists (row i -> columns j < i, ascending)
    std::vector<long long> cnt(n + 1, 0);
    for (long long j = 0; j < n; ++j)
        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p)
            if (row_idx[p] > j) cnt[row_idx[p] + 1]++;
    for (long long i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<long long> pos(cnt.begin(), cnt.end() - 1), cols(cnt[n]);
    for (long long j = 0; j < n; ++j)
        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            const long long i = row_idx[p];
            if (i > j) cols[pos[i]++] = j;
        }
    std::vector<long long> anc(n, -1);
    for (long long i = 0; i < n; ++i) parent[i] = -1;
    for (long long i = 0; i < n; ++i) {
        for (long long p = cnt[i]; p < cnt[i + 1]; ++p) {
            long long j = cols[p];
            while (true) {
                const long long a = anc[j];
                anc[j] = i;
                if (a == -1) { parent[j] = i; break; }
                if (a == i) break;
                j = a;
            }
        }
    }
    return 0;
}

// The same elimination tree with the rows of nr disjoint column ranges (ND
// subtrees: an entry (i, j), j < i, with j inside a range has i inside it or in no
// range) processed on host threads first, each range's own row lists transposed
// locally; the remaining rows follow in ascending order.  Liu's row sweep gives the
// unique etree in any processing order that keeps each row's ancestors current, and
// a range's walks only touch its own columns.  Returns 1 (parent untouched) when the
// ranges are not closed, so the caller can fall back.
int rsc_sym_etree_par(long long n, const long long *col_ptr, const long long *row_idx, long long nr,
                      const long long *ranges, long long *parent) {
    if (n < 0) return -1;
    if (!col_ptr || !row_idx || !parent) return -2;
    std::vector<int> rng(n, -1);
    for (long long r = 0; r < nr; ++r)
        for (long long c = ranges[2 * r]; c < ranges[2 * r + 1]; ++c) rng[c] = (int)r;
    std::vector<long long> anc(n, -1);
    for (long long i = 0; i < n; ++i) parent[i] = -1;
    auto walk = [&](long long i, long long j) {
        while (true) {
            const long long a = anc[j];
            anc[j] = i;
            if (a == -1) { parent[j] = i; break; }
            if (a == i) break;
            j = a;
        }
    };
    std::atomic<bool> bad{false};
    {
        std::atomic<long long> next{0};
        const int T = std::max(1, std::min<int>(rsc_host_threads(), (int)nr));
        std::vector<std::thread> th;
        for (int w = 0; w < T; ++w)
            th.emplace_back([&] {
                std::vector<long long> cnt, cols;
                for (long long r; (r = next.fetch_add(1)) < nr;) {
                    const long long lo = ranges[2 * r], hi = ranges[2 * r + 1];
                    cnt.assign(hi - lo + 1, 0);
                    for (long long j = lo; j < hi; ++j)
                        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
                            const long long i = row_idx[p];
                            if (i <= j) continue;
                            if (i < hi) cnt[i - lo + 1]++;
                            else if (rng[i] >= 0) bad = true;  // reaches another range
                        }
                    for (long long q = 0; q < hi - lo; ++q) cnt[q + 1] += cnt[q];
                    cols.resize(cnt[hi - lo]);
                    std::vector<long long> pos(cnt.begin(), cnt.end() - 1);
                    for (long long j = lo; j < hi; ++j)
                        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
                            const long long i = row_idx[p];
                            if (i > j && i < hi) cols[pos[i - lo]++] = j;
                        }
                    for (long long i = lo; i < hi; ++i)
                        for (long long q = cnt[i - lo]; q < cnt[i - lo + 1]; ++q) walk(i, cols[q]);
                }
            });
        for (auto &x : th) x.join();
    }
    if (bad) return 1;
    // rows outside every range, ascending: their (strict lower) entries from all columns
    std::vector<long long> cnt(n + 1, 0);
    for (long long j = 0; j < n; ++j)
        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            const long long i = row_idx[p];
            if (i > j && rng[i] < 0) cnt[i + 1]++;
        }
    for (long long i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
    std::vector<long long> pos(cnt.begin(), cnt.end() - 1), cols(cnt[n]);
    for (long long j = 0; j < n; ++j)
        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            const long long i = row_idx[p];
            if (i > j && rng[i] < 0) cols[pos[i]++] = j;
        }
    for (long long i = 0; i < n; ++i)
        if (rng[i] < 0)
            for (long long q = cnt[i]; q < cnt[i + 1]; ++q) walk(i, cols[q]);
    return 0;
}

// postorder of the forest, children visited in ascending index, roots ascending
int rsc_sym_postorder(long long n, const long long *parent, long long *post) {
    if (n < 0) return -1;
    std::vector<long long> head(n, -1), next(n, -1), stack;
    for (long long j = n - 1; j >= 0; --j) {
        const long long p = parent[j];
        if (p != -1) { next[j] = head[p]; head[p] = j; }
    }
    long long k = 0;
    stack.reserve(64);
    for (long long r = 0; r < n; ++r) {
        if (parent[r] != -1) continue;
        stack.push_back(r);
        while (!stack.empty()) {
            const long long v = stack.back();
            const long long c = head[v];
            if (c != -1) { head[v] = next[c]; stack.push_back(c); }
            else { post[k++] = v; stack.pop_back(); }
        }
    }
    return 0;
}

// Column counts of L (diagonal included): skeleton-matrix / least-common-ancestor
// counting over the postorder (Gilbert, Ng & Peyton).
int rsc_sym_colcounts(long long n, const long long *col_ptr, const long long *row_idx, const long long *parent,
                      const long long *post, long long *counts) {
    if (n < 0) return -1;
    std::vector<long long> first(n, -1), delta(n, 0), maxfirst(n, -1), prevleaf(n, -1), anc(n);
    for (long long k = 0; k < n; ++k) {
        long long j = post[k];
        delta[j] = (first[j] == -1) ? 1 : 0;
        while (j != -1 && first[j] == -1) { first[j] = k; j = parent[j]; }
    }
    for (long long i = 0; i < n; ++i) anc[i] = i;
    for (long long k = 0; k < n; ++k) {
        const long long j = post[k];
        if (parent[j] != -1) delta[parent[j]]--;
        for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
            const long long i = row_idx[p];
            if (i <= j || first[j] <= maxfirst[i]) continue;
            maxfirst[i] = first[j];
            const long long jprev = prevleaf[i];
            prevleaf[i] = j;
            if (jprev == -1) {
                delta[j]++;
            } else {
                long long q = jprev;
                while (q != anc[q]) q = anc[q];
                delta[j]++;
                delta[q]--;
                long long s = jprev;
                while (s != q) { const long long sn = anc[s]; anc[s] = q; s = sn; }
            }
        }
        if (parent[j] != -1) anc[j] = parent[j];
    }
    for (long long j = 0; j < n; ++j) counts[j] = delta[j];
    for (long long j = 0; j < n; ++j)
        if (parent[j] != -1) counts[parent[j]] += counts[j];
    return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Relaxed supernode amalgamation of one gap of fundamental supernodes
// (symbolic.py:_amalgamate, reference symbolic.py:244-277): merge a supernode into
// its successor while the successor is the parent of its last column and the
// explicit-zero fraction stays under the width tier's bound.  bounds[0..nb] are the
// fundamental boundaries; the kept starts are written to out (count returned).
// tiers: ntier (width, bound) pairs, width < 0 = unbounded.  The fraction is the same
// IEEE double division Python performs on the exact integers.
extern "C" long long rsc_sym_amalgamate(long long nb, const long long *bounds, const long long *parent,
                                        const long long *counts, int ntier, const long long *tw,
                                        const double *tb, long long *out) {
    if (nb < 0) return -1;
    std::vector<long long> st, nc, nr, zr;
    st.reserve(nb);
    for (long long i = 0; i < nb; ++i) {
        st.push_back(bounds[i]);
        nc.push_back(bounds[i + 1] - bounds[i]);
        nr.push_back(counts[bounds[i]] - (bounds[i + 1] - bounds[i]));
        zr.push_back(0);
    }
    // singly linked list over the surviving supernodes (Python deletes from lists)
    std::vector<long long> nxt(nb);
    for (long long i = 0; i < nb; ++i) nxt[i] = i + 1;
    long long i = 0;
    while (i < nb && nxt[i] < nb) {
        const long long s = nxt[i];
        const long long last = st[i] + nc[i] - 1;
        if (parent[last] != st[s]) { i = s; continue; }
        const long long ns = nc[i], nt = nc[s], rs = nr[i], rt = nr[s];
        const long long mc = ns + nt;
        const long long tot = zr[i] + zr[s] + ns * (nt + rt - rs);
        const double frac = (double)tot / (double)(mc * (mc + 1) / 2 + mc * rt);
        bool ok = false;
        for (int q = 0; q < ntier; ++q) {
            if (tw[q] < 0 || mc <= tw[q]) {
                ok = frac < tb[q] || tb[q] >= 1.0;
                break;
            }
        }
        if (ok) {
            nc[i] = mc; nr[i] = rt; zr[i] = tot;
            nxt[i] = nxt[s];
        } else {
            i = s;
        }
    }
    long long k = 0;
    for (long long j = 0; j < nb; j = nxt[j]) out[k++] = st[j];
    return k;
}

// Row structures R_j of every supernode (symbolic.py:compute_row_structures,
// reference symbolic.py:280-306): the rows >= c1 of A's columns c0..c1 united with
// the pieces the children pass up (their rows beyond the parent's columns).
// Two calls: compute (returns a handle and the total row count), then fetch
// (ptr[M+1], rows[total]) which frees the handle.
struct RowStructs {
    std::vector<long long> ptr, rows;
};

namespace {

// The sequential sweep over supernodes [j0, j1): R_j into rows[j], pieces for
// targets t in [j0, j1) into pending[t], pieces for targets outside into outbox.
void rows_sweep(long long j0, long long j1, long long M, const long long *starts, const long long *col_ptr,
                const long long *row_idx, std::vector<std::vector<long long>> &pending,
                std::vector<std::vector<long long>> &rows,
                std::vector<std::pair<long long, std::vector<long long>>> *outbox, const char *done = nullptr,
                bool *bad = nullptr) {
    std::vector<long long> buf;
    for (long long j = j0; j < j1; ++j) {
        const long long c0 = starts[j], c1 = starts[j + 1];
        buf.swap(pending[j]);
        std::vector<long long>().swap(pending[j]);
        for (long long p = col_ptr[c0]; p < col_ptr[c1]; ++p)
            if (row_idx[p] >= c1) buf.push_back(row_idx[p]);
        std::sort(buf.begin(), buf.end());
        buf.erase(std::unique(buf.begin(), buf.end()), buf.end());
        rows[j].assign(buf.begin(), buf.end());
        if (!buf.empty()) {
            // supernode t containing the first row; pass up the rows beyond its columns
            const long long t = (long long)(std::upper_bound(starts, starts + M + 1, buf[0]) - starts) - 1;
            const long long t1 = starts[t + 1];
            auto it = std::lower_bound(buf.begin(), buf.end(), t1);
            if (done && done[t]) *bad = true;  // a piece for an already swept range
            if (t < j1 || !outbox) pending[t].insert(pending[t].end(), it, buf.end());
            else if (it != buf.end()) outbox->emplace_back(t, std::vector<long long>(it, buf.end()));
        }
        buf.clear();
    }
}

}  // namespace

// nr disjoint supernode ranges [ranges[2i], ranges[2i+1]) closed under the
// pass-up (ND subtrees: every piece goes to a supernode inside the range or after
// it) are swept on host threads first; the rest sequentially after merging the
// ranges' outgoing pieces.  A piece's content does not depend on the order pieces
// arrive (each R_j is sorted and de-duplicated), so the result equals the
// sequential sweep.  nr = 0: fully sequential.
extern "C" void *rsc_sym_rows_compute_par(long long M, const long long *starts, const long long *col_ptr,
                                          const long long *row_idx, long long nr, const long long *ranges,
                                          long long *total) {
    auto *h = new RowStructs();
    h->ptr.assign(M + 1, 0);
    std::vector<std::vector<long long>> pending(M), rows(M);
    std::vector<char> done(M, 0);
    if (nr > 0) {
        std::vector<std::vector<std::pair<long long, std::vector<long long>>>> out(nr);
        const int T = std::max(1, std::min<int>(rsc_host_threads(), (int)nr));
        std::atomic<long long> next{0};
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&] {
                for (long long r; (r = next.fetch_add(1)) < nr;)
                    rows_sweep(ranges[2 * r], ranges[2 * r + 1], M, starts, col_ptr, row_idx, pending, rows, &out[r]);
            });
        for (auto &x : th) x.join();
        for (long long r = 0; r < nr; ++r)
            for (long long j = ranges[2 * r]; j < ranges[2 * r + 1]; ++j) done[j] = 1;
        bool bad = false;
        for (long long r = 0; r < nr; ++r)
            for (auto &pc : out[r]) {
                bad |= done[pc.first] != 0;
                pending[pc.first].insert(pending[pc.first].end(), pc.second.begin(), pc.second.end());
            }
        for (long long j = 0; j < M && !bad;) {  // the remaining supernodes, in order
            if (done[j]) { ++j; continue; }
            long long e = j;
            while (e < M && !done[e]) ++e;
            rows_sweep(j, e, M, starts, col_ptr, row_idx, pending, rows, nullptr, done.data(), &bad);
            j = e;
        }
        if (bad) {  // the ranges were not closed under the pass-up: sequential sweep
            for (auto &v : pending) std::vector<long long>().swap(v);
            rows_sweep(0, M, M, starts, col_ptr, row_idx, pending, rows, nullptr);
        }
    } else {
        rows_sweep(0, M, M, starts, col_ptr, row_idx, pending, rows, nullptr);
    }
    for (long long j = 0; j < M; ++j) h->ptr[j + 1] = h->ptr[j] + (long long)rows[j].size();
    h->rows.resize(h->ptr[M]);
    rsc_parallel_chunks(M, rsc_host_threads(), [&](int, long long lo, long long hi) {
        for (long long j = lo; j < hi; ++j) std::copy(rows[j].begin(), rows[j].end(), h->rows.begin() + h->ptr[j]);
    });
    *total = h->ptr[M];
    return h;
}

extern "C" void *rsc_sym_rows_compute(long long M, const long long *starts, const long long *col_ptr,
                                      const long long *row_idx, long long *total) {
    return rsc_sym_rows_compute_par(M, starts, col_ptr, row_idx, 0, nullptr, total);
}

extern "C" int rsc_sym_rows_fetch(void *handle, long long *ptr, long long *rows) {
    auto *h = static_cast<RowStructs *>(handle);
    if (!h) return -1;
    std::copy(h->ptr.begin(), h->ptr.end(), ptr);
    std::copy(h->rows.begin(), h->rows.end(), rows);
    delete h;
    return 0;
}

// ---------------------------------------------------------------------------
// Full symmetric CSR (both triangles, rows sorted) of a lower-CSC matrix in one
// column-order pass: column j appends j to the rows of its entries (i, j), i >= j,
// and its entries i > j to row j -- rows come out sorted without a sort.
// With values, stored zeros are dropped (what scipy's low + tril(low, -1).T does);
// adjacency != 0 also drops the diagonal ((full - diag(full)).eliminate_zeros(), the
// ND adjacency of symbolic.py:_adjacency).  values may be null (pattern only).
// Returns the entry count (<0: bad argument).
extern "C" long long rsc_sym_full_csr(long long n, const long long *col_ptr, const long long *row_idx,
                                      const double *values, int adjacency, long long *indptr,
                                      long long *indices, double *data) {
    if (n < 0 || !col_ptr || !row_idx || !indptr || !indices) return -1;
    if (adjacency && !values) return -2;
    // Row r of the full matrix = [j < r : (r, j) stored in column j] ascending j
    //                           ++ [i >= r : (i, r) stored in column r] ascending i.
    // The first part is a transpose of the strict lower triangle, done in parallel
    // over column chunks with per-chunk row counts (chunk t's entries of row r go
    // after chunks < t, columns ascending inside a chunk: rows come out sorted and
    // the result is independent of the thread count).
    auto keep = [&](long long p, long long i, long long j) {
        return !((values && values[p] == 0.0) || (adjacency && i == j));
    };
    const int T = (int)std::min<long long>(rsc_host_threads(), std::max<long long>(1, col_ptr[n] / 200000));
    const std::vector<long long> cut = rsc_balanced_cuts(n, col_ptr, T);
    std::vector<std::vector<int>> cnt(T);
    std::vector<long long> bcnt(n, 0);
    rsc_parallel_chunks(T, T, [&](int, long long t0, long long t1) {
        for (long long t = t0; t < t1; ++t) {
            cnt[t].assign(n, 0);
            for (long long j = cut[t]; j < cut[t + 1]; ++j) {
                long long b = 0;
                for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
                    const long long i = row_idx[p];
                    if (!keep(p, i, j)) continue;
                    if (i > j) cnt[t][i]++;
                    if (i >= j) ++b;
                }
                bcnt[j] = b;
            }
        }
    });
    // row sizes and per-chunk offsets
    indptr[0] = 0;
    std::vector<long long> acnt(n, 0);
    rsc_parallel_chunks(n, T, [&](int, long long r0, long long r1) {
        for (long long r = r0; r < r1; ++r) {
            long long a = 0;
            for (int t = 0; t < T; ++t) a += cnt[t][r];
            acnt[r] = a;
        }
    });
    for (long long r = 0; r < n; ++r) indptr[r + 1] = indptr[r] + acnt[r] + bcnt[r];
    rsc_parallel_chunks(n, T, [&](int, long long r0, long long r1) {
        for (long long r = r0; r < r1; ++r) {
            long long o = indptr[r];
            for (int t = 0; t < T; ++t) {
                const int c = cnt[t][r];
                cnt[t][r] = (int)(o - indptr[r]);  // chunk t's first slot in row r (offset)
                o += c;
            }
        }
    });
    rsc_parallel_chunks(T, T, [&](int, long long t0, long long t1) {
        for (long long t = t0; t < t1; ++t)
            for (long long j = cut[t]; j < cut[t + 1]; ++j) {
                long long q2 = indptr[j] + acnt[j];  // this column's own row j: rows i >= j
                for (long long p = col_ptr[j]; p < col_ptr[j + 1]; ++p) {
                    const long long i = row_idx[p];
                    if (!keep(p, i, j)) continue;
                    if (i > j) {
                        const long long q = indptr[i] + cnt[t][i]++;
                        indices[q] = j;
                        if (data) data[q] = values[p];
                    }
                    if (i >= j) {
                        indices[q2] = i;
                        if (data) data[q2] = values[p];
                        ++q2;
                    }
                }
            }
    });
    return indptr[n];
}

// Lower-storage (row, col) of every entry of A under the permutation p, sorted by
// (col, row), with the source position of each (symmetric permutation,
// sparse.py:171-189): a counting pass by permuted column, then per-column row sorts
// in parallel.
extern "C" int rsc_sym_permute_lower(long long n, const long long *col_ptr, const long long *row_idx,
                                     const long long *p, long long *out_rows, long long *out_cols,
                                     long long *order) {
    if (n < 0 || !col_ptr || !row_idx || !p) return -1;
    const long long nnz = col_ptr[n];
    const int T = (int)std::min<long long>(rsc_host_threads(), std::max<long long>(1, nnz / 200000));
    const std::vector<long long> src = rsc_balanced_cuts(n, col_ptr, T);  // source-column chunks
    // per-chunk counts of every permuted column (chunk order = source order, so the
    // unsorted runs are deterministic; the per-column sort fixes the final order)
    std::vector<std::vector<int>> cnt(T);
    rsc_parallel_chunks(T, T, [&](int, long long t0, long long t1) {
        for (long long t = t0; t < t1; ++t) {
            cnt[t].assign(n, 0);
            for (long long j = src[t]; j < src[t + 1]; ++j)
                for (long long e = col_ptr[j]; e < col_ptr[j + 1]; ++e) {
                    const long long a = p[row_idx[e]], b = p[j];
                    cnt[t][a < b ? a : b]++;
                }
        }
    });
    std::vector<long long> cp(n + 1, 0);
    rsc_parallel_chunks(n, T, [&](int, long long c0, long long c1) {
        for (long long c = c0; c < c1; ++c) {
            long long s = 0;
            for (int t = 0; t < T; ++t) s += cnt[t][c];
            cp[c + 1] = s;
        }
    });
    for (long long c = 0; c < n; ++c) cp[c + 1] += cp[c];
    rsc_parallel_chunks(n, T, [&](int, long long c0, long long c1) {
        for (long long c = c0; c < c1; ++c) {
            long long o = cp[c];
            for (int t = 0; t < T; ++t) {
                const int k = cnt[t][c];
                cnt[t][c] = (int)(o - cp[c]);
                o += k;
            }
        }
    });
    std::vector<std::pair<long long, long long>> tmp(nnz);
    rsc_parallel_chunks(T, T, [&](int, long long t0, long long t1) {
        for (long long t = t0; t < t1; ++t)
            for (long long j = src[t]; j < src[t + 1]; ++j)
                for (long long e = col_ptr[j]; e < col_ptr[j + 1]; ++e) {
                    const long long a = p[row_idx[e]], b = p[j];
                    const long long c = a < b ? a : b, r = a < b ? b : a;
                    tmp[cp[c] + cnt[t][c]++] = {r, e};
                }
    });
    const std::vector<long long> cut = rsc_balanced_cuts(n, cp.data(), T);
    rsc_parallel_chunks(T, T, [&](int, long long t0, long long t1) {
        for (long long t = t0; t < t1; ++t)
            for (long long c = cut[t]; c < cut[t + 1]; ++c) {
                std::sort(tmp.begin() + cp[c], tmp.begin() + cp[c + 1]);
                for (long long q = cp[c]; q < cp[c + 1]; ++q) {
                    out_rows[q] = tmp[q].first;
                    out_cols[q] = c;
                    order[q] = tmp[q].second;
                }
            }
    });
    return 0;
}
