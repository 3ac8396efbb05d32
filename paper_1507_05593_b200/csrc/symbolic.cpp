// Host-side symbolic analysis kernels (C++, no device code): elimination tree,
// postorder and Cholesky column counts of the permuted lower-CSC matrix.
// These are the sequential union-find sweeps of the symbolic phase
// (reference symbolic.py:44-151); their results are unique for a given pattern,
// so any correct algorithm is bit-exact with the reference.
#include <cstdint>
#include <vector>

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
