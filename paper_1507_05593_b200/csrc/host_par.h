// Minimal host thread-parallel loop for the symbolic phase's O(nnz) passes.
// RSC_HOST_THREADS overrides the thread count (default: hardware threads, <= 32).
#pragma once
#include <algorithm>
#include <cstdlib>
#include <thread>
#include <vector>

inline int rsc_host_threads() {
    static const int nt = [] {
        const char *e = getenv("RSC_HOST_THREADS");
        int v = e ? atoi(e) : (int)std::thread::hardware_concurrency();
        return std::max(1, std::min(v, 32));
    }();
    return nt;
}

// fn(t, lo, hi) on T contiguous pieces of [0, n) (T <= rsc_host_threads()).
template <class F>
void rsc_parallel_chunks(long long n, int T, F fn) {
    if (T <= 1 || n < 2) {
        fn(0, 0LL, n);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    for (int t = 0; t < T; ++t) {
        const long long lo = n * t / T, hi = n * (t + 1) / T;
        th.emplace_back([=] { fn(t, lo, hi); });
    }
    for (auto &x : th) x.join();
}

// Split [0, n) into T ranges of roughly equal weight w[0..n) given its prefix sums
// (pref[n+1], non-decreasing): returns the T+1 boundaries.
inline std::vector<long long> rsc_balanced_cuts(long long n, const long long *pref, int T) {
    std::vector<long long> cut(T + 1, 0);
    cut[T] = n;
    const long long tot = pref[n];
    for (int t = 1; t < T; ++t) {
        const long long target = tot * t / T;
        cut[t] = std::lower_bound(pref, pref + n + 1, target) - pref;
        cut[t] = std::max(cut[t], cut[t - 1]);
    }
    return cut;
}
