// Dependency graph of the preconditioner apply as one dataflow program
// (factor.py:175-218; the kernel is apply_flow_kernel in apply.cu).
//
// Input: the apply's GEMV ops in a valid sequential order (the level phases of both
// sweeps, apply.py), each with the vector elements it reads (x) and writes (y): a
// contiguous range or an index list into one of the program's vectors (y, y2, the
// low-rank intermediates).  Output: for every op the number of predecessors it must
// wait for and its successor list (CSR) -- the read-after-write, write-after-read and
// write-after-write hazards of the sequential order, where accumulations into the
// same element commute (FP64 atomics at L2) and an assignment does not.
//
// Hazards are tracked per *segment*: the vector elements are cut at the start of every
// contiguous access (unit columns, tree-node ranges, low-rank intermediates), and an
// indexed access (a unit's row structure) touches the segments its indices fall in.
// A segment is one conflict unit, which is conservative (never misses a hazard).
// Because a low-rank intermediate of capacity `cap` starts its own segment and the
// next one starts `cap` elements later, the graph does not depend on kept ranks <= cap.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" long long rsc_flow_deps(int nops, const long long *xaddr, const long long *xidx, const int *xlen,
                                   const long long *yaddr, const long long *yidx, const int *ylen,
                                   const int *yassign, int nbuf, const long long *buf_base,
                                   const long long *buf_len, const int *idx_host, long long idx_dev,
                                   long long idx_len, int *need, int *succ_ptr, int *succ, long long succ_cap) {
    if (nops < 0 || nbuf <= 0) return -1;
    if (nops == 0) { succ_ptr[0] = 0; return 0; }
    // element id space: buffers back to back
    std::vector<long long> eoff(nbuf + 1, 0);
    for (int b = 0; b < nbuf; ++b) eoff[b + 1] = eoff[b] + buf_len[b];
    const long long nel = eoff[nbuf];
    auto elem = [&](long long addr) -> long long {
        for (int b = 0; b < nbuf; ++b) {
            const long long off = addr - buf_base[b];
            if (off >= 0 && off < 8 * buf_len[b]) return eoff[b] + off / 8;
        }
        return -1;
    };
    auto host_idx = [&](long long dev) -> const int * {
        const long long o = (dev - idx_dev) / 4;
        if (dev < idx_dev || o >= idx_len) return nullptr;
        return idx_host + o;
    };
    // segment starts
    std::vector<long long> xe(nops), ye(nops);
    std::vector<char> cut(nel + 1, 0);
    for (int b = 0; b <= nbuf; ++b) cut[std::min(eoff[b], nel)] = 1;
    for (int o = 0; o < nops; ++o) {
        xe[o] = elem(xaddr[o]);
        ye[o] = elem(yaddr[o]);
        if (xe[o] < 0 || ye[o] < 0) return -2;
        if (!xidx[o]) cut[xe[o]] = 1;
        if (!yidx[o]) cut[ye[o]] = 1;
    }
    std::vector<int> seg(nel);
    int ns = -1;
    for (long long e = 0; e < nel; ++e) {
        if (cut[e]) ++ns;
        seg[e] = ns;
    }
    ++ns;
    // W: the writers of the current epoch (one assignment, or accumulations that commute
    // with each other); R: readers since; base: the ops every member of W must follow
    std::vector<std::vector<int>> W(ns), R(ns), base(ns);
    std::vector<char> wassign(ns, 0);
    std::vector<int> stamp(ns, -1), pstamp(nops, -1);
    std::vector<std::vector<int>> preds(nops);
    std::vector<int> segs;
    auto collect = [&](int o, long long base, long long dev_idx, int len) -> int {
        segs.clear();
        if (len <= 0) return 0;
        if (!dev_idx) {
            const long long e1 = base + len - 1;
            if (e1 >= nel) return -3;
            for (int s = seg[base]; s <= seg[e1]; ++s) segs.push_back(s);
            return 0;
        }
        const int *ix = host_idx(dev_idx);
        if (!ix || (dev_idx - idx_dev) / 4 + len > idx_len) return -4;
        int last = -1;
        for (int k = 0; k < len; ++k) {
            const long long e = base + ix[k];
            if (e < 0 || e >= nel) return -3;
            const int s = seg[e];
            if (s == last || stamp[s] == o) continue;
            stamp[s] = o;
            last = s;
            segs.push_back(s);
        }
        return 0;
    };
    auto addpred = [&](int o, int p) {
        if (p == o || pstamp[p] == o) return;
        pstamp[p] = o;
        preds[o].push_back(p);
    };
    for (int o = 0; o < nops; ++o) {
        // reads: after every outstanding writer
        int rc = collect(o, xe[o], xidx[o], xlen[o]);
        if (rc) return rc;
        for (int s : segs) {
            for (int p : W[s]) addpred(o, p);
            if (R[s].empty() || R[s].back() != o) R[s].push_back(o);
        }
        // writes: after the readers since the last write; accumulations commute
        rc = collect(nops + o, ye[o], yidx[o], ylen[o]);  // stamp space offset: no clash with reads
        if (rc) return rc;
        const bool asg = yassign[o] != 0;
        for (int s : segs) {
            if (!R[s].empty()) {
                for (int p : R[s]) addpred(o, p);
                base[s].swap(R[s]);
                R[s].clear();
                W[s].assign(1, o);
                wassign[s] = asg;
            } else if (asg || wassign[s]) {
                for (int p : W[s]) addpred(o, p);
                base[s].swap(W[s]);
                W[s].assign(1, o);
                wassign[s] = asg;
            } else {  // an accumulation joins the epoch: after what the epoch follows
                for (int p : base[s]) addpred(o, p);
                W[s].push_back(o);
            }
        }
    }
    // successor CSR
    std::vector<int> cnt(nops + 1, 0);
    long long ne = 0;
    for (int o = 0; o < nops; ++o) {
        need[o] = (int)preds[o].size();
        ne += need[o];
        for (int p : preds[o]) ++cnt[p + 1];
    }
    if (ne > succ_cap) return ne;  // caller retries with a larger buffer
    succ_ptr[0] = 0;
    for (int o = 0; o < nops; ++o) succ_ptr[o + 1] = succ_ptr[o] + cnt[o + 1];
    std::vector<int> fill(succ_ptr, succ_ptr + nops);
    for (int o = 0; o < nops; ++o)
        for (int p : preds[o]) succ[fill[p]++] = o;
    return ne;
}
