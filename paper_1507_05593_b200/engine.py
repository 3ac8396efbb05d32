"""Device-level wrappers over the C ABI, operating on torch CUDA tensors.

torch is used only as the device allocator and stream owner; every FLOP runs in
librsc_b200.so.  Matrices are row-major FP64 views `(tensor, rows, cols, ld)` or
plain 2-D tensors with unit column stride.
"""

import os

import numpy as np
import torch

from . import _lib
from ._lib import GEMM_DTYPE, addr, check, int_array, ptr_array

F64 = torch.float64
I32 = torch.int32


_CUDA_OK = False


def require_cuda():
    global _CUDA_OK
    if not _CUDA_OK:
        if not torch.cuda.is_available():
            raise RuntimeError("rsc_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
        _CUDA_OK = True
    return _lib.load()


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle():
    """cudaStream_t of torch's current stream (the capture stream inside a graph
    capture).  The raw accessor skips building a torch.cuda.Stream object per call
    (tens of thousands of calls per one-shot numeric pass)."""
    if _RAW_STREAM is not None:
        return _RAW_STREAM(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def dev():
    return torch.device("cuda", torch.cuda.current_device())


def empty(*shape, dtype=F64):
    return torch.empty(*shape, dtype=dtype, device=dev())


def zeros(*shape, dtype=F64):
    return torch.zeros(*shape, dtype=dtype, device=dev())


class gc_paused:
    """Pause Python's cyclic collector for the duration of a host-bound call: a
    one-shot factorization builds ~10^6 short-lived descriptor objects (arrays, views,
    tuples, none of them in reference cycles), and every generation-0/1/2 scan of the
    collector walks the long-lived plan objects again.  Re-enabled on exit when it was
    enabled on entry; RSC_GC=1 leaves the collector alone."""

    _keep = os.environ.get("RSC_GC") == "1"

    def __enter__(self):
        import gc

        self.was = gc.isenabled() and not self._keep
        if self.was:
            gc.disable()
        return self

    def __exit__(self, *exc):
        if self.was:
            import gc

            gc.enable()
        return False


_CHUNK_POOL = []  # device chunks of dead arenas, reused before any new cudaMalloc


def _take_chunk(n):
    best = None
    for i, c in enumerate(_CHUNK_POOL):
        if c.numel() >= n and (best is None or c.numel() < _CHUNK_POOL[best].numel()):
            best = i
    if best is not None:
        return _CHUNK_POOL.pop(best)
    return torch.empty(n, dtype=F64, device=dev())


class Arena:
    """Bump allocator over large FP64 device chunks.

    The numeric pass creates tens of thousands of small blocks; carving them out of
    a few big allocations keeps cudaMalloc (and its implicit device syncs) off the
    critical path.  Single-stream use only: memory handed out again after
    reset() is reused by kernels that are stream-ordered after the earlier ones.
    """

    ALIGN = 32  # doubles (256 B)

    def __init__(self, chunk_elems=1 << 25):
        self.chunk = int(chunk_elems)
        self.chunks = []
        self.i = 0
        self.off = 0

    def empty(self, *shape):
        n = 1
        for s in shape:
            n *= int(s)
        need = max(-(-n // self.ALIGN) * self.ALIGN, self.ALIGN)
        while True:
            if self.i < len(self.chunks):
                buf = self.chunks[self.i]
                if self.off + need <= buf.numel():
                    t = buf[self.off:self.off + n].view(*shape) if n else buf[:0].view(*shape)
                    self.off += need
                    return t
                self.i += 1
                self.off = 0
                continue
            self.chunks.append(_take_chunk(max(self.chunk, need)))

    def __del__(self):
        try:
            for c in self.chunks:
                _CHUNK_POOL.append(c)
            self.chunks = []
        except Exception:
            pass

    def zeros(self, *shape):
        t = self.empty(*shape)
        if t.numel():
            t.zero_()
        return t

    def zeros_many(self, shapes):
        """Several zeroed 2-D blocks carved from one allocation (one memset)."""
        sizes = [max(-(-(int(a) * int(b)) // self.ALIGN) * self.ALIGN, self.ALIGN) for a, b in shapes]
        flat = self.empty(sum(sizes))
        if flat.numel():
            flat.zero_()
        out, o = [], 0
        for (a, b), sz in zip(shapes, sizes):
            out.append(flat[o:o + int(a) * int(b)].view(int(a), int(b)))
            o += sz
        return out

    def reset(self):
        self.i = 0
        self.off = 0

    @property
    def reserved_bytes(self):
        return 8 * sum(c.numel() for c in self.chunks)


def capture_graph(fn):
    """Record fn()'s launches into a CUDA graph on a side stream and return it.
    torch.cuda.graph() also synchronizes, runs gc.collect() and empties the caching
    allocator on entry -- 0.37 s on config[4], where GBs of cached blocks go back to the
    driver and are cudaMalloc'ed again afterwards; the raw capture_begin / capture_end
    pair records into a private pool without touching the cache."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        g.capture_begin()
        try:
            fn()
        finally:
            g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    return g


SCRATCH = None


def scratch(*shape):
    """Transient FP64 buffer: from the active scratch arena, else torch's allocator."""
    if SCRATCH is not None:
        return SCRATCH.empty(*shape)
    return empty(*shape)


def torch_from_numpy(a):
    return torch.from_numpy(np.ascontiguousarray(a))


def to_dev(a, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(dev(), non_blocking=False)


def ld(t):
    """Leading dimension (row stride) of a 2-D row-major tensor view (called for
    every operand of every launch: one shape and one stride query)."""
    try:
        (r, c), (s0, s1) = t.shape, t.stride()
    except ValueError:
        raise ValueError("expected a 2-D tensor") from None
    if r == 0 or c == 0:
        return c if c > 1 else 1
    if c > 1 and s1 != 1:
        raise ValueError("tensor must have unit column stride")
    return s0 if s0 > c else (c if c > 1 else 1)


# ---------------------------------------------------------------------------
# GEMM


def gemm_problems(n):
    return np.zeros(n, dtype=GEMM_DTYPE)


def gcat(parts):
    """Concatenate GEMM_DTYPE problem arrays through byte views (np.concatenate on
    structured arrays runs numpy's field promotion per call: ~20x slower)."""
    if len(parts) == 1:
        return parts[0]
    return np.concatenate([np.ascontiguousarray(q).view(np.uint8) for q in parts]).view(GEMM_DTYPE)


class KernelProfile:
    """Optional CUDA-event timing of every grouped-GEMM launch (bench.py roofline):
    records (start, end, flops) with flops = sum of 2 M N K * batch of the launch."""

    def __init__(self):
        self.records = []

    def summary(self):
        torch.cuda.synchronize()
        t = sum(r[0].elapsed_time(r[1]) for r in self.records) * 1e-3
        f = sum(r[2] for r in self.records)
        return {"launch_groups": len(self.records), "seconds": t, "flops": f}

    def by_tag(self):
        torch.cuda.synchronize()
        out = {}
        for s, e, fl, tag in self.records:
            d = out.setdefault(tag, [0, 0.0, 0.0])
            d[0] += 1
            d[1] += s.elapsed_time(e) * 1e-3
            d[2] += fl
        return out


PROFILE = None
TAG = "untagged"  # call-site label recorded with each profiled launch


class region:
    """`with region("name"):` -- CUDA-event timing of a host-issued section when a
    KernelProfile is active (records flops 0, tag = name); free otherwise."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        if PROFILE is not None:
            self.s = torch.cuda.Event(enable_timing=True)
            self.s.record()
        return self

    def __exit__(self, *exc):
        if PROFILE is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            PROFILE.records.append((self.s, e, 0.0, "region:" + self.name))


GEMM_WS_BYTES = int(os.environ.get("RSC_GEMM_WS_MB", "512")) << 20
_GEMM_WS = {}  # stream handle (None = device default) -> workspace tensor


def ensure_gemm_workspace():
    """Register the current stream's ordered-accumulation workspace (the partials of
    a launch's accumulating problems, rsc_gemm_set_workspace).  A device-wide default
    is registered on first use; streams seen outside graph capture get their own so
    that concurrent streams never share partials.  During capture the stream uses
    the default (nothing is allocated inside a capture)."""
    lib = require_cuda()
    if None not in _GEMM_WS:
        t = torch.empty(GEMM_WS_BYTES // 8, dtype=F64, device=dev())
        check(lib.rsc_gemm_set_workspace(None, t.data_ptr(), GEMM_WS_BYTES, 1), "rsc_gemm_set_workspace")
        _GEMM_WS[None] = t
    h = stream_handle()
    if h not in _GEMM_WS and not torch.cuda.is_current_stream_capturing():
        t = torch.empty(GEMM_WS_BYTES // 8, dtype=F64, device=dev())
        check(lib.rsc_gemm_set_workspace(h, t.data_ptr(), GEMM_WS_BYTES, 0), "rsc_gemm_set_workspace")
        _GEMM_WS[h] = t
    return lib


def gemm_grouped(probs, transA=False, transB=False):
    """Launch a grouped DMMA GEMM from a GEMM_DTYPE numpy array of problems.
    Accumulating problems (atomic=1) are summed deterministically in array order
    (see rsc_gemm_grouped); mapped ones need ext_r/ext_c = their target's extent."""
    probs = np.ascontiguousarray(probs, dtype=GEMM_DTYPE)
    if probs.size == 0:
        return
    lib = ensure_gemm_workspace() if (probs["atomic"] != 0).any() else require_cuda()
    prof = PROFILE
    if prof is not None:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
    check(lib.rsc_gemm_grouped(int(transA), int(transB), addr(probs), int(probs.size), stream_handle()),
          "rsc_gemm_grouped")
    if prof is not None:
        e.record()
        fl = float(np.sum(2.0 * probs["M"].astype(np.float64) * probs["N"] * probs["K"] * probs["batch"]))
        prof.records.append((s, e, fl, TAG))


def gemm_balanced(probs, transA=False, transB=False, ctas=None):
    """gemm_grouped(balance_k(probs)) with the K balancing done in the library
    (rsc_gemm_grouped_balanced: same splits, no numpy rebuild of the problem array)."""
    probs = np.ascontiguousarray(probs, dtype=GEMM_DTYPE)
    if probs.size == 0:
        return
    lib = ensure_gemm_workspace() if (probs["atomic"] != 0).any() or (probs["beta"] == 1.0).any() else require_cuda()
    prof = PROFILE
    if prof is not None:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
    check(lib.rsc_gemm_grouped_balanced(int(transA), int(transB), addr(probs), int(probs.size),
                                        int(ctas or GEMM_CONCURRENT_CTAS), stream_handle()),
          "rsc_gemm_grouped_balanced")
    if prof is not None:
        e.record()
        fl = float(np.sum(2.0 * probs["M"].astype(np.float64) * probs["N"] * probs["K"] * probs["batch"]))
        prof.records.append((s, e, fl, TAG))


def split_k(p, transA, transB, ks):
    """Cut every problem's K into slabs of at most `ks`, accumulated (in slab order,
    deterministically) into C: tall-K products (few output tiles, long K) then spread
    over many CTAs.  Problems that get split must have C zeroed by the caller (their
    beta is dropped: every slab adds).  Handles the b_rows gather (the index pointer
    advances).  Problem order is preserved (slabs replace their problem in place)."""
    return split_k_var(p, transA, transB, np.full(p.size, int(ks), dtype=np.int64))


def split_k_var(p, transA, transB, ks):
    """split_k with a per-problem slab length ks[i]."""
    K = p["K"].astype(np.int64)
    ks = np.asarray(ks, dtype=np.int64)
    nsl = np.maximum(1, -(-K // ks))
    if (nsl == 1).all():
        return p
    idx = np.repeat(np.arange(p.size), nsl)
    q = p[idx].copy()
    first = np.repeat(np.cumsum(nsl) - nsl, nsl)
    k0 = ((np.arange(q.size) - first) * ks[idx]).astype(np.int64)
    q["K"] = np.minimum(ks[idx], K[idx] - k0)
    k0u = k0.astype(np.uint64)
    q["A"] = q["A"] + (k0u * q["lda"].astype(np.uint64) * np.uint64(8) if transA else k0u * np.uint64(8))
    if transB:
        q["B"] = q["B"] + k0u * np.uint64(8)
    else:
        rows = q["b_rows"] != 0
        q["B"] = np.where(rows, q["B"], q["B"] + k0u * q["ldb"].astype(np.uint64) * np.uint64(8))
        q["b_rows"] = np.where(rows, q["b_rows"] + k0u * np.uint64(4), q["b_rows"])
    split = nsl[idx] > 1
    q["atomic"] = np.where(split, 1, q["atomic"])
    q["beta"] = np.where(split, 1.0, q["beta"])
    return q


GEMM_CONCURRENT_CTAS = int(os.environ.get("RSC_GEMM_CTAS", 148 * 5))  # balance_k target CTAs (5 per SM)


def balance_k(p, transA, transB, ctas=GEMM_CONCURRENT_CTAS):
    """Split the K of problems whose single-tile k-loop would outlast the launch.

    A grouped launch finishes with its longest CTA.  In the sparse sweep one launch
    mixes tall-K products with many small ones (the longest CTA bound was 2.6x the
    balanced time on config[2]), so every problem that accumulates (atomic, or
    beta = 1) and whose K exceeds ~1.5x the balanced per-CTA share is cut into K
    slabs of that share, accumulated in slab order (split_k)."""
    if p.size == 0:
        return p
    tiles = np.ceil(p["M"] / 64.0) * np.ceil(p["N"] / 64.0) * p["batch"]
    ks = np.ceil(p["K"] / 16.0)
    target = max(8, int(np.ceil(float((tiles * ks).sum()) / ctas)))
    need = ((p["atomic"] == 1) | (p["beta"] == 1.0)) & (ks > 1.5 * target)
    if not need.any():
        return p
    # split in place: accumulation order stays the launch order (deterministic sums)
    K = p["K"].astype(np.int64)
    lim = np.where(need, 16 * target, np.maximum(K, 1))
    return split_k_var(p, transA, transB, lim)


def gemm(A, B, C, transA=False, transB=False, alpha=1.0, beta=0.0):
    """C = alpha op(A) op(B) + beta C for 2-D tensors (views allowed)."""
    M = A.shape[1] if transA else A.shape[0]
    K = A.shape[0] if transA else A.shape[1]
    N = B.shape[0] if transB else B.shape[1]
    if C.shape[0] != M or C.shape[1] != N:
        raise ValueError("gemm shape mismatch")
    p = gemm_problems(1)
    p["A"], p["B"], p["C"] = A.data_ptr(), B.data_ptr(), C.data_ptr()
    p["M"], p["N"], p["K"] = M, N, K
    p["lda"], p["ldb"], p["ldc"] = ld(A), ld(B), ld(C)
    p["batch"], p["alpha"], p["beta"] = 1, alpha, beta
    gemm_grouped(p, transA, transB)


def gemm_strided_batched(A, B, C, transA=False, transB=False, alpha=1.0, beta=0.0, splitk=1):
    """Batched GEMM over the leading dim of 3-D contiguous tensors.

    splitk > 1 cuts K into `splitk` slabs accumulated in slab order (C is
    zeroed first when beta == 0) -- for the tall-K sketch products L_O^T X whose
    output tile count alone cannot fill 148 SMs."""
    nb = A.shape[0]
    M = A.shape[2] if transA else A.shape[1]
    K = A.shape[1] if transA else A.shape[2]
    N = B.shape[1] if transB else B.shape[2]
    splitk = max(1, min(int(splitk), K // 16 if K >= 32 else 1))
    if splitk > 1:
        if beta == 0.0:
            C.zero_()
        elif beta != 1.0:
            C.mul_(beta)
    kc = -(-K // splitk)
    kc = -(-kc // 16) * 16
    starts = list(range(0, K, kc))
    p = gemm_problems(len(starts))
    for i, k0 in enumerate(starts):
        a_off = (k0 * A.stride(1)) if transA else k0
        b_off = k0 if transB else (k0 * B.stride(1))
        p[i]["A"] = A.data_ptr() + 8 * a_off
        p[i]["B"] = B.data_ptr() + 8 * b_off
        p[i]["C"] = C.data_ptr()
        p[i]["K"] = min(kc, K - k0)
    p["sA"], p["sB"], p["sC"] = A.stride(0), B.stride(0), C.stride(0)
    p["M"], p["N"] = M, N
    p["lda"], p["ldb"], p["ldc"] = A.stride(1), B.stride(1), C.stride(1)
    p["batch"], p["alpha"] = nb, alpha
    if len(starts) > 1:
        p["atomic"] = 1
        p["beta"] = 1.0
    else:
        p["beta"] = beta
    gemm_grouped(p, transA, transB)


# ---------------------------------------------------------------------------
# POTRF / TRSM


class TriFactors:
    """A batch of device lower triangles with their inverse 64x64 diagonal blocks."""

    def __init__(self, ptrs, n, lds, dinv_ptrs, keep=()):
        self.ptrs = ptr_array(ptrs)
        self.n = int_array(n)
        self.lds = int_array(lds)
        self.dinv = ptr_array(dinv_ptrs)
        self._keep = list(keep)  # owning tensors

    @property
    def count(self):
        return int(self.n.size)


def potrf_batched(ptrs, n, lds, dinv_ptrs, info):
    """In-place batched Cholesky; returns nothing, failures land in `info` (device int32)."""
    lib = require_cuda()
    ptrs, n, lds, dinv_ptrs = ptr_array(ptrs), int_array(n), int_array(lds), ptr_array(dinv_ptrs)
    if n.size == 0:
        return
    check(lib.rsc_potrf_batched(int(n.size), addr(ptrs), addr(n), addr(lds), addr(dinv_ptrs),
                                info.data_ptr(), stream_handle()), "rsc_potrf_batched")


def trtri_diag_batched(ptrs, n, lds, dinv_ptrs):
    lib = require_cuda()
    ptrs, n, lds, dinv_ptrs = ptr_array(ptrs), int_array(n), int_array(lds), ptr_array(dinv_ptrs)
    if n.size == 0:
        return
    check(lib.rsc_trtri_diag_batched(int(n.size), addr(ptrs), addr(n), addr(lds), addr(dinv_ptrs),
                                     stream_handle()), "rsc_trtri_diag_batched")


def trsm_batched(side, trans, Lptrs, n, ldl, dinv_ptrs, Bptrs, m, ldb):
    """side 'left'/'right'; see rsc_trsm_batched."""
    lib = require_cuda()
    Lptrs, n, ldl, dinv_ptrs = ptr_array(Lptrs), int_array(n), int_array(ldl), ptr_array(dinv_ptrs)
    Bptrs, m, ldb = ptr_array(Bptrs), int_array(m), int_array(ldb)
    if n.size == 0:
        return
    s = 0 if side == "left" else 1
    check(lib.rsc_trsm_batched(s, int(trans), int(n.size), addr(Lptrs), addr(n), addr(ldl),
                               addr(dinv_ptrs), addr(Bptrs), addr(m), addr(ldb), stream_handle()),
          "rsc_trsm_batched")


def trsm_right(Lptrs, n, ldl, dinv_ptrs, src_ptrs, Bptrs, m, ldb):
    """B = Bsrc L^{-T} (out of place; src_ptrs None = in place), n <= 320."""
    lib = require_cuda()
    Lptrs, n, ldl, dinv_ptrs = ptr_array(Lptrs), int_array(n), int_array(ldl), ptr_array(dinv_ptrs)
    Bptrs, m, ldb = ptr_array(Bptrs), int_array(m), int_array(ldb)
    src = None if src_ptrs is None else ptr_array(src_ptrs)
    if n.size == 0:
        return
    check(lib.rsc_trsm_right_batched(int(n.size), addr(Lptrs), addr(n), addr(ldl), addr(dinv_ptrs), addr(src),
                                     addr(Bptrs), addr(m), addr(ldb), stream_handle()), "rsc_trsm_right_batched")


# ---------------------------------------------------------------------------
# QRCP


def qrcp_batched(Gptrs, m, k, ldg, Qptrs, ldq, rank_out, alloc=None):
    """Column-pivoted QR + cutoff; rank_out is a device int32 tensor (len = count).
    `alloc(n)` provides the FP64 workspace (default: torch allocator)."""
    lib = require_cuda()
    Gptrs, m, k, ldg = ptr_array(Gptrs), int_array(m), int_array(k), int_array(ldg)
    Qptrs, ldq = ptr_array(Qptrs), int_array(ldq)
    if m.size == 0:
        return
    wbytes = int(lib.rsc_qrcp_workspace_bytes(int(m.size), addr(m), addr(k)))
    nw = max(wbytes // 8, 1)
    work = alloc(nw) if alloc is not None else torch.empty(nw, dtype=F64, device=dev())
    check(lib.rsc_qrcp_batched(int(m.size), addr(Gptrs), addr(m), addr(k), addr(ldg), addr(Qptrs),
                               addr(ldq), rank_out.data_ptr(), work.data_ptr(), stream_handle()),
          "rsc_qrcp_batched")
    return work  # keep alive until the stream passes it


# ---------------------------------------------------------------------------
# Gaussian sketches (device PCG64 + numpy ziggurat)


def pcg64_block_states(keys):
    """keys: (master, tag, ...) int tuples, or a 2-D uint64 array of equal-length
    keys -> (seeds uint64[count], PCG64 states uint64[count, 4]) exactly as the
    reference seeds each sketch (factor.py:324-326 then np.random.PCG64(seed)).
    Host integer work in the library, no device."""
    lib = _lib.load()
    if isinstance(keys, np.ndarray):
        K = np.ascontiguousarray(keys, dtype=np.uint64)
        count, width = K.shape
        nk = np.full(count, width, dtype=np.int32)
    else:
        count = len(keys)
        width = max((len(k) for k in keys), default=1)
        K = np.zeros((count, width), dtype=np.uint64)
        nk = np.empty(count, dtype=np.int32)
        for i, k in enumerate(keys):
            K[i, :len(k)] = [int(v) for v in k]
            nk[i] = len(k)
    seeds = np.empty(count, dtype=np.uint64)
    states = np.empty((count, 4), dtype=np.uint64)
    if count:
        check(lib.rsc_pcg64_block_states(count, width, addr(K), addr(nk), addr(seeds), addr(states)),
              "rsc_pcg64_block_states")
    return seeds, states


def pcg64_seed_states(seeds):
    lib = _lib.load()
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    states = np.empty((seeds.size, 4), dtype=np.uint64)
    if seeds.size:
        check(lib.rsc_pcg64_seed_states(int(seeds.size), addr(seeds), addr(states)), "rsc_pcg64_seed_states")
    return states


def normal_pcg64(states, n, out_ptrs, alloc=None):
    """out_ptrs[i][0:n[i]] <- numpy's standard_normal stream of PCG64 state i
    (bit-identical), generated on the current stream.  Returns the workspace
    (keep alive until the stream passes it)."""
    lib = require_cuda()
    states = np.ascontiguousarray(np.asarray(states, dtype=np.uint64).reshape(-1, 4))
    n = np.ascontiguousarray(np.asarray(n, dtype=np.int64))
    outs = ptr_array(out_ptrs)
    count = int(n.size)
    if count == 0:
        return None
    wbytes = int(lib.rsc_normal_workspace_bytes(count, addr(n)))
    nw = max((wbytes + 7) // 8, 1)
    work = alloc(nw) if alloc is not None else torch.empty(nw, dtype=F64, device=dev())
    check(lib.rsc_normal_pcg64(count, addr(states), addr(n), addr(outs), work.data_ptr(), nw * 8,
                               stream_handle()), "rsc_normal_pcg64")
    return work


# ---------------------------------------------------------------------------
# sparse + vector


class DeviceCSR:
    """A CSR matrix (or block) resident on the device, int32 indices."""

    def __init__(self, nrows, ncols, indptr, indices, data):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.indptr = to_dev(np.asarray(indptr, dtype=np.int32))
        self.indices = to_dev(np.asarray(indices, dtype=np.int32))
        self.data = to_dev(np.asarray(data, dtype=np.float64))
        self.nnz = int(len(data))

    @classmethod
    def from_scipy(cls, S):
        S = S.tocsr()
        S.sort_indices()
        return cls(S.shape[0], S.shape[1], S.indptr, S.indices, S.data)


def spmm(S, X, Y, alpha=1.0, beta=0.0):
    """Y = alpha S X + beta Y (S: DeviceCSR, X/Y 2-D tensors)."""
    lib = require_cuda()
    check(lib.rsc_spmm_csr(S.nrows, int(X.shape[1]), S.indptr.data_ptr(), S.indices.data_ptr(),
                           S.data.data_ptr(), X.data_ptr(), ld(X), float(alpha), float(beta),
                           Y.data_ptr(), ld(Y), stream_handle()), "rsc_spmm_csr")


def spmv(S, x, y):
    lib = require_cuda()
    check(lib.rsc_spmv_csr(S.nrows, S.indptr.data_ptr(), S.indices.data_ptr(), S.data.data_ptr(),
                           x.data_ptr(), y.data_ptr(), stream_handle()), "rsc_spmv_csr")


def csr_to_dense_batched(rowptrs, colidx, values, nrows, Dptrs, ldd):
    lib = require_cuda()
    rowptrs, colidx, values = ptr_array(rowptrs), ptr_array(colidx), ptr_array(values)
    nrows, Dptrs, ldd = int_array(nrows), ptr_array(Dptrs), int_array(ldd)
    if nrows.size == 0:
        return
    check(lib.rsc_csr_to_dense_batched(int(nrows.size), addr(rowptrs), addr(colidx), addr(values),
                                       addr(nrows), addr(Dptrs), addr(ldd), stream_handle()),
          "rsc_csr_to_dense_batched")


def gather_rows(idx, src, dst):
    lib = require_cuda()
    check(lib.rsc_gather_rows(int(idx.numel()), int(src.shape[1]), idx.data_ptr(), src.data_ptr(), ld(src),
                              dst.data_ptr(), ld(dst), stream_handle()), "rsc_gather_rows")


def scatter_add_rows(idx, src, dst, alpha=1.0):
    lib = require_cuda()
    check(lib.rsc_scatter_add_rows(int(idx.numel()), int(src.shape[1]), idx.data_ptr(), float(alpha),
                                   src.data_ptr(), ld(src), dst.data_ptr(), ld(dst), stream_handle()),
          "rsc_scatter_add_rows")


class DotWorkspace:
    def __init__(self):
        self.part = empty(512)


def dot(x, y, out, ws):
    lib = require_cuda()
    check(lib.rsc_dot(int(x.numel()), x.data_ptr(), y.data_ptr(), out.data_ptr(), ws.part.data_ptr(),
                      stream_handle()), "rsc_dot")


def pcg_update_xr(rz, pap, x, r, p, ap):
    lib = require_cuda()
    check(lib.rsc_pcg_update_xr(int(x.numel()), rz.data_ptr(), pap.data_ptr(), x.data_ptr(), r.data_ptr(),
                                p.data_ptr(), ap.data_ptr(), stream_handle()), "rsc_pcg_update_xr")


def pcg_update_p(rznew, rz, z, p):
    lib = require_cuda()
    check(lib.rsc_pcg_update_p(int(z.numel()), rznew.data_ptr(), rz.data_ptr(), z.data_ptr(), p.data_ptr(),
                               stream_handle()), "rsc_pcg_update_p")
