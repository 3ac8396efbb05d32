"""Plan compiler: flattens the symbolic plan into the static index data the GPU
numeric phase consumes, uploaded once.

Everything the reference recomputes on every call is a function of the symbolic
structure alone, so it is computed here once (SURVEY §7 "Plan"):

  * the update sources of every compressed supernode j, in reference order
    (the bucket walk of factor.py:545-554,572 visits exactly the sources whose row
    set meets C_j, sorted by their first column);
  * per (source, target) pair the descendant map of symbolic.py:309-356:
    lo/hi = searchsorted(rows_s, (c0, c1)), cpos = rows_s[lo:hi] - c0 and
    rpos = searchsorted(R_j, rows_s[hi:])  (factor.py:389-398, 450-455, 477-482);
  * the A blocks A(C_j, C_j), A(R_j, C_j), A(C_j, R_j) as device CSR blocks
    (factor.py:378-379, 444, 471);
  * interior blocks' off_rows (interior.py:152-154) -- these are structural.

Interior blocks are materialized: Y_B = A(off_rows, C_B) L_B^{-T} is formed once,
which turns every interior source into a dense panel (exactly the operator
L(rows, C_B) of interior.py:77-95; rows outside off_rows are exact zeros).
"""

import numpy as np
import torch

from . import engine as E


def _pattern_key(A):
    """Digest of a lower-CSC sparsity pattern (col_ptr, row_idx): two 64-bit
    chunked multiply-xor hashes (rsc_hash64, host threads)."""
    from . import _lib

    lib = _lib.load()
    cp = np.ascontiguousarray(A.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.row_idx, dtype=np.int64)
    return (A.n, cp.size, ri.size, int(lib.rsc_hash64(cp.ctypes.data, cp.nbytes)),
            int(lib.rsc_hash64(ri.ctypes.data, ri.nbytes)))


class Source:
    """One update source: an interior block (rows = off_rows) or a compressed
    supernode (rows = R_j).  `order` is its first column (factor.py:565,639)."""

    __slots__ = ("sid", "kind", "unit", "rows", "order", "c0", "c1")

    def __init__(self, sid, kind, unit, rows, c0, c1):
        self.sid, self.kind, self.unit = sid, kind, unit
        self.rows = rows
        self.order = c0
        self.c0, self.c1 = c0, c1


class Pair:
    """Descendant map of source s into target supernode j."""

    __slots__ = ("s", "lo", "hi", "n_rd", "n_ro", "cpos_off", "rpos_off")

    def __init__(self, s, lo, hi, cpos_off, rpos_off, nrows):
        self.s = s
        self.lo, self.hi = lo, hi
        self.n_rd = hi - lo
        self.n_ro = nrows - hi
        self.cpos_off, self.rpos_off = cpos_off, rpos_off


class IndexPool:
    """Host accumulator of int32 index arrays, uploaded as one device buffer."""

    def __init__(self):
        self.chunks = []
        self.size = 0

    def add(self, arr):
        arr = np.asarray(arr, dtype=np.int32)
        off = self.size
        if arr.size:
            self.chunks.append(arr)
            self.size += arr.size
        return off

    def upload(self):
        host = np.concatenate(self.chunks) if self.chunks else np.zeros(1, np.int32)
        self.host = host
        self.dev = E.to_dev(host)
        return self.dev

    def ptr(self, off):
        return self.dev.data_ptr() + 4 * int(off)


class CsrPool:
    """Many small CSR blocks in three device buffers (rowptr int32 per block,
    colidx int32, values f64).  Blocks are windows of one host CSR matrix (`full`),
    requested with `add` and cut together by one rsc_csr_windows call at upload."""

    def __init__(self, full=None):
        self.full = full
        self.sel, self.nsel = [], 0
        self.req, self.blocks = [], []
        self.nrp = 0

    def _spec(self, x):
        if isinstance(x, tuple):  # contiguous range [lo, hi)
            return -1, x[1] - x[0], x[0]
        x = np.ascontiguousarray(x, dtype=np.int64)
        off = self.nsel
        self.sel.append(x)
        self.nsel += x.size
        return off, x.size, 0

    def add(self, rows, cols):
        """Block full[rows, cols]; rows / cols = (lo, hi) ranges or ascending index arrays."""
        ro, rn, rl = self._spec(rows)
        co, cn, cl = self._spec(cols)
        blk = CsrBlock(self, rn, cn, self.nrp, 0, 0)
        self.nrp += rn + 1
        self.req.append((ro, rn, rl, co, cn, cl))
        self.blocks.append(blk)
        return blk

    def cut(self):
        """Host arrays of every requested block (two passes of rsc_csr_windows).
        The windows are cut from the position matrix: values are 1-based positions
        into B's storage, returned 0-based in `pos`."""
        from . import _lib

        lib = _lib.load()
        full = self.full
        if full.nnz >= 2**31 - 1:
            raise ValueError("matrix too large for int32 block positions")
        indptr = np.ascontiguousarray(full.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(full.indices, dtype=np.int64)
        data = np.ascontiguousarray(full.data, dtype=np.float64)
        sel = np.concatenate(self.sel) if self.sel else np.zeros(1, np.int64)
        q = np.array(self.req, dtype=np.int64).reshape(-1, 6).T.copy()
        nq = q.shape[1]
        nnz = np.zeros(max(nq, 1), dtype=np.int64)
        rp_off = np.array([b.rp_off for b in self.blocks] or [0], dtype=np.int64)
        args = [nq, full.shape[0], indptr.ctypes.data, indices.ctypes.data, data.ctypes.data, sel.ctypes.data]
        args += [q[i].ctypes.data for i in range(6)] + [nnz.ctypes.data, rp_off.ctypes.data]
        _lib.check(lib.rsc_csr_windows(*args, None, None, None, None), "rsc_csr_windows")
        offs = np.concatenate(([0], np.cumsum(nnz[:nq])))
        tot = int(offs[-1])
        self.rp = np.zeros(max(self.nrp, 1), dtype=np.int32)
        self.ci = np.empty(max(tot, 1), dtype=np.int32)
        self.pos = np.empty(max(tot, 1), dtype=np.int32)
        if tot == 0:
            self.ci[:] = 0
            self.pos[:] = 0
        _lib.check(lib.rsc_csr_windows(*args, offs.ctypes.data, self.rp.ctypes.data, self.ci.ctypes.data,
                                       self.pos.ctypes.data), "rsc_csr_windows")
        for blk, o, z in zip(self.blocks, offs[:nq].tolist(), nnz[:nq].tolist()):
            blk.nz_off, blk.nnz = o, z
        self.nnz = tot

    def upload(self, b_values):
        """Device buffers; the values are gathered on the device (pos -> values)."""
        self.cut()
        self.rp_dev = E.to_dev(self.rp)
        self.ci_dev = E.to_dev(self.ci)
        self.pos_dev = E.to_dev(self.pos)  # int32
        self.v_dev = torch.empty(self.pos.size, dtype=torch.float64, device=E.dev())
        self.gather(E.to_dev(np.asarray(b_values)), self.pos_dev)

    def gather(self, vals_dev, index_dev):
        if self.nnz:
            torch.index_select(vals_dev, 0, index_dev, out=self.v_dev)
        else:
            self.v_dev.zero_()


class CsrBlock:
    """View of one block of a CsrPool (rowptr entries are block-local offsets)."""

    def __init__(self, pool, nrows, ncols, rp_off, nz_off, nnz):
        self.pool, self.nrows, self.ncols = pool, nrows, ncols
        self.rp_off, self.nz_off, self.nnz = rp_off, nz_off, nnz

    @property
    def indptr_ptr(self):
        return self.pool.rp_dev.data_ptr() + 4 * self.rp_off

    @property
    def indices_ptr(self):
        return self.pool.ci_dev.data_ptr() + 4 * self.nz_off

    @property
    def data_ptr(self):
        return self.pool.v_dev.data_ptr() + 8 * self.nz_off


class TreeBlockMaps:
    """Window maps of one source into one diagonal-tree block (diagblocks.py:230-262):
    rows of the source inside the row window [r0,r1) and column window [c0,c1)."""

    __slots__ = ("s", "clo", "chi", "rlo", "rhi", "cidx_off", "ridx_off")


class NumericPlan:
    """Static device-side plan for the numeric phase of one symbolic plan."""

    def __init__(self, sym, interior_enabled, A=None):
        self.sym = sym
        part = sym.partition
        B = sym.B
        # Every A block of the plan is cut from a copy of B whose values are 1-based
        # positions into B's storage, so one gather index maps any matrix with this
        # pattern onto the device value buffer (load_values: refactorization).
        from .sparse import SparseSpdMatrix

        posB = SparseSpdMatrix(B.n, B.col_ptr, B.row_idx, np.arange(1, B.nnz_lower + 1, dtype=np.float64),
                               validate=False)
        full = posB.to_csr_full()
        self.full = full
        # B.values = A.values[b_from_a] (the gather analyze used to permute A)
        self.b_from_a = getattr(sym, "b_from_a", None) if A is not None else None
        self.source = A
        self.pattern_key = _pattern_key(A) if A is not None else None  # load_values checks it
        self.idx = IndexPool()
        self.csr = CsrPool(full)
        self.sources = []
        self.unit_source = {}      # unit index -> source id
        self.targets = {}          # node j -> [Pair] (reference order)
        self.node_blocks = {}      # node j -> (A_CC, A_RC, A_CR)
        self.rows_off = {}         # node j / ("int", u) -> index offset of its row set
        self.interior = []         # (unit index, members, c0, c1, off_rows, A_off csr, A_BB csr)
        # every row structure R_j enters the index pool once, as one chunk
        R_ptr, R_all = _rows_flat(part)
        rows_base = self.idx.add(R_all[:int(R_ptr[-1])])
        for u, (kind, payload) in enumerate(sym.units):
            if kind == "interior":
                ids = payload
                c0, c1 = int(part.starts[ids[0]]), int(part.starts[ids[-1] + 1])
                tails = []
                for j in ids:
                    rj = part.rows[j]
                    nib = int(np.searchsorted(rj, c1))
                    if rj.size > nib:
                        tails.append(rj[nib:])
                off_rows = np.unique(np.concatenate(tails)) if tails else np.empty(0, np.int64)
                A_BB = self.csr.add((c0, c1), (c0, c1))
                A_off = self.csr.add(off_rows, (c0, c1)) if off_rows.size else None
                roff = self.idx.add(off_rows)
                self.rows_off[("int", u)] = roff
                self.interior.append((u, ids, c0, c1, off_rows, A_off, A_BB))
                if off_rows.size:
                    sid = len(self.sources)
                    self.sources.append(Source(sid, "interior", u, off_rows, c0, c1))
                    self.unit_source[u] = sid
                continue
            j = payload
            c0, c1 = part.cols(j)
            R = part.rows[j]
            self.targets[j] = []
            A_CC = self.csr.add((c0, c1), (c0, c1))
            A_RC = self.csr.add(R, (c0, c1)) if R.size else None
            A_CR = self.csr.add((c0, c1), R) if R.size else None  # full[R, C]^T (symmetric)
            self.node_blocks[j] = (A_CC, A_RC, A_CR)
            self.rows_off[j] = rows_base + int(R_ptr[j])
            if R.size:
                sid = len(self.sources)
                self.sources.append(Source(sid, "node", u, R, c0, c1))
                self.unit_source[u] = sid
        self._build_targets(part)
        self.tree_maps = {}
        self._build_tree_maps(part)
        self.idx.upload()
        self.csr.upload(B.values)
        # unit indices of the nodes that get a diagonal tree (restart rule)
        self.tree_units = np.array(
            [u for u, (k, j) in enumerate(sym.units)
             if k == "node" and part.is_separator[j] and j in sym.sep_splits], dtype=np.int64)
        # node units grouped by height in the source DAG: a node only reads sources of
        # strictly lower height (interior blocks count as height -1), so each level
        # is a set of independent nodes
        height = {}
        for u, (k, j) in enumerate(sym.units):
            if k != "node":
                continue
            h = 0
            for ps in self.tarr[j]["s"].tolist():
                su = self.sources[ps].unit
                if su in height:
                    h = max(h, height[su] + 1)
            height[u] = h
        nlev = max(height.values()) + 1 if height else 0
        self.node_levels = [[] for _ in range(nlev)]
        for u in sorted(height):
            self.node_levels[height[u]].append(u)

    def load_values(self, A):
        """Refactorization: put the values of A (same pattern as the prepared matrix)
        into the plan's device A blocks -- one host gather and one copy."""
        if A is self.source:
            return
        if self.b_from_a is None:
            raise ValueError("plan was prepared without its source matrix; cannot load new values")
        if A.n != self.sym.B.n or A.nnz_lower != self.b_from_a.size or _pattern_key(A) != self.pattern_key:
            raise ValueError("matrix pattern differs from the prepared one")
        if getattr(self, "_a_index", None) is None:  # A position of every block entry
            self._a_index = E.to_dev(self.b_from_a.astype(np.int32))[self.csr.pos_dev.long()]
        self.csr.gather(E.to_dev(np.asarray(A.values)), self._a_index)
        self.source = A

    def sketch_specs(self, cfg, alpha_d):
        """(key, m, r, seed key) of every Gaussian sketch one numeric pass draws, in sweep
        order: off-diagonal blocks (seed tag (0, j), factor.py:620-625) and compressed
        diagonal-tree blocks (seed tag (1, j, s), factor.py:605-610)."""
        from .symbolic import block_rank

        part = self.sym.partition
        specs = []
        for u in [u for lev in self.node_levels for u in lev]:  # level-batched use order
            j = self.sym.units[u][1]
            if not part.is_separator[j]:
                continue
            c0, c1 = part.cols(j)
            nc = c1 - c0
            R = part.rows[j]
            if j in self.sym.sep_splits:
                shape = self.tree_shapes[j]
                for s in shape.order:
                    nd = shape.nodes[s]
                    if nd.is_leaf:
                        continue
                    nr, ncl = nd.hi - nd.split, nd.split - nd.lo
                    r = block_rank(nr, ncl, alpha_d, cfg.oversample)
                    if r < 0.75 * min(nr, ncl):
                        specs.append((("diag", j, s), nr, min(r, nr, ncl), (cfg.seed, 1, j, s)))
            r_off = block_rank(R.size, nc, cfg.alpha_o, cfg.oversample)
            if R.size and r_off < 0.75 * min(R.size, nc):
                specs.append((("off", j), R.size, min(r_off, R.size, nc), (cfg.seed, 0, j)))
        return specs

    def sketches_for(self, cfg, alpha_d):
        return DeviceSketches(self.sketch_specs(cfg, alpha_d))


    def _build_targets(self, part):
        """Descendant maps of every (source, target) pair (rsc_plan_pairs, host
        threads): the pairs of target j in reference order (sources by first column,
        factor.py:545-554,572), lo/hi = the run of the source's rows inside C_j,
        cpos = rows[lo:hi] - c0, rpos = searchsorted(R_j, rows[hi:])."""
        import ctypes

        from . import _lib

        lib = _lib.load()
        srcs = self.sources
        nsrc = len(srcs)
        src_len = np.fromiter((x.rows.size for x in srcs), dtype=np.int64, count=nsrc)
        src_ptr = np.zeros(nsrc + 1, dtype=np.int64)
        np.cumsum(src_len, out=src_ptr[1:])
        src_rows = np.concatenate([x.rows for x in srcs]).astype(np.int64) if nsrc else np.zeros(1, np.int64)
        src_order = np.fromiter((x.order for x in srcs), dtype=np.int64, count=nsrc)
        M = part.count
        is_t = np.zeros(max(M, 1), dtype=np.uint8)
        tj = np.fromiter(self.targets.keys(), dtype=np.int64, count=len(self.targets))
        is_t[tj] = 1
        R_ptr, R_rows = _rows_flat(part)
        st = np.ascontiguousarray(part.starts, dtype=np.int64)
        npairs, nidx = ctypes.c_longlong(0), ctypes.c_longlong(0)
        h = lib.rsc_plan_pairs(nsrc, src_ptr.ctypes.data, src_rows.ctypes.data, src_order.ctypes.data, M,
                               st.ctypes.data, is_t.ctypes.data, R_ptr.ctypes.data, R_rows.ctypes.data,
                               ctypes.byref(npairs), ctypes.byref(nidx))
        npr = npairs.value
        out = [np.empty(max(npr, 1), dtype=np.int64) for _ in range(6)]
        chunk = np.empty(max(nidx.value, 1), dtype=np.int32)
        _lib.check(lib.rsc_plan_pairs_fetch(h, *[o.ctypes.data for o in out], chunk.ctypes.data),
                   "rsc_plan_pairs_fetch")
        tgt, sid, lo, hi, cpos, rpos = (o[:npr] for o in out)
        base = self.idx.add(chunk[:nidx.value])
        cpos = cpos + base
        rpos = rpos + base
        nro = src_len[sid] - hi
        self._src_ptr, self._src_rows = src_ptr, src_rows
        self.pair_arrays = {"tgt": tgt, "s": sid, "lo": lo, "hi": hi, "cpos": cpos, "rpos": rpos}
        bnd = np.searchsorted(tgt, tj, side="left"), np.searchsorted(tgt, tj, side="right")
        self.pair_range = {}
        self.tarr = {}
        for j, a, b in zip(tj.tolist(), bnd[0].tolist(), bnd[1].tolist()):
            self.pair_range[j] = (a, b)
            self.tarr[j] = {"s": sid[a:b], "lo": lo[a:b], "hi": hi[a:b], "nrd": hi[a:b] - lo[a:b],
                            "nro": nro[a:b], "cpos": cpos[a:b], "rpos": rpos[a:b]}
        self.targets = _TargetPairs(self.tarr)

    def _build_tree_maps(self, part):
        """Window maps for every (tree node j, block s, source) with both windows
        non-empty (diagblocks.py:231-234, 252-255; rsc_plan_tree_maps, host threads),
        plus the A windows of every tree block."""
        import ctypes

        from . import _lib
        from .diagtree import TreeShape

        lib = _lib.load()
        self.tree_shapes = {}
        self.tmap = {}
        trees = []
        spans_all, blk_ptr, pair_ptr = [], [0], []
        for j, split in self.sym.sep_splits.items():
            c0, c1 = part.cols(j)
            shape = TreeShape(c1 - c0, c0, split)
            self.tree_shapes[j] = shape
            order = list(shape.order)
            spans = np.array([shape.span(s) for s in order], dtype=np.int64).reshape(len(order), 4) + c0
            trees.append((j, order, spans))
            spans_all.append(spans)
            blk_ptr.append(blk_ptr[-1] + len(order))
            pair_ptr.append(self.pair_range[j])
        keys = ("s", "clo", "chi", "rlo", "rhi", "cidx", "ridx")
        if trees:
            spans_c = np.ascontiguousarray(np.concatenate(spans_all), dtype=np.int64)
            bp = np.asarray(blk_ptr, dtype=np.int64)
            # pairs of tree t = [pp[2t], pp[2t+1]) in the global pair arrays: pass a
            # per-tree copy of those source ids so the ranges are contiguous
            psrc = np.concatenate([self.pair_arrays["s"][a:b] for a, b in pair_ptr]).astype(np.int64)
            pp = np.zeros(len(pair_ptr) + 1, dtype=np.int64)
            np.cumsum([b - a for a, b in pair_ptr], out=pp[1:])
            nm, ni = ctypes.c_longlong(0), ctypes.c_longlong(0)
            h = lib.rsc_plan_tree_maps(len(trees), bp.ctypes.data, spans_c.ctypes.data, pp.ctypes.data,
                                       psrc.ctypes.data, self._src_ptr.ctypes.data, self._src_rows.ctypes.data,
                                       ctypes.byref(nm), ctypes.byref(ni))
            out = [np.empty(max(nm.value, 1), dtype=np.int64) for _ in range(9)]
            chunk = np.empty(max(ni.value, 1), dtype=np.int32)
            ptrs = (ctypes.c_void_p * 9)(*[o.ctypes.data for o in out])
            _lib.check(lib.rsc_plan_tree_maps_fetch(h, ptrs, chunk.ctypes.data), "rsc_plan_tree_maps_fetch")
            out = [o[:nm.value] for o in out]
            base = self.idx.add(chunk[:ni.value])
            gblk = bp[out[0]] + out[1]  # global block index: maps are grouped by it
            cut = np.searchsorted(gblk, np.arange(bp[-1] + 1), side="left")
            cols = [out[2], out[3], out[4], out[5], out[6], out[7] + base, out[8] + base]
        for t, (j, order, spans) in enumerate(trees):
            gr0, gr1, gc0, gc1 = spans.T
            for k, s in enumerate(order):
                g = (int(gr0[k]), int(gr1[k])), (int(gc0[k]), int(gc1[k]))
                blk = self.csr.add(g[0], g[1])
                blkT = self.csr.add(g[1], g[0]) if g[0] != g[1] else None
                self.tree_maps[(j, s)] = (None, blk, blkT)
                a, b = int(cut[blk_ptr[t] + k]), int(cut[blk_ptr[t] + k + 1])
                self.tmap[(j, s)] = {kk: cols[i][a:b] for i, kk in enumerate(keys)}


def _rows_flat(part):
    """(ptr[M+1], rows) of the row structures R_j (one array when
    compute_row_structures made them)."""
    fl = getattr(part, "rows_flat", None)
    if fl is not None:
        return fl
    lens = np.fromiter((r.size for r in part.rows), dtype=np.int64, count=len(part.rows))
    ptr = np.zeros(len(part.rows) + 1, dtype=np.int64)
    np.cumsum(lens, out=ptr[1:])
    rows = np.concatenate(part.rows).astype(np.int64) if part.rows else np.zeros(1, np.int64)
    return ptr, rows


class _TargetPairs:
    """targets[j] -> [Pair] in reference order, built on first access from the
    plan's flat pair arrays (tarr)."""

    def __init__(self, tarr):
        self._tarr = tarr
        self._cache = {}

    def __getitem__(self, j):
        got = self._cache.get(j)
        if got is None:
            t = self._tarr[j]
            got = [Pair(s, lo, hi, c, r, hi + nro)
                   for s, lo, hi, c, r, nrd, nro in zip(t["s"].tolist(), t["lo"].tolist(), t["hi"].tolist(),
                                                        t["cpos"].tolist(), t["rpos"].tolist(),
                                                        t["nrd"].tolist(), t["nro"].tolist())]
            self._cache[j] = got
        return got

    def __contains__(self, j):
        return j in self._tarr

    def get(self, j, default=None):
        return self[j] if j in self._tarr else default

    def __iter__(self):
        return iter(self._tarr)

    def __len__(self):
        return len(self._tarr)

    def keys(self):
        return self._tarr.keys()

    def items(self):
        return ((j, self[j]) for j in self._tarr)

    def values(self):
        return (self[j] for j in self._tarr)


class DeviceSketches:
    """All Gaussian sketches of one numeric pass, generated on the device by one
    rsc_normal_pcg64 call before the sweep starts, bit-identical to the reference's
    host draws np.random.Generator(np.random.PCG64(_block_seed(seed, *tags)))
    .standard_normal((m, r)) (kernels.py:85-92, factor.py:324-326).  The buffer
    lives in the pass's own arena, released with the pass."""

    def __init__(self, specs):
        self.index = {}
        keys, ns, offs = [], [], []
        off = 0
        for key, m, r, seed_key in specs:
            self.index[key] = (off, m, r)
            keys.append(seed_key)
            ns.append(m * r)
            offs.append(off)
            off += -(-(m * r) // 32) * 32
        self.arena = E.Arena(max(off, 32))
        self.buf = self.arena.empty(max(off, 32))
        if keys:
            _, states = E.pcg64_block_states(keys)
            base = self.buf.data_ptr()
            ptrs = np.asarray(offs, dtype=np.uint64) * 8 + base
            E.normal_pcg64(states, ns, ptrs, alloc=self.arena.empty)

    def device(self, key, m, r, arena=None):
        off, m0, r0 = self.index[key]
        assert (m0, r0) == (m, r), (key, m0, r0, m, r)
        return self.buf[off:off + m * r].view(m, r)
