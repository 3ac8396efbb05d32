"""Multi-GPU decomposition of the numeric sweep by nested-dissection subtree.

One process per GPU (torch.distributed over NCCL; gloo on CPU for tests).  For P
ranks the top L = log2(P) levels of the separator tree hold P-1 separators; the
2^L subtrees below them depend only on their own descendants (the post-order unit
list of factor.py:524-532), so each rank factors one subtree with no
communication.  A top separator j needs, for every product it forms (Schur
assembly, Alg. 2/5 implicit products), a sum over update sources from every
subtree below it.  Each such term is linear in the source panels, so every rank
forms the partial sum over the sources it owns and one reduction (NCCL
all-reduce / reduce) yields the exact total (up to summation order); the owner of
j then runs the diagonal solve / POTRF / QRCP and broadcasts G1 or U for the next
product.

This module holds the rank assignment and the reduction step; config[1]'s
independent supernodes need neither (pure replicas, `shard_blocks`).
"""

import math

import numpy as np


def shard_blocks(nb, rank, world):
    """Contiguous block range of config[1]'s independent supernodes for `rank`
    (strong-scaling split; the bench runs weak scaling with a full batch per rank)."""
    per = -(-nb // world)
    lo = min(nb, rank * per)
    return lo, min(nb, lo + per)


def subtree_ranks(septree, world):
    """Map every separator-tree node to its owning rank.

    Returns (owner, top): owner maps id(node) -> rank for nodes inside the 2^L
    subtrees (L = ceil(log2 world)), top is the list of the shared top separators
    (pre-order), owned by the rank of their leftmost subtree."""
    L = max(0, math.ceil(math.log2(max(world, 1))))
    owner = {}
    top = []
    counter = [0]

    def assign(nd, r):
        stack = [nd]
        while stack:
            x = stack.pop()
            if x is None:
                continue
            owner[id(x)] = r
            stack.extend([x.left, x.right])

    def walk(nd, depth):
        if nd is None:
            return None
        if depth == L or not nd.is_separator:
            r = counter[0] % world
            counter[0] += 1
            assign(nd, r)
            return r
        top.append(nd)
        rl = walk(nd.left, depth + 1)
        walk(nd.right, depth + 1)
        owner[id(nd)] = rl
        return rl

    walk(septree.root, 0)
    return owner, top


def unit_ranks(sym, world):
    """Owning rank of every unit of a symbolic plan (column ranges are contiguous
    per subtree, so ownership is decided by the unit's first column)."""
    owner, top = subtree_ranks(sym.septree, world)
    spans = []

    def collect(nd):
        if nd is None:
            return
        spans.append((nd.subtree_lo, nd.hi, owner[id(nd)], nd.is_separator, nd.lo))
        collect(nd.left)
        collect(nd.right)

    collect(sym.septree.root)
    part = sym.partition
    top_ranges = {(nd.lo, nd.hi) for nd in top}
    out = []
    for kind, payload in sym.units:
        j0 = payload[0] if kind == "interior" else payload
        c0, c1 = part.cols(j0)
        if kind == "node" and any(lo <= c0 < hi for lo, hi in top_ranges):
            out.append(-1)  # shared top separator: partial sums from every rank
            continue
        best = None
        for lo, hi, r, _, _ in spans:
            if lo <= c0 < hi and (best is None or hi - lo < best[1] - best[0]):
                best = (lo, hi, r)
        out.append(best[2] if best else 0)
    return np.array(out, dtype=np.int64)


def allreduce_partial(tensor, group=None):
    """Sum a per-rank partial product (all ranks get the total)."""
    import torch.distributed as dist

    dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


# ---------------------------------------------------------------------------
# moving factor blocks between ranks


class _Packer:
    """Pickle an object graph with its tensors replaced by slots of one flat
    buffer per dtype (the buffers then travel as single collectives; the host only
    carries the small structural payload)."""

    def __init__(self):
        self.slots = {}    # id(tensor) -> slot
        self.tensors = []  # slot -> tensor

    def persistent_id(self, obj):
        import torch

        if isinstance(obj, torch.Tensor):
            k = self.slots.get(id(obj))
            if k is None:
                k = self.slots[id(obj)] = len(self.tensors)
                self.tensors.append(obj)
            return ("rsc_tensor", k)
        return None

    def dumps(self, obj):
        import io
        import pickle

        f = io.BytesIO()
        p = pickle.Pickler(f, protocol=pickle.HIGHEST_PROTOCOL)
        p.persistent_id = self.persistent_id
        p.dump(obj)
        return f.getvalue()


def pack_tensors(obj, device):
    """obj -> (payload bytes, layout, {dtype name: flat buffer})."""
    import torch

    pk = _Packer()
    payload = pk.dumps(obj)
    groups, layout = {}, []
    for t in pk.tensors:
        key = str(t.dtype).replace("torch.", "")
        lst = groups.setdefault(key, [])
        off = sum(x.numel() for x in lst)
        lst.append(t.reshape(-1))
        layout.append((key, off, tuple(t.shape)))
    bufs = {k: torch.cat(v) if v else torch.empty(0) for k, v in groups.items()}
    sizes = {k: (int(b.numel()), k) for k, b in bufs.items()}
    return payload, layout, sizes, bufs


def unpack_tensors(payload, layout, bufs):
    import io
    import pickle

    views = []
    for key, off, shape in layout:
        n = 1
        for d in shape:
            n *= d
        views.append(bufs[key][off:off + n].view(shape))

    up = pickle.Unpickler(io.BytesIO(payload))
    up.persistent_load = lambda pid: views[pid[1]]
    return up.load()


def _bcast(buf, src, group):
    """Broadcast a (device) tensor; gloo groups stage CUDA tensors through the host."""
    import torch.distributed as dist

    if buf.is_cuda and dist.get_backend(group) == "gloo":
        h = buf.cpu()
        dist.broadcast(h, src, group=group)
        if dist.get_rank(group) != src:
            buf.copy_(h)
        return
    dist.broadcast(buf, src, group=group)


def all_gather_blocks(obj, device, group=None):
    """Every rank contributes an object graph holding device tensors; returns the
    list of all ranks' objects, the remote ones rebuilt as views of one received
    buffer per (rank, dtype) -- one broadcast per rank and dtype."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    payload, layout, sizes, bufs = pack_tensors(obj, device)
    metas = [None] * world
    dist.all_gather_object(metas, (payload, layout, sizes), group=group)
    out = []
    for src in range(world):
        p, lay, sz = metas[src]
        if src == rank:
            rb = bufs
        else:
            rb = {k: torch.empty(n, dtype=getattr(torch, k), device=device) for k, (n, _) in sz.items()}
        for k in sorted(sz):
            if sz[k][0]:
                _bcast(rb[k] if src != rank else bufs[k], src, group)
        out.append(obj if src == rank else unpack_tensors(p, lay, rb))
    return out


# ---------------------------------------------------------------------------
# the sharded factorization


def factorize_distributed(A, config=None, coords=None, group=None, prepared=None):
    """Multi-GPU factorize (one process per GPU, torch.distributed initialised).

    Every rank runs the (deterministic) host symbolic phase, then
      1. sweeps the units of its own nested-dissection subtrees (unit_ranks) --
         no communication: a subtree's update sources all lie inside it;
      2. exchanges only the source panels the shared top separators read (one
         broadcast per rank and dtype; the rest of a subtree never leaves its GPU);
      3. sweeps the top separators with their source sums split: every sum over
         update sources (Schur assembly, Alg. 2/5 implicit products, leaf windows)
         is launched on each rank for the sources it owns, rank 0 adds the A-matrix
         and root-path terms, and each accumulated block is all-reduced before the
         step that consumes it; diagonal solves, POTRFs and QRCPs on the summed
         blocks run replicated;
      4. agrees on the earliest pivot failure in sweep order (restart protocol of
         factor.py:702-718, identical on all ranks).
    The factor stays distributed: each rank keeps its subtrees' blocks and the top
    separators (F.dist); F.apply and pcg_solve run the distributed solve (local
    sweeps, one all-reduce of the top rows per application).  The split sums add
    each rank's partial in a different order than one GPU would, so kept ranks can
    differ from the single-GPU factor only where a QRCP decision sits within
    rounding of the cutoff."""
    import time

    import torch
    import torch.distributed as dist

    from .errors import IndefiniteError, TooManyRestarts
    from .factor import RankStructuredFactor, SolverConfig, _Indefinite, _normalize, prepare
    from .numeric import LevelPass
    from .sparse import as_spd

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    A = _normalize(as_spd(A))
    if prepared is None:
        prepared = prepare(A, config if config is not None else SolverConfig(), coords)
        sym, plan, config, t0, t_plan0, t2 = prepared
    else:
        sym, plan, config, _, _, _ = prepared
        t0 = t_plan0 = time.perf_counter()
        sym.t_ordering = sym.t_symbolic = 0.0
        plan.load_values(A)
        t2 = time.perf_counter()
    owner = unit_ranks(sym, world)
    device = torch.device("cuda", torch.cuda.current_device())
    # the update sources any shared top separator reads (their panels are the only
    # factor data that crosses GPUs)
    top_src = set()
    for u, (kind, j) in enumerate(sym.units):
        if kind == "node" and owner[u] == -1:
            top_src.update(plan.tarr[j]["s"].tolist())
    alpha_d = config.alpha_d
    history, restarts = [alpha_d], 0
    sent = 0
    while True:
        ps = LevelPass(plan, config, alpha_d)
        ps._by_unit = {}
        ps._run_units(lambda u: owner[u] == rank)
        ps.mark_phase()
        counters_a = dict(ps.counters)
        mine = {sid: ps.src_panel[sid] for u, sid in plan.unit_source.items()
                if owner[u] == rank and sid in ps.src_panel and sid in top_src}
        sent = sum(int(t.numel()) * 8 for pr in mine.values() for t in {id(x): x for x in pr}.values())
        remote = {}
        for r, got in enumerate(all_gather_blocks(mine, device, group)):
            if r != rank:
                for sid, (raw, eff) in got.items():
                    ps._set_source(sid, raw, eff)
                    remote[sid] = raw
        src_owner = np.array([max(int(owner[src.unit]), 0) for src in plan.sources], dtype=np.int64)
        ps.split = (rank, world, src_owner, group)
        ps._run_units(lambda u: owner[u] == -1)
        ps.split = None
        try:
            ps.check_pivots()
            cand = None
        except _Indefinite as e:
            cand = (e.unit, e.pivot, e.trees)
        torch.cuda.current_stream().synchronize()
        cands = [None] * world
        dist.all_gather_object(cands, cand, group=group)
        fails = [c for c in cands if c is not None]
        if not fails:
            break
        unit, pivot, trees = min(fails)
        if trees == 0:
            raise IndefiniteError(pivot)
        restarts += 1
        if restarts > config.max_restarts:
            raise TooManyRestarts(
                f"still indefinite after {config.max_restarts} restarts (alpha_d reached {alpha_d:g})")
        alpha_d *= config.alpha_d_growth
        history.append(alpha_d)
    counters_top = {k: ps.counters[k] - counters_a[k] for k in ps.counters}
    node_unit = {payload: u for u, (kind, payload) in enumerate(sym.units) if kind == "node"}
    own_ranks = {k: v for k, v in ps.ranks.items() if owner[node_unit[k[1]]] == rank}
    keep = [u for u in range(len(sym.units)) if owner[u] in (rank, -1)]
    local_stored = 0
    F = RankStructuredFactor(A.n, sym, plan, config)
    F.dunits = [ps._by_unit[u] for u in keep]
    F._mem = ps.P
    mine_units = [ps._by_unit[u] for u in keep if owner[u] == rank]
    top_units = [ps._by_unit[u] for u in keep if owner[u] == -1]
    G = RankStructuredFactor(A.n, sym, plan, config)
    G.dunits = mine_units
    local_stored = G.stored_scalars()
    G.dunits = top_units
    top_stored = G.stored_scalars()
    # small per-rank summaries (host objects): kept ranks, counters, stored scalars
    info = [None] * world
    dist.all_gather_object(info, (own_ranks, counters_a, local_stored, sent), group=group)
    ranks_all = dict(ps.ranks)
    counters = dict(counters_top)
    stored = top_stored
    for r, (ranks_r, cnt_r, st_r, _) in enumerate(info):
        for k in counters:
            counters[k] += cnt_r[k]
        stored += st_r
        if r != rank:
            ranks_all.update(ranks_r)
    src_key = {sid: ("off", sym.units[u][1]) for u, sid in plan.unit_source.items() if sym.units[u][0] == "node"}
    ps.extra_kept = {int(raw.data_ptr()): ranks_all[src_key[sid]] for sid, raw in remote.items()
                     if sid in src_key and src_key[sid] in ranks_all}
    ps._finalize_ranks(ps._last_info)
    flops_a = [0.0] * world
    dist.all_gather_object(flops_a, ps.flops_phase_a, group=group)
    t3 = time.perf_counter()
    F.ranks = ranks_all
    F.source_matrix = A
    F.dist = {"rank": rank, "world": world, "group": group, "top_units": [un.u for un in top_units],
              "local_units": [un.u for un in mine_units], "exchanged_bytes": [x[3] for x in info]}
    part = sym.partition
    st = F.stats
    st.n, st.nnz_lower = A.n, A.nnz_lower
    st.supernodes = part.count
    st.separator_supernodes = int(part.is_separator.sum())
    st.interior_block_count = len(plan.interior)
    st.compressed_offdiag = counters["compressed_off"]
    st.compressed_diag = counters["compressed_diag"]
    st.dense_fallback = counters["dense_fallback"]
    st.stored_scalars = stored
    st.restarts = restarts
    st.alpha_d_final = alpha_d
    st.alpha_d_history = history
    from . import numeric as _nm

    st.model_gflop = (sum(flops_a) + ps.flops - ps.flops_phase_a) / 1e9 if _nm.FLOP_MODEL else float("nan")
    st.phase_times = {"ordering": sym.t_ordering, "symbolic": sym.t_symbolic + (t2 - t_plan0),
                      "numeric": t3 - t2, "total": t3 - t0}
    F.world = world
    return F
