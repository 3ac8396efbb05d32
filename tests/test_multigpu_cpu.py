"""The N>1 decomposition on CPU with gloo, world size 2.

Checks (1) the subtree ownership of units, (2) that the exchange step -- per-rank
partial sums of a top separator's source terms, all-reduced -- reproduces the
single-process Schur block exactly, using the oracle's arithmetic, and (3) the
max-over-ranks timing reduction bench.py uses.
"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import numeric as on
        from paper_1507_05593_b200.distributed import allreduce_partial, unit_ranks
        from paper_1507_05593_b200.problems import laplacian_3d
        from paper_1507_05593_b200.symbolic import analyze

        A, coords = laplacian_3d(10)
        cfg = on.Config(tau_o=16, oversample=4, tau_d=10**9)
        sym = analyze(A, cfg.tau_o, cfg.tau_d, True, coords=coords)
        owners = unit_ranks(sym, world)
        F = on.factorize(A, cfg, coords=coords, plan=sym)
        full = sym.B.to_csr_full()
        # the root separator is the last unit; its update sources live in both subtrees
        root = F.units[-1][1]
        srcs_by_rank = {}
        for u, (kind, obj) in enumerate(F.units[:-1]):
            rows = obj.off_rows if kind == "interior" else obj.rows
            if rows is None or not rows.size:
                continue
            lo, hi = np.searchsorted(rows, (root.c0, root.c1))
            if lo == hi:
                continue
            src = on.Src("interior", rows, obj.c0, blk=obj) if kind == "interior" else on.Src("node", rows, obj.c0,
                                                                                              node=obj)
            srcs_by_rank.setdefault(int(owners[u]), []).append(src)
        # every rank: its partial sum of source terms of the root Schur block
        mine = sorted(srcs_by_rank.get(rank, []), key=lambda s: s.order)
        UD_full, _ = on.assemble_schur(full, root, root.rows, [s for r in srcs_by_rank for s in srcs_by_rank[r]],
                                       want_off=False)
        A_CC = full[root.c0:root.c1, root.c0:root.c1].toarray()
        part, _ = on.assemble_schur(full, root, root.rows, mine, want_off=False)
        contrib = torch.from_numpy(A_CC - part)  # this rank's sum of source terms
        allreduce_partial(contrib)
        UD_dist = A_CC - contrib.numpy()
        err = np.linalg.norm(UD_dist - UD_full) / np.linalg.norm(UD_full)
        t = torch.tensor([0.1 * (rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        out.put((rank, float(err), sorted(srcs_by_rank), float(t.item()),
                 int((owners == 0).sum()), int((owners == 1).sum()), int((owners == -1).sum())))
    finally:
        dist.destroy_process_group()


def test_subtree_exchange_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, err, ranks_with_sources, tmax, n0, n1, nshared in res:
        assert err < 1e-13, err
        assert ranks_with_sources == [0, 1]  # the root really needs both subtrees
        assert abs(tmax - 0.2) < 1e-15  # max over ranks
        assert n0 > 0 and n1 > 0 and nshared >= 1


def test_shard_blocks_cover_batch():
    from paper_1507_05593_b200.distributed import shard_blocks

    for world in (1, 2, 3, 8):
        spans = [shard_blocks(512, r, world) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == 512
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def _block_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1507_05593_b200.distributed import all_gather_blocks
        from paper_1507_05593_b200.factor import DenseTri, DevLR, NodeUnit

        g = torch.Generator().manual_seed(rank)
        L = torch.randn(5, 5, generator=g, dtype=torch.float64)
        V = torch.randn(7, 6, generator=g, dtype=torch.float64)[:, :3]  # trimmed (non-contiguous) view
        U = torch.randn(4, 3, generator=g, dtype=torch.float64)
        un = NodeUnit(10 + rank, rank, 0, 4, np.arange(rank, rank + 7))
        un.diag = DenseTri(L, torch.zeros(5, 64, dtype=torch.float64))
        un.off = DevLR(V, U, V * 2)
        obj = {"unit": un, "twice": (U, U), "ranks": {("off", rank): 3}, "ints": torch.arange(rank + 2, dtype=torch.int32)}
        got = all_gather_blocks(obj, torch.device("cpu"))
        res = []
        for r, o in enumerate(got):
            g = torch.Generator().manual_seed(r)
            L = torch.randn(5, 5, generator=g, dtype=torch.float64)
            V = torch.randn(7, 6, generator=g, dtype=torch.float64)[:, :3]
            U = torch.randn(4, 3, generator=g, dtype=torch.float64)
            u = o["unit"]
            res.append(bool(torch.equal(u.diag.L, L) and torch.equal(u.off.V, V) and torch.equal(u.off.E, 2 * V)
                            and torch.equal(u.off.U, U) and u.u == 10 + r and np.array_equal(u.rows, np.arange(r, r + 7))
                            and o["twice"][0] is o["twice"][1] and o["ranks"] == {("off", r): 3}
                            and torch.equal(o["ints"], torch.arange(r + 2, dtype=torch.int32))))
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_all_gather_blocks_gloo_world2():
    """Factor blocks (unit records holding tensors, trimmed views, shared tensors,
    int tensors) travel between ranks as one flat buffer per dtype + a pickled
    structure, and come back identical on every rank."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        assert ok == [True, True], (rank, ok)
