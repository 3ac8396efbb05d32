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
