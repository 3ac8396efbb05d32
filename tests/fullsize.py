"""Full-size parity helpers (test infrastructure): L multiply of the device factor,
the shared-probe Hutchinson residual and the comparison against the reference
fixtures written by tests/golden/make_fullsize.py."""
import hashlib
import os

import numpy as np

from conftest import GOLDEN

KNOBS = dict(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=256, power_iters=1, seed=0,
             interior_blocks=True, max_restarts=10)
HUTCH_SEED = 20251020  # same probes as make_fullsize.py
HUTCH_K = 8


def fixture(cfg):
    p = os.path.join(GOLDEN, f"full_cfg{cfg}.npz")
    return np.load(p) if os.path.exists(p) else None


def sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), dtype=np.uint8).copy()


def lower_mul(F, X, transpose=False):
    """Y = L X (or L^T X) for the device factor F, X an n x k torch tensor in the
    permuted ordering.  Block layout as RankStructuredFactor.dense_lower."""
    import torch

    from paper_1507_05593_b200.factor import DeviceTree, DevLR

    Y = torch.zeros_like(X)
    dev = X.device

    def idx(rows):
        return torch.as_tensor(np.asarray(rows, dtype=np.int64), device=dev)

    def put(block, r0, r1, c0, c1):
        # dense block at rows [r0, r1) x cols [c0, c1)
        if transpose:
            Y[c0:c1] += block.T @ X[r0:r1]
        else:
            Y[r0:r1] += block @ X[c0:c1]

    def put_lr(b, rr, c0, c1):
        if b.k == 0:
            return
        if transpose:
            Y[c0:c1] += b.U @ (b.V.T @ X[rr])
        else:
            Y.index_add_(0, rr, b.V @ (b.U.T @ X[c0:c1]))

    def put_rows(block, rr, c0, c1):
        if transpose:
            Y[c0:c1] += block.T @ X[rr]
        else:
            Y.index_add_(0, rr, block @ X[c0:c1])

    for un in F.dunits:
        c0, c1 = un.c0, un.c1
        if isinstance(un.diag, DeviceTree):
            shape = un.diag.shape
            for s, nd in shape.nodes.items():
                (r0, r1), (k0, k1) = shape.span(s)
                b = un.diag.blocks[s]
                if nd.is_leaf:
                    put(torch.tril(b.L), c0 + r0, c0 + r1, c0 + k0, c0 + k1)
                elif isinstance(b, DevLR):
                    put_lr(b, torch.arange(c0 + r0, c0 + r1, device=dev), c0 + k0, c0 + k1)
                else:
                    put(b, c0 + r0, c0 + r1, c0 + k0, c0 + k1)
        else:
            put(torch.tril(un.diag.L), c0, c1, c0, c1)
        if un.rows.size and un.off is not None:
            rr = idx(un.rows)
            if isinstance(un.off, DevLR):
                put_lr(un.off, rr, c0, c1)
            else:
                put_rows(un.off, rr, c0, c1)
    return Y


def hutchinson(A, F):
    """||P A P^T - L L^T||_F estimate with the fixture's probes."""
    import torch

    from paper_1507_05593_b200.sparse import permute_symmetric

    B = permute_symmetric(A, F.perm)
    Bf = B.to_csr_full()
    Z = np.random.default_rng(HUTCH_SEED).standard_normal((A.n, HUTCH_K))
    BZ = Bf @ Z
    Zd = torch.as_tensor(Z, device="cuda")
    LLtZ = lower_mul(F, lower_mul(F, Zd, transpose=True)).cpu().numpy()
    a_fro = float(np.sqrt(np.sum(np.asarray(Bf.data) ** 2)))
    return float(np.linalg.norm(BZ - LLtZ) / np.sqrt(HUTCH_K) / a_fro)


def factor_digest(F):
    """Order-sensitive 64-bit digest of every numeric block of the device factor
    (bitwise: two factors agree iff every stored FP64 word agrees, up to hash
    collisions)."""
    import torch

    from paper_1507_05593_b200.factor import DeviceTree, DevLR

    acc = torch.zeros((), dtype=torch.int64, device="cuda")
    k = 0

    def mix(t):
        nonlocal acc, k
        if t is None or t.numel() == 0:
            return
        x = t.contiguous().view(-1).view(torch.int64)
        w = torch.arange(1, x.numel() + 1, device=x.device, dtype=torch.int64) * 2654435761 + k
        acc = acc + ((x ^ (x >> 31)) * w).sum()
        k += 1

    for un in F.dunits:
        blocks = []
        if isinstance(un.diag, DeviceTree):
            for s in sorted(un.diag.blocks):
                blocks.append(un.diag.blocks[s])
        else:
            blocks.append(un.diag)
        blocks.append(un.off)
        for b in blocks:
            if isinstance(b, DevLR):
                mix(b.V), mix(b.U)
            elif hasattr(b, "L"):
                mix(b.L)
            elif b is not None:
                mix(b)
    return int(acc.item())


def rank_list(F):
    return sorted((k[1], k[2] if k[0] == "diag" else -1, r) for k, r in F.ranks.items())


def rank_diff(F, g):
    """Compressed blocks whose kept rank differs from the reference, with the
    reference's decision margins (|R_ii| / cutoff of the last kept / first dropped
    column) for that block: [(j, s, ours, ref, last_kept_margin, first_drop_margin)]."""
    ref = {(int(j), int(s)): int(r) for j, s, r in g["ranks"]}
    ours = {(k[1], k[2] if k[0] == "diag" else -1): r for k, r in F.ranks.items()}
    marg = {}
    for (kind, j, s, m, k, kept), (a, b) in zip(g["qr_tag"], g["qr_margin"]):
        marg[(int(j), int(s) if kind == 1 else -1)] = (float(a), float(b))
    out = []
    for key in sorted(set(ref) | set(ours)):
        if ref.get(key) != ours.get(key):
            out.append(key + (ours.get(key), ref.get(key)) + marg.get(key, (np.nan, np.nan)))
    return out
