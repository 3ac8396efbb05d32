"""The algorithm-level API (rschol/__init__.py:34-58) on the device factor: SPEC
known answers and identities that pin each function against the stored factor."""
import math

import numpy as np
import pytest

from conftest import relerr
from factor_cases import KNOBS

pytestmark = pytest.mark.gpu


def _factor(N=12, **over):
    from paper_1507_05593_b200 import factorize
    from paper_1507_05593_b200.factor import SolverConfig
    from paper_1507_05593_b200.problems import laplacian_3d
    from paper_1507_05593_b200.sparse import permute_symmetric

    A, coords = laplacian_3d(N)
    F = factorize(A, SolverConfig(**dict(KNOBS, **over)), coords=coords)
    return F, permute_symmetric(A, F.perm)


def test_spec_factor_supernode_2x2(cuda):
    """A = [[4,2],[2,3]] -> L = [[2,0],[1,sqrt 2]]."""
    from paper_1507_05593_b200 import factor_supernode, factorize
    from paper_1507_05593_b200.factor import SolverConfig
    from paper_1507_05593_b200.sparse import SparseSpdMatrix

    A = SparseSpdMatrix.from_dense(np.array([[4.0, 2.0], [2.0, 3.0]]))
    F = factorize(A, SolverConfig(tau_o=float("inf"), interior_blocks=False))
    LD, LO = factor_supernode(A, 0, F)
    assert np.allclose(LD, [[2.0, 0.0], [1.0, math.sqrt(2.0)]], rtol=0, atol=1e-15)
    assert LO.shape == (0, 2)


def test_spec_block_rank():
    """SPEC.md:385-387."""
    from paper_1507_05593_b200.alg import block_rank

    assert block_rank(16, 16, 1.0, 5) == 16
    assert block_rank(1024, 1024, 0.5, 10) == 170
    assert block_rank(1, 1, 1.0, 10) == 1
    assert block_rank(107, 500, 1.0, 10) == 80 and block_rank(108, 500, 1.0, 10) == 81


def test_spec_hand_tree_solve(cuda):
    """leaves D1=[2], D3=[1], coupling V2=U2=[1] (L = [[2,0],[1,1]]):
    L x = [2,3] -> x = [1,2], through the batched Alg. 4 waves of the sweep."""
    import torch

    from paper_1507_05593_b200 import engine as E
    from paper_1507_05593_b200.diagtree import TreeShape
    from paper_1507_05593_b200.factor import DenseTri, DeviceTree, DevLR
    from paper_1507_05593_b200.numeric import diag_solve_many

    class Piece:
        def __init__(self, size, left=None, right=None):
            self.size, self.left, self.right = size, left, right

        @property
        def is_leaf(self):
            return self.left is None

    shape = TreeShape(2, 0, Piece(2, Piece(1), Piece(1)))
    tree = DeviceTree(shape)
    for s, v in ((1, 2.0), (3, 1.0)):
        L = E.to_dev(np.array([[v]]))
        D = E.empty(1, 64)
        E.trtri_diag_batched([L.data_ptr()], [1], [1], [D.data_ptr()])
        tree.blocks[s] = DenseTri(L, D)
    one = E.to_dev(np.array([[1.0]]))
    tree.blocks[2] = DevLR(one, one.clone(), one.clone())

    class Node:
        diag = tree

    X = E.to_dev(np.array([[2.0], [3.0]]))
    diag_solve_many([(Node, X, False)], E.scratch)
    torch.cuda.synchronize()
    assert np.allclose(X.cpu().numpy()[:, 0], [1.0, 2.0], rtol=0, atol=1e-15)


def test_factor_object_model(cuda):
    """.nodes / .interior / .units mirror rschol's containers (factor.py:163-172)."""
    from paper_1507_05593_b200 import DiagBlockTree, InteriorBlock, LowRankBlock, SupernodeFactor

    F, B = _factor(16, tau_d=64)
    kinds = [k for k, _ in F.units]
    assert len(F.units) == len(F.sym.units) and set(kinds) <= {"interior", "node"}
    assert all(isinstance(o, InteriorBlock) for k, o in F.units if k == "interior")
    assert len(F.interior) == kinds.count("interior")
    nodes = [o for k, o in F.units if k == "node"]
    assert all(isinstance(o, SupernodeFactor) and F.nodes[o.j] is o for o in nodes)
    assert any(isinstance(o.diag, DiagBlockTree) for o in nodes)
    assert any(isinstance(o.offdiag, LowRankBlock) for o in nodes)
    # the views reassemble the dense factor exactly
    L = np.zeros((F.n, F.n))
    for kind, o in F.units:
        if kind == "interior":
            for m in o.members:
                L[m.c0:m.c1, m.c0:m.c1] = m.diag
                if m.nrows_in_block:
                    L[m.rows[:m.nrows_in_block], m.c0:m.c1] = m.offdiag
            if o.off_rows.size:
                L[o.off_rows, o.c0:o.c1] = o.solve(o.coupling.T.toarray()).T
        else:
            L[o.c0:o.c1, o.c0:o.c1] = o.diag.assemble_dense() if isinstance(o.diag, DiagBlockTree) else o.diag
            if o.rows.size and o.offdiag is not None:
                L[o.rows, o.c0:o.c1] = o.offdiag.dense() if isinstance(o.offdiag, LowRankBlock) else o.offdiag
    assert relerr(L, F.dense_lower()) < 1e-13
    assert sum(o.stored_scalars() if k == "interior" else 0 for k, o in F.units) > 0


def test_alg_products_against_stored_factor(cuda):
    """Alg. 2/3 and mirrors: the implicit product applied to the kept basis U is the
    stored V (V = L_O U, factor.py:503-504); Alg. 3 with the block's own seed repeats
    the sweep's kept rank and V U^T; the transposed product is the adjoint."""
    from paper_1507_05593_b200 import (LowRankBlock, approximate_off_diagonal, collect_sources,
                                       off_diagonal_multiply, off_diagonal_multiply_trans)
    from paper_1507_05593_b200.factor import _block_seed

    F, B = _factor(16, tau_d=64)
    comp = [o for k, o in F.units if k == "node" and isinstance(o.offdiag, LowRankBlock)]
    assert comp
    rng = np.random.default_rng(3)
    for o in comp[:3]:
        srcs = collect_sources(F, o.j)
        V = off_diagonal_multiply(B, o.j, F, o.offdiag.U, sources=srcs)
        assert relerr(V, o.offdiag.V) < 1e-12
        g, h = rng.standard_normal((o.ncols, 3)), rng.standard_normal((o.rows.size, 3))
        lhs = np.sum(off_diagonal_multiply(B, o.j, F, g) * h)
        rhs = np.sum(g * off_diagonal_multiply_trans(B, o.j, F, h))
        assert abs(lhs - rhs) <= 1e-11 * abs(lhs)
        from paper_1507_05593_b200.symbolic import block_rank

        r = block_rank(o.rows.size, o.ncols, F.config.alpha_o, F.config.oversample)
        lr = approximate_off_diagonal(B, o.j, F, r, power_iters=F.config.power_iters,
                                      seed=_block_seed(F.config.seed, 0, o.j))
        assert lr.rank == o.offdiag.rank
        assert relerr(lr.dense(), o.offdiag.dense()) < 1e-10


def test_alg_supernode_and_tree_functions(cuda):
    """Alg. 1 on a dense-diagonal node equals the stored (L_D, L_O); Alg. 4 equals a
    dense solve with the assembled tree; Alg. 6 repeats every stored leaf; Alg. 3 on
    tree blocks repeats the stored compressed blocks."""
    from paper_1507_05593_b200 import (DiagBlockTree, LowRankBlock, approximate_diagonal_block, diagonal_multiply,
                                       diagonal_solve, factor_diagonal, factor_supernode)
    from paper_1507_05593_b200.factor import _block_seed
    from paper_1507_05593_b200.symbolic import block_rank

    F, B = _factor(16, tau_d=64)
    nodes = [o for k, o in F.units if k == "node"]
    dense = [o for o in nodes if not isinstance(o.diag, DiagBlockTree) and not isinstance(o.offdiag, LowRankBlock)]
    for o in dense[:3]:
        LD, LO = factor_supernode(B, o.j, F)
        assert relerr(LD, o.diag) < 1e-12
        if o.rows.size:
            assert relerr(LO, o.offdiag) < 1e-12
    trees = [o for o in nodes if isinstance(o.diag, DiagBlockTree)]
    assert trees
    rng = np.random.default_rng(4)
    for o in trees[:2]:
        Ld = o.diag.assemble_dense()
        G = rng.standard_normal((o.ncols, 2))
        assert relerr(diagonal_solve(F, o.j, G), np.linalg.solve(Ld, G)) < 1e-12
        assert relerr(diagonal_solve(F, o.j, G, transpose=True), np.linalg.solve(Ld.T, G)) < 1e-12
        for s in o.diag.inorder_ids():
            nd = o.diag.nodes[s]
            if nd.is_leaf:
                assert relerr(factor_diagonal(B, F, o.j, s), o.diag.blocks[s]) < 1e-12
                continue
            b = o.diag.blocks[s]
            (r0, r1), (c0, c1) = o.diag.col_span(s)
            if isinstance(b, LowRankBlock):
                W = diagonal_multiply(B, F, o.j, s, b.U)
                assert relerr(W, b.V) < 1e-12
                r = block_rank(r1 - r0, c1 - c0, F.stats.alpha_d_final, F.config.oversample)
                lr = approximate_diagonal_block(B, F, o.j, s, r, power_iters=F.config.power_iters,
                                                seed=_block_seed(F.config.seed, 1, o.j, s))
                assert lr.rank == b.rank and relerr(lr.dense(), b.dense()) < 1e-10
            else:
                W = diagonal_multiply(B, F, o.j, s, np.eye(c1 - c0))
                assert relerr(W, b) < 1e-12


def test_factor_interior_block_matches_factor(cuda):
    """interior.py:105-156: the block factor equals the sweep's interior unit."""
    from paper_1507_05593_b200 import factor_interior_block

    F, B = _factor(16, tau_d=64)
    blk = F.interior[0]
    ids = [m.j for m in blk.members]
    mine = factor_interior_block(B, F.partition, ids, block_id=0)
    assert np.array_equal(mine.off_rows, blk.off_rows)
    for a, b in zip(mine.members, blk.members):
        assert relerr(a.diag, b.diag) < 1e-13
    G = np.random.default_rng(5).standard_normal((blk.ncols, 2))
    assert relerr(mine.solve(G), blk.solve(G)) < 1e-13
