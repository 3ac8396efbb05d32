"""Full-size parity on the BASELINE configs (VERDICT r01 "missing" item 1).

The reference's own outputs at full size (tests/golden/full_cfg*.npz, written by
tests/golden/make_fullsize.py from /root/reference in the build container) pin:
symbolic structure (sha256 of perm / supernode starts / row structures), the kept
rank of every compressed block, stored scalars, PCG iterations (+-1) and solution
(1e-8), and the shared-probe Hutchinson estimate of ||PAP^T - LL^T||_F / ||A||_F
(within 1%).  Three factorizations (one-shot, refactorization, graph replay) must
give identical kept ranks and a bit-identical factor (ordered, atomic-free
accumulation in every grouped GEMM).  A kept rank may differ from the reference only where the
reference's own decision sits within rounding of the cutoff: |R_ii|/cutoff of the
last kept or first dropped column within MARGIN of 1 (1e-13 relative
perturbations of G flip such decisions); every such block is reported.
"""
import numpy as np
import pytest

from conftest import golden
import fullsize as FS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

MARGIN = 0.05  # decisions within 5% of the cutoff count as knife-edge


def _check_ranks(F, g):
    diff = FS.rank_diff(F, g)
    hard = [d for d in diff if not (abs(d[4] - 1.0) < MARGIN or abs(d[5] - 1.0) < MARGIN)]
    assert not hard, f"kept ranks differ from the reference away from the cutoff: {hard[:10]}"
    return diff


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_fullsize_config(cuda, cfg):
    from paper_1507_05593_b200 import factorize, pcg_solve
    from paper_1507_05593_b200.factor import SolverConfig, prepare
    from paper_1507_05593_b200.problems import config_problem

    g = FS.fixture(cfg)
    if g is None:
        pytest.skip(f"full_cfg{cfg}.npz not generated")
    A, coords = config_problem(cfg)
    assert A.n == int(g["n"][0]) and A.nnz_lower == int(g["nnz_lower"][0])
    conf = SolverConfig(**FS.KNOBS)
    F = factorize(A, conf, coords=coords)
    # symbolic structure: bit-exact
    assert np.array_equal(FS.sha(F.perm.forward.astype(np.int64)), g["perm_sha"])
    assert np.array_equal(FS.sha(F.partition.starts.astype(np.int64)), g["starts_sha"])
    assert np.array_equal(FS.sha(np.concatenate(F.partition.rows).astype(np.int64)), g["rows_sha"])
    assert F.stats.restarts == int(g["restarts"][0])
    diff = _check_ranks(F, g)
    if not diff:
        assert F.stored_scalars() == int(g["stored_scalars"][0])
    # determinism: refactorizations (eager, then graph replay) repeat every kept rank
    # and every stored FP64 word of the factor
    r = np.random.default_rng(1).standard_normal(A.n)
    z0 = F.apply(r)
    ranks0, dig0 = FS.rank_list(F), FS.factor_digest(F)
    prep = prepare(A, conf, coords)
    for _ in range(2):
        F2 = factorize(A, prepared=prep)
        assert FS.rank_list(F2) == ranks0
        assert FS.factor_digest(F2) == dig0
        z = F2.apply(r)  # the apply's level sums still use FP64 atomics: rounding only
        assert np.abs(z - z0).max() <= 1e-13 * np.abs(z0).max()
        del F2
    b = np.random.default_rng(0).standard_normal(A.n)
    x, rep = pcg_solve(A, b, preconditioner=F, tol=1e-6)
    assert rep.converged
    assert abs(rep.iterations - int(g["pcg_iters"][0])) <= 1
    assert np.linalg.norm(x - g["pcg_x"]) / np.linalg.norm(g["pcg_x"]) < 1e-8
    h, href = FS.hutchinson(A, F), float(g["resid_hutch"][0])
    assert abs(h - href) <= 0.01 * href


def test_cfg1_all_512_blocks(cuda):
    """Config[1] on all 512 blocks: kept rank 48 everywhere, L_D diagonals, factor
    norms and V U^T w against the reference."""
    import torch

    from paper_1507_05593_b200.batched import BatchedSupernodes
    from paper_1507_05593_b200.problems import batched_supernodes

    g = golden("full_cfg1.npz")
    D, B = batched_supernodes(nb=512)
    bs = BatchedSupernodes(512, 256, 2048, 58, q=1)
    bs.D.copy_(torch.from_numpy(D))
    bs.B.copy_(torch.from_numpy(B))
    bs.run()
    torch.cuda.synchronize()
    bs.check_info()
    w = np.random.default_rng(FS.HUTCH_SEED).standard_normal(256)
    ranks, ldd, fro, vuw = [], [], [], []
    for i in range(512):
        LD, LO, V, U = bs.results(i)
        ranks.append(U.shape[1])
        ldd.append(np.diag(LD))
        fro.append((np.linalg.norm(LD), np.linalg.norm(LO), np.linalg.norm(V @ U.T)))
        vuw.append((V @ (U.T @ w))[:64])
    assert ranks == g["ranks"].tolist()
    assert np.abs(np.array(ldd) - g["ld_diag"]).max() <= 1e-12 * np.abs(g["ld_diag"]).max()
    assert np.abs(np.array(fro) / g["fro"] - 1).max() < 1e-11
    vuw, ref = np.array(vuw), g["vuw_head"]
    assert (np.linalg.norm(vuw - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() < 1e-10
    # the reference's rank decisions have a wide margin here
    assert np.nanmin(g["qr_margin"][:, 0]) > 2 and np.nanmax(g["qr_margin"][:, 1]) < 0.5
