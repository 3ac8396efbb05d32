"""Config[1] batched pipeline on the GPU vs the oracle and the reference goldens."""
import numpy as np
import pytest

from conftest import golden, relerr

pytestmark = pytest.mark.gpu


def test_cfg1_batched_matches_reference(cuda):
    import torch
    from oracle import kernels as ok
    from paper_1507_05593_b200.batched import BatchedSupernodes, make_sketches
    from paper_1507_05593_b200.problems import batched_supernodes

    nb = 8
    D, B = batched_supernodes(nb=nb)
    bs = BatchedSupernodes(nb, 256, 2048, 58, q=1, chunk=3)
    bs.D.copy_(torch.from_numpy(D))
    bs.B.copy_(torch.from_numpy(B))
    bs.run()  # device sketches
    torch.cuda.synchronize()
    # the device sketches are the reference's host stream, bit for bit
    assert np.array_equal(bs.Om.cpu().numpy(), make_sketches(nb, 2048, 58, master=0, threads=4))
    bs.check_info()
    g = golden("cfg1.npz")
    for i in range(nb):
        LD, LO, V, U = bs.results(i)
        assert U.shape[1] == 48, i  # kept rank exact
        if i < 4:
            assert int(g[f"rank_{i}"][0]) == U.shape[1]
            assert relerr(LD, g[f"LD_{i}"]) < 1e-12
            assert relerr(LO[:64], g[f"LO_{i}_head"]) < 1e-12
            assert relerr((V @ U.T)[:64], g[f"VUt_{i}_head"]) < 1e-10
        LDo, LOo, Vo, Uo = ok.cfg1_block(D[i], B[i], 58, 1, ok.block_seed(0, 0, i))
        assert relerr(LD, LDo) < 1e-12
        assert relerr(LO, LOo) < 1e-12
        assert relerr(V @ U.T, Vo @ Uo.T) < 1e-10
        assert np.abs(U.T @ U - np.eye(48)).max() < 1e-12


def test_cfg1_indefinite_block_reported(cuda):
    import torch
    from paper_1507_05593_b200.batched import BatchedSupernodes
    from paper_1507_05593_b200.errors import IndefiniteError

    nb, n, m, r = 3, 96, 128, 10
    rng = np.random.default_rng(0)
    D = np.stack([np.eye(n) * 2 for _ in range(nb)])
    D[1, 70, 70] = -1.0
    bs = BatchedSupernodes(nb, n, m, r, q=1)
    bs.D.copy_(torch.from_numpy(D))
    bs.B.copy_(torch.from_numpy(rng.standard_normal((nb, m, n))))
    bs.Om.copy_(torch.from_numpy(rng.standard_normal((nb, m, r))))
    bs.run(sketches=False)
    with pytest.raises(IndefiniteError) as e:
        bs.check_info()
    assert e.value.pivot == 70


def test_cfg1_host_api_round_trip(cuda):
    """factor_compress_host (pinned H2D, device sketches, D2H) == the device path."""
    import torch
    from paper_1507_05593_b200.batched import BatchedSupernodes
    from paper_1507_05593_b200.problems import batched_supernodes

    nb = 4
    D, B = batched_supernodes(nb=nb)
    bs = BatchedSupernodes(nb, 256, 2048, 58, q=1)
    LD, V, U, rank = bs.factor_compress_host(D, B, master=0)
    LD, V, U = LD.copy(), V.copy(), U.copy()
    bs.D.copy_(torch.from_numpy(D))
    bs.B.copy_(torch.from_numpy(B))
    bs.run(master=0)
    torch.cuda.synchronize()
    assert list(rank) == [48] * nb
    assert np.array_equal(LD, bs.D.cpu().numpy())
    # the split-K sketch products accumulate with FP64 atomics: equal up to rounding;
    # columns past the rank are unspecified
    assert relerr(V[:, :, :48], bs.V.cpu().numpy()[:, :, :48]) < 1e-12
    assert relerr(U[:, :, :48], bs.U.cpu().numpy()[:, :, :48]) < 1e-12
