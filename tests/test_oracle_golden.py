"""Pin the CPU oracle to golden vectors produced by the reference itself."""
import numpy as np
import pytest

from conftest import golden, relerr
from oracle import kernels as ok


def test_chol_matches_reference():
    g = golden("kernels.npz")
    for n in (1, 7, 23, 50, 64, 65, 130, 256):
        assert relerr(ok.chol(g[f"chol_in_{n}"]), g[f"chol_out_{n}"]) < 1e-14


def test_chol_known_answers():
    L = ok.chol(np.array([[4.0, 2.0], [2.0, 3.0]]))
    assert np.allclose(L, [[2, 0], [1, np.sqrt(2)]])
    with pytest.raises(ok.OracleIndefinite) as e:
        ok.chol(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert e.value.pivot == 1


def test_trisolve_matches_reference():
    g = golden("kernels.npz")
    L, B = g["tri_L"], g["tri_B"]
    assert relerr(ok.trisolve(L, B), g["tri_left"]) < 1e-14
    assert relerr(ok.trisolve(L, B, transpose=True), g["tri_left_t"]) < 1e-14
    assert relerr(ok.trisolve(L, B.T, transpose=True, side="right"), g["tri_right_t"]) < 1e-14
    assert relerr(ok.trisolve(L, B.T, side="right"), g["tri_right"]) < 1e-14


def test_orth_matches_reference():
    g = golden("kernels.npz")
    for tag in "abc":
        Q = ok.orth(g[f"orth_in_{tag}"])
        Qr = g[f"orth_out_{tag}"]
        assert Q.shape == Qr.shape
        assert relerr(Q @ Q.T, Qr @ Qr.T) < 1e-12


def test_seeds_and_sketch_stream():
    g = golden("kernels.npz")
    assert np.array_equal(ok.gauss(7, 3, 99), g["gauss_7x3_99"])
    assert ok.block_seed(0, 0, 5) == int(g["block_seed_0_0_5"][0])
    assert ok.block_seed(0, 1, 9, 3) == int(g["block_seed_0_1_9_3"][0])


def test_range_finder_matches_reference():
    g = golden("kernels.npz")
    V, U = ok.range_finder(g["lra_in"], 30, power_iters=1, seed=5)
    assert U.shape == g["lra_U"].shape
    assert relerr(V @ U.T, g["lra_V"] @ g["lra_U"].T) < 1e-12


def test_cfg1_composition_matches_reference():
    from paper_1507_05593_b200.problems import batched_supernodes

    g = golden("cfg1.npz")
    D, B = batched_supernodes(nb=4)
    assert np.array_equal(D[0], g["D0"]) and np.array_equal(B[0, :8], g["B0_head"])
    for i in range(4):
        LD, LO, V, U = ok.cfg1_block(D[i], B[i], 58, 1, ok.block_seed(0, 0, i))
        assert U.shape[1] == int(g[f"rank_{i}"][0]) == 48
        assert relerr(LD, g[f"LD_{i}"]) < 1e-14
        assert relerr(LO[:64], g[f"LO_{i}_head"]) < 1e-13
        assert relerr((V @ U.T)[:64], g[f"VUt_{i}_head"]) < 1e-12
