"""The CPU oracle's factorization/apply/PCG vs the reference goldens."""
import numpy as np
import pytest

from conftest import golden, relerr
from factor_cases import CASES, load_case


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference(name):
    from oracle import numeric as on

    A, coords, knobs, keep_dense = load_case(name)
    if A.n > 5000:
        pytest.skip("large case covered by the GPU suite")
    g = golden(f"factor_{name}.npz")
    F = on.factorize(A, on.Config(**knobs), coords=coords)
    assert F.stored_scalars() == int(g["stored_scalars"][0])
    assert F.stats["restarts"] == int(g["restarts"][0])
    got = sorted((k[1], k[2] if k[0] == "diag" else -1, r) for k, r in F.ranks.items())
    assert sorted(tuple(x) for x in g["ranks"].tolist()) == got
    # compressed blocks carry the oracle's own BLAS-threading noise (up to ~7e-9,
    # SURVEY §8(c)); exact factors must agree to rounding
    tol = 1e-8 if g["ranks"].size else 1e-12
    r = np.random.default_rng(1).standard_normal(A.n)
    assert relerr(F.apply(r), g["apply_r"]) < tol
    b = np.random.default_rng(0).standard_normal(A.n)
    x, rep = on.pcg(A, b, F, tol=1e-6)
    assert abs(rep.iterations - int(g["pcg_iters"][0])) <= 1
    assert relerr(x, g["pcg_x"]) < 1e-8
    if keep_dense:
        assert relerr(F.dense_lower(), g["L_dense"]) < tol
