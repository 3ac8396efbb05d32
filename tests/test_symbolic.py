"""Host symbolic phase vs the reference's own symbolic output (bit-exact)."""
import numpy as np
import pytest

from conftest import golden
from factor_cases import CASES, load_case


def units_code(units):
    out = []
    for kind, payload in units:
        out.append((0, payload[0], payload[-1]) if kind == "interior" else (1, payload, payload))
    return np.array(out, dtype=np.int64).reshape(-1, 3)


@pytest.mark.parametrize("name", sorted(CASES))
def test_symbolic_plan_bit_exact(name):
    from paper_1507_05593_b200.symbolic import analyze

    A, coords, knobs, _ = load_case(name)
    g = golden(f"factor_{name}.npz")
    plan = analyze(A, knobs["tau_o"], knobs["tau_d"], knobs["interior_blocks"], coords=coords)
    part = plan.partition
    assert np.array_equal(plan.perm.forward, g["perm"])
    assert np.array_equal(part.starts, g["starts"])
    assert np.array_equal(part.is_separator, g["is_sep"])
    ptr = np.concatenate([[0], np.cumsum([r.size for r in part.rows])])
    assert np.array_equal(ptr, g["rows_ptr"])
    assert np.array_equal(np.concatenate(part.rows), g["rows_idx"])
    assert np.array_equal(units_code(plan.units), g["units"])
    for key in g.files:
        if key.startswith("leaves_"):
            j = int(key.split("_")[1])
            assert plan.sep_splits[j].leaf_sizes() == list(g[key])


def test_block_rank_kats():
    from paper_1507_05593_b200.symbolic import block_rank

    assert block_rank(16, 16, 1.0, 5) == 16
    assert block_rank(1024, 2000, 0.5, 10) == 170
    assert block_rank(1, 1, 1.0, 10) == 1
    assert block_rank(0, 5, 1.0, 10) == 0
    # the compression threshold of SURVEY §8(a15): k >= 107 and k != 108 at alpha 1, p 10
    comp = [k for k in range(2, 400) if block_rank(k, k, 1.0, 10) < 0.75 * k]
    assert comp[0] == 107 and 108 not in comp and 109 in comp


def test_etree_colcounts_against_dense_symbolic():
    """Elimination tree / column counts vs a brute-force dense symbolic factorization."""
    from paper_1507_05593_b200.sparse import SparseSpdMatrix
    from paper_1507_05593_b200.symbolic import etree_postorder_counts

    rng = np.random.default_rng(3)
    for n in (1, 5, 17, 40):
        M = (rng.random((n, n)) < 0.15).astype(float)
        M = M + M.T + n * np.eye(n)
        A = SparseSpdMatrix.from_dense(M)
        P = np.tril(M != 0)
        for j in range(n):
            for k in range(j):
                if P[j, k]:
                    P[j + 1:, j] |= P[j + 1:, k]
        parent, post, counts = etree_postorder_counts(A)
        assert np.array_equal(counts, P.sum(axis=0))
        for j in range(n):
            below = np.nonzero(P[j + 1:, j])[0]
            assert parent[j] == (j + 1 + below[0] if below.size else -1)
        assert sorted(post.tolist()) == list(range(n))
