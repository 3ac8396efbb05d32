"""Matrix Market / coordinate I/O (reference sparse.py:250-312, ordering.py:561-590;
cases after the reference's tests/test_sparse.py)."""
import numpy as np
import pytest


def _write(tmp_path, text, name="a.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_round_trip_laplacian(tmp_path):
    from paper_1507_05593_b200.mmio import read_matrix_market, write_matrix_market
    from paper_1507_05593_b200.problems import elasticity_3d

    A, _ = elasticity_3d(4, strip_zeros=True)
    p = tmp_path / "el.mtx"
    write_matrix_market(A, p)
    B = read_matrix_market(p)
    assert B.n == A.n and np.array_equal(B.col_ptr, A.col_ptr) and np.array_equal(B.row_idx, A.row_idx)
    assert np.array_equal(B.values, A.values)  # %.17g round-trips FP64 exactly


def test_upper_entries_mirrored_and_duplicates_summed(tmp_path):
    from paper_1507_05593_b200.mmio import read_matrix_market

    p = _write(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 5\n"
                         "1 1 4\n2 2 3\n3 3 2\n1 2 -1\n2 1 -0.5\n")
    A = read_matrix_market(p)
    D = A.dense()
    assert np.allclose(D, [[4, -1.5, 0], [-1.5, 3, 0], [0, 0, 2]])


@pytest.mark.parametrize("text,exc", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n2 2 1\n", "NotSymmetric"),
    ("%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n2 2 1\n", "ParseError"),
    ("%%MatrixMarket matrix array real symmetric\n2 2\n1\n2\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate complex symmetric\n2 2 1\n1 1 1 0\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n2 2 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n3 2 1\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n2 2 x\n", "ParseError"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 1 1\n", "MissingDiagonal"),
    ("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1\n2 2 -1\n", "NonPositiveDiagonal"),
])
def test_errors(tmp_path, text, exc):
    from paper_1507_05593_b200 import errors
    from paper_1507_05593_b200.mmio import read_matrix_market

    with pytest.raises(getattr(errors, exc)):
        read_matrix_market(_write(tmp_path, text))


def test_coordinates_round_trip(tmp_path):
    from paper_1507_05593_b200 import errors
    from paper_1507_05593_b200.mmio import read_coordinates, write_coordinates

    xyz = np.random.default_rng(0).standard_normal((7, 3))
    p = tmp_path / "c.xyz"
    write_coordinates(xyz, p)
    assert np.array_equal(read_coordinates(p, n=7).xyz, xyz)
    with pytest.raises(errors.ParseError):
        read_coordinates(p, n=8)
    with pytest.raises(errors.ParseError):
        read_coordinates(_write(tmp_path, "1 2\n", "bad.xyz"))
