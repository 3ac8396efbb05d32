"""engine.split_k: descriptor arithmetic of the K-slab split (host only)."""
import numpy as np

from paper_1507_05593_b200 import engine as E


def test_split_k_offsets_and_flags():
    p = E.gemm_problems(3)
    p["A"], p["B"], p["C"] = 1000, 50000, 90000
    p["M"], p["N"] = 40, 30
    p["K"] = [600, 100, 513]
    p["lda"], p["ldb"], p["ldc"] = 64, 32, 30
    p["b_rows"] = [0, 0, 7000]
    p["beta"] = 0.0
    q = E.split_k(p, True, False, 256)
    assert q.size == 3 + 1 + 3
    assert list(q["K"]) == [256, 256, 88, 100, 256, 256, 1]
    assert int(q["K"][:3].sum()) == 600 and int(q["K"][4:].sum()) == 513
    # transA: A advances k0 rows of lda doubles; B advances k0 rows (no gather)
    assert list(q["A"][:3]) == [1000, 1000 + 256 * 64 * 8, 1000 + 512 * 64 * 8]
    assert list(q["B"][:3]) == [50000, 50000 + 256 * 32 * 8, 50000 + 512 * 32 * 8]
    # gathered B: the index pointer advances, B stays
    assert list(q["B"][4:]) == [50000] * 3
    assert list(q["b_rows"][4:]) == [7000, 7000 + 4 * 256, 7000 + 4 * 512]
    # split problems accumulate atomically, the unsplit one keeps its epilogue
    assert list(q["atomic"]) == [1, 1, 1, 0, 1, 1, 1]
    assert list(q["beta"]) == [1.0, 1.0, 1.0, 0.0, 1.0, 1.0, 1.0]
    # no split needed: same array back
    assert E.split_k(p, True, False, 1024) is p
