"""paper_1507_05593_b200 -- B200-native numeric engine of the rank-structured
supernodal Cholesky preconditioner (Chadwick & Bindel, arXiv 1507.05593).

Drop-in for the hot path of the reference package `rschol`: the numeric
factorization (`factorize`, `RankStructuredFactor.apply`) and its use as a PCG
preconditioner (`pcg_solve`).  Host code is Python; every FLOP of the numeric
phase runs in hand-written sm_100a kernels (librsc_b200.so, C ABI in
include/rsc_b200.h).  There is no CPU fallback.
"""

from .errors import (
    BreakdownNonSPD,
    DimensionMismatch,
    IndefiniteError,
    MissingCoordinates,
    MissingDiagonal,
    NoConvergenceWarning,
    NonPositiveDiagonal,
    NotSubset,
    NotSymmetric,
    ParseError,
    RscholError,
    ShapeMismatch,
    SingularDiagonal,
    TooManyRestarts,
)
from .sparse import Permutation, SparseSpdMatrix, permute_symmetric, strip_explicit_zeros

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-backed modules load lazily so that the host-only parts (symbolic
    # analysis, generators) import without torch.cuda
    import importlib

    lazy = {
        "dense_cholesky": "kernels", "tri_solve": "kernels", "orthonormalize": "kernels",
        "gaussian_matrix": "kernels", "low_rank_approx": "kernels",
        "factorize": "factor", "SolverConfig": "factor", "RankStructuredFactor": "factor",
        "FactorStats": "factor", "block_rank": "factor",
        "pcg_solve": "pcg", "SolveReport": "pcg", "jacobi_preconditioner": "pcg",
        "apply_preconditioner": "pcg",
        # algorithm-level API of rschol/__init__.py:34-58, on the device factor
        "collect_sources": "alg", "factor_supernode": "alg", "off_diagonal_multiply": "alg",
        "off_diagonal_multiply_trans": "alg", "approximate_off_diagonal": "alg", "diagonal_solve": "alg",
        "diagonal_multiply": "alg", "factor_diagonal": "alg", "approximate_diagonal_block": "alg",
        "factor_interior_block": "alg", "build_diag_tree": "alg",
        # reference-shaped factor containers (views over the device blocks)
        "LowRankBlock": "views", "SupernodeFactor": "views", "InteriorBlock": "views",
        "DiagBlockTree": "views", "UpdateSource": "views",
        "read_matrix_market": "mmio", "write_matrix_market": "mmio", "read_coordinates": "mmio",
        "write_coordinates": "mmio", "compare_solvers": "mmio",
    }
    if name in lazy:
        mod = importlib.import_module(f".{lazy[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
