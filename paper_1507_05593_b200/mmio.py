"""Matrix Market / coordinate file I/O and the solver comparison protocol.

Same contracts as the reference (sparse.py:250-312, ordering.py:561-590,
cli.py:176-219): symmetric real coordinate Matrix Market in (upper entries mirrored,
duplicates summed) and canonical lower-triangle out; `x y z` coordinate lines; the
`compare` protocol runs PCG with no preconditioner, Jacobi and the rank-structured
factor on b = ones and reports iterations, convergence, times and stored scalars.
Parsing is vectorized (one numpy pass over the entry block) so external matrices of
the paper's sizes load in seconds.
"""

import io

import numpy as np

from .errors import ParseError, NotSymmetric
from .problems import Coordinates
from .sparse import SparseSpdMatrix

__all__ = ["read_matrix_market", "write_matrix_market", "read_coordinates", "write_coordinates",
           "compare_solvers"]

_HEADER = "%%matrixmarket"


def read_matrix_market(path):
    """Symmetric real coordinate Matrix Market -> SparseSpdMatrix (sparse.py:250-302):
    NotSymmetric for a non-symmetric header, ParseError for anything malformed,
    MissingDiagonal / NonPositiveDiagonal from the matrix validation."""
    with open(path, "r", encoding="ascii") as f:
        header = f.readline()
        if not header.lower().startswith(_HEADER):
            raise ParseError("missing %%MatrixMarket header")
        words = header.split()
        if len(words) != 5:
            raise ParseError(f"malformed header: {header.strip()!r}")
        _, obj, fmt, field, symmetry = (w.lower() for w in words)
        if obj != "matrix" or fmt != "coordinate":
            raise ParseError("only coordinate matrices are supported")
        if field != "real":
            raise ParseError(f"unsupported field {field!r} (only real)")
        if symmetry != "symmetric":
            raise NotSymmetric(f"header declares {symmetry!r}, need symmetric")
        line = f.readline()
        while line and line.lstrip().startswith("%"):
            line = f.readline()
        try:
            m, n, nnz = (int(t) for t in line.split())
        except (ValueError, AttributeError) as exc:
            raise ParseError(f"bad size line: {line.strip()!r}") from exc
        if m != n:
            raise ParseError(f"matrix is {m}x{n}, must be square")
        body = [s for s in (ln.strip() for ln in f) if s and not s.startswith("%")]
    if len(body) != nnz:
        raise ParseError(f"declared {nnz} entries, found {len(body)}")
    if nnz == 0:
        return SparseSpdMatrix.from_coo(n, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    try:
        tab = np.loadtxt(io.StringIO("\n".join(body)), dtype=np.float64, ndmin=2)
    except ValueError as exc:
        raise ParseError(f"bad entry line: {exc}") from exc
    if tab.shape[1] != 3:
        raise ParseError("bad entry line: expected 'i j value'")
    ij = tab[:, :2]
    if np.any(ij != np.round(ij)):
        raise ParseError("bad entry line: non-integer index")
    i, j = ij[:, 0].astype(np.int64), ij[:, 1].astype(np.int64)
    if np.any((i < 1) | (i > n) | (j < 1) | (j > n)):
        bad = int(np.nonzero((i < 1) | (i > n) | (j < 1) | (j > n))[0][0])
        raise ParseError(f"entry ({i[bad]},{j[bad]}) out of range")
    return SparseSpdMatrix.from_coo(n, i - 1, j - 1, tab[:, 2])


def write_matrix_market(A, path):
    """Lower triangle in canonical coordinate form (sparse.py:305-312)."""
    cols = np.repeat(np.arange(A.n, dtype=np.int64), np.diff(A.col_ptr))
    with open(path, "w", encoding="ascii") as f:
        f.write("%%MatrixMarket matrix coordinate real symmetric\n")
        f.write(f"{A.n} {A.n} {A.nnz_lower}\n")
        f.write("".join(f"{r + 1} {c + 1} {v:.17g}\n" for r, c, v in zip(A.row_idx.tolist(), cols.tolist(),
                                                                       A.values.tolist())))


def read_coordinates(path, n=None):
    """`x y z` lines, one per matrix index (ordering.py:561-579)."""
    rows = []
    with open(path, "r", encoding="ascii") as f:
        for line in f:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            parts = s.split()
            if len(parts) != 3:
                raise ParseError(f"bad coordinate line: {s!r}")
            try:
                rows.append([float(p) for p in parts])
            except ValueError as exc:
                raise ParseError(f"bad coordinate line: {s!r}") from exc
    xyz = np.asarray(rows, dtype=np.float64).reshape(-1, 3)
    if n is not None and xyz.shape[0] != n:
        raise ParseError(f"expected {n} coordinate lines, found {xyz.shape[0]}")
    return Coordinates(xyz, source="geometric-file")


def write_coordinates(coords_or_xyz, path):
    """(ordering.py:582-590)."""
    xyz = coords_or_xyz.xyz if hasattr(coords_or_xyz, "xyz") else np.asarray(coords_or_xyz)
    with open(path, "w", encoding="ascii") as f:
        for x, y, z in xyz:
            f.write(f"{x:.17g} {y:.17g} {z:.17g}\n")


def compare_solvers(A, config=None, coords=None, tol=1e-5, max_iter=None, matrix_name=""):
    """The `rschol compare` protocol (cli.py:176-219) on the device: PCG on b = ones
    with no preconditioner, Jacobi and the rank-structured factor; returns the
    report payload {"matrix", "n", "nnz", "config", "methods": {name: {...}}}."""
    from .factor import SolverConfig, factorize
    from .pcg import jacobi_preconditioner, pcg_solve

    config = config if config is not None else SolverConfig()
    F = factorize(A, config, coords=coords)
    b = np.ones(A.n)
    runs = {}
    _, rep = pcg_solve(A, b, preconditioner=None, tol=tol, max_iter=max_iter)
    runs["none"] = (rep, 0)
    _, rep = pcg_solve(A, b, preconditioner=jacobi_preconditioner(A), tol=tol, max_iter=max_iter)
    runs["jacobi"] = (rep, A.n)
    _, rep = pcg_solve(A, b, preconditioner=F, tol=tol, max_iter=max_iter,
                       setup_time=F.stats.phase_times.get("total", 0.0))
    runs["rsc"] = (rep, F.stats.stored_scalars)
    methods = {}
    for name, (rep, scalars) in runs.items():
        methods[name] = {"iterations": rep.iterations, "converged": rep.converged,
                         "relative_residual": rep.relative_residual,
                         "setup_time": rep.wall_times.get("setup", 0.0),
                         "solve_time": rep.wall_times.get("solve", 0.0), "stored_scalars": scalars}
    return {"matrix": str(matrix_name), "n": A.n, "nnz": A.nnz_lower, "config": config.to_dict(),
            "methods": methods}
