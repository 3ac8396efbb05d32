"""One eager config[2] numeric pass (for ncu kernel captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_05593_b200.factor as FM  # noqa: E402
from paper_1507_05593_b200.benchsparse import KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare  # noqa: E402

FM.GRAPH_REFACTOR = False
A, coords = _problem(2, int(sys.argv[1]) if len(sys.argv) > 1 else 64)
prep = prepare(A, SolverConfig(**KNOBS), coords)
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
F = None
F = factorize(A, prepared=prep)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
