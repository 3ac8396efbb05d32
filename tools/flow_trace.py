"""Trace of one dataflow apply (rsc_apply_flow_trace): per item take / go / end
times and SM, plus the op table and graph, saved to gpurun_out/flow_trace_cfgN.npz
for offline critical-path analysis.  python tools/flow_trace.py CFG"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench_sparse import GRID, KNOBS, _problem  # noqa: E402
from paper_1507_05593_b200 import _lib  # noqa: E402
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.apply import DeviceApply  # noqa: E402
from paper_1507_05593_b200.factor import SolverConfig, factorize  # noqa: E402

cfg = int(sys.argv[1])
A, coords = _problem(cfg, GRID[cfg])
F = factorize(A, SolverConfig(**KNOBS), coords=coords)
r = E.to_dev(np.random.default_rng(1).standard_normal(A.n))
DeviceApply.FLOW = True
ap = DeviceApply(F)
z = E.empty(A.n)
for _ in range(3):
    ap(r, z)
lib = _lib.load()
d, io, nd, sp, sc, st = ap.flow_dev
tr = torch.zeros(4 * ap.flow_items, dtype=torch.int64, device="cuda")
for _ in range(3):
    ap.tall.zero_()
    torch.cuda.synchronize()
    _lib.check(lib.rsc_apply_flow_trace(d.data_ptr(), io.data_ptr(), nd.data_ptr(), sp.data_ptr(), sc.data_ptr(),
                                        st.data_ptr(), ap.flow_nops, ap.flow_items, tr.data_ptr(),
                                        E.stream_handle()), "trace")
    torch.cuda.synchronize()
items = [it for ph in ap.phases for it in ph.items]
phase = np.concatenate([np.full(len(ph.items), i) for i, ph in enumerate(ap.phases)])
c = list(zip(*items))
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed(f"gpurun_out/flow_trace_cfg{cfg}.npz", trace=tr.cpu().numpy().reshape(-1, 4),
                    item_op=io.cpu().numpy(), need=nd.cpu().numpy(), succ_ptr=sp.cpu().numpy(),
                    succ=sc.cpu().numpy(), rows=np.asarray(c[1]), cols=np.asarray(c[2]), mode=np.asarray(c[8]),
                    phase=phase, n_fwd=ap.n_fwd)
print("saved", ap.flow_items, "items", ap.flow_nops, "ops")
