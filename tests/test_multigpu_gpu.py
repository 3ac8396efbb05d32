"""The sharded (multi-rank) factorization on the GPU: two ranks share cuda:0 over
gloo (host-staged collectives, so no kernel ever waits on another rank) and must
reproduce the single-GPU factor -- identical kept ranks, stored scalars and
counters, the same preconditioner application and PCG solution."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_factorization_matches_single_gpu(cuda, world):
    env = dict(os.environ, RSC_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "tools", "dist_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-4000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["world"] == world
    for name, c in out["cases"].items():
        assert c["top_units"] >= 1 and c["owned_units"] >= 1, (name, c)
        assert c["ranks_equal"] and c["stored_equal"] and c["counters_equal"], (name, c)
        g1, gd = c["model_gflop"]
        assert abs(g1 - gd) <= 1e-9 * g1, (name, c)
        # compressed blocks: the same band as two single-GPU runs (FP64 atomic sums)
        assert c["apply_relerr"] < max(1e-8, 10 * c["apply_relerr_self"]), (name, c)
        # PCG stops at relres 1e-6, so x inherits the preconditioner's run-to-run noise
        # amplified by the solve: the same band rule as the apply (sharded vs single
        # GPU measured 1.0-1.15e-8 on l3d20 in some runs, below 1e-8 in others)
        assert abs(c["pcg_its"][0] - c["pcg_its"][1]) <= 1, (name, c)
        assert c["x_relerr"] < max(1e-8, 10 * c["x_relerr_self"]), (name, c)
