"""Per-stage device time of one config[1] step (CUDA events around each stage of
BatchedSupernodes.run, repeated, median), plus the stage's algorithmic TF/s."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200 import engine as E  # noqa: E402
from paper_1507_05593_b200.batched import BatchedSupernodes  # noqa: E402
from paper_1507_05593_b200.problems import batched_supernodes  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n, m, r, q = 256, 2048, 58, 1
D, B = batched_supernodes(nb=nb)
bs = BatchedSupernodes(nb, n, m, r, q=q)
D0 = torch.from_numpy(D).cuda()
B0 = torch.from_numpy(B).cuda()
states = bs.sketch_states(0)
P = BatchedSupernodes._ptrs
Dp, Ip, Bp, Sp, Gp, Up = (P(T, 0, nb) for T in (bs.D, bs.Dinv, bs.B, B0, bs.G, bs.U))

stages = [
    ("rng", lambda: bs.generate_sketches(0, states=states), 0.0),
    ("potrf", lambda: E.potrf_batched(Dp, [n] * nb, [n] * nb, Ip, bs.info), nb * n**3 / 3),
    ("trsm", lambda: E.trsm_right(Dp, [n] * nb, [n] * nb, Ip, Sp, Bp, [m] * nb, [n] * nb), nb * m * n * n),
    ("LOt_Om", lambda: E.gemm_strided_batched(bs.B, bs.Om, bs.G, transA=True, splitk=bs.splitk), nb * 2.0 * m * n * r),
    ("LO_G", lambda: E.gemm_strided_batched(bs.B, bs.G, bs.H), nb * 2.0 * m * n * r),
    ("LOt_H", lambda: E.gemm_strided_batched(bs.B, bs.H, bs.G, transA=True, splitk=bs.splitk), nb * 2.0 * m * n * r),
    ("qrcp", lambda: E.qrcp_batched(Gp, [n] * nb, [r] * nb, [r] * nb, Up, [r] * nb, bs.rank), nb * 4.0 * n * r * r),
    ("V", lambda: E.gemm_strided_batched(bs.B, bs.U, bs.V), nb * 2.0 * m * n * r),
]
times = {k: [] for k, _, _ in stages}
for it in range(reps + 2):
    bs.D.copy_(D0)
    torch.cuda.synchronize()
    for name, fn, _ in stages:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        if it >= 2:
            times[name].append(e0.elapsed_time(e1))
tot = 0.0
for name, _, fl in stages:
    t = statistics.median(times[name])
    tot += t
    print(f"{name:8s} {t:8.3f} ms  {fl / t / 1e9 if fl else 0:7.2f} TF/s")
print(f"total    {tot:8.3f} ms  {sum(f for _, _, f in stages) / tot / 1e9:7.2f} TF/s")
