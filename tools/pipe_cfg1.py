"""config[1] step time (CUDA events, 20 steps) for several (chunk, pipeline) schedules."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200.batched import BatchedSupernodes  # noqa: E402
from paper_1507_05593_b200.problems import batched_supernodes  # noqa: E402

nb = 512
D, B = batched_supernodes(nb=nb)
D0 = torch.from_numpy(D).cuda()
B0 = torch.from_numpy(B).cuda()
for spec in sys.argv[1:] or ["512x1", "256x2", "128x2", "128x3", "64x2"]:
    chunk, pipe = (int(x) for x in spec.split("x"))
    bs = BatchedSupernodes(nb, 256, 2048, 58, q=1, chunk=chunk, pipeline=pipe)

    def step():
        bs.D.copy_(D0)
        bs.run(master=0, B_src=B0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        step()
    e1.record()
    torch.cuda.synchronize()
    bs.check_info()
    ranks = set(bs.rank.cpu().numpy().tolist())
    print(f"chunk {chunk:4d} pipeline {pipe}: {e0.elapsed_time(e1) / 20:.3f} ms/step ranks {ranks}", flush=True)
    del bs
    torch.cuda.empty_cache()
