"""Short config[1] run for ncu captures: warm-up pass + one profiled pass (nb blocks)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200.batched import BatchedSupernodes  # noqa: E402
from paper_1507_05593_b200.problems import batched_supernodes  # noqa: E402

nb = int(sys.argv[1]) if len(sys.argv) > 1 else 64
D, B = batched_supernodes(nb=nb)
bs = BatchedSupernodes(nb, 256, 2048, 58, q=1)
for _ in range(2):
    bs.D.copy_(torch.from_numpy(D))
    bs.B.copy_(torch.from_numpy(B))
    bs.run()
torch.cuda.synchronize()
bs.check_info()
print("ranks", sorted(set(bs.rank.cpu().numpy().tolist())))
