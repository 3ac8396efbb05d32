"""config[1] host-API step time vs pipeline depth (pieces)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1507_05593_b200.batched import BatchedSupernodes  # noqa: E402
from paper_1507_05593_b200.problems import batched_supernodes  # noqa: E402

nb = 512
D, B = batched_supernodes(nb=nb)
bs = BatchedSupernodes(nb, 256, 2048, 58, q=1)
st = bs.pinned_staging()
Dh, Bh = torch.from_numpy(D).pin_memory(), torch.from_numpy(B).pin_memory()
t0 = time.perf_counter()
x = torch.empty_like(Dh, device="cuda")
for _ in range(3):
    x.copy_(Dh, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D alone {Dh.numel()*8*3/(time.perf_counter()-t0)/1e9:.1f} GB/s")
for pieces in (1, 2, 4, 8, 16, 32):
    bs.factor_compress_host(Dh, Bh, pinned=st, pieces=pieces)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        bs.factor_compress_host(Dh, Bh, pinned=st, pieces=pieces)
    print(f"pieces {pieces:3d}: {(time.perf_counter()-t)/5*1e3:.1f} ms/step", flush=True)
