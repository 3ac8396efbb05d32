"""Time the device sketch generator on the config[1] workload (512 x 2048 x 58)."""
import time

import numpy as np
import torch

from paper_1507_05593_b200 import engine as E

nb, m, r = 512, 2048, 58
t = time.perf_counter()
seeds, states = E.pcg64_block_states([(0, 0, i) for i in range(nb)])
t_seed = time.perf_counter() - t
Om = torch.empty(nb, m, r, dtype=torch.float64, device="cuda")
ptrs = [Om[i].data_ptr() for i in range(nb)]
ns = np.full(nb, m * r, np.int64)
work = torch.empty(int(E._lib.load().rsc_normal_workspace_bytes(nb, ns.ctypes.data)) // 8 + 1,
                   dtype=torch.float64, device="cuda")
alloc = lambda n: work[:n]
for _ in range(3):
    E.normal_pcg64(states, [m * r] * nb, ptrs, alloc=alloc)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    E.normal_pcg64(states, [m * r] * nb, ptrs, alloc=alloc)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"seed states {t_seed*1e3:.2f} ms; device normals {ms:.3f} ms for {nb*m*r/1e6:.1f} M "
      f"({nb*m*r*8/ms/1e6:.1f} GB/s written)")
t = time.perf_counter()
h = np.empty((8, m, r))
for i in range(8):
    np.random.Generator(np.random.PCG64(int(seeds[i]))).standard_normal((m, r), out=h[i])
print(f"host numpy per sketch {(time.perf_counter()-t)/8*1e3:.2f} ms")
