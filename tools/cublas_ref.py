"""cuBLAS (torch fp64) on config[1]'s exact batched shapes, for calibration only."""
import torch

nb, n, m, r = 512, 256, 2048, 58
LO = torch.randn(nb, m, n, dtype=torch.float64, device="cuda")
Om = torch.randn(nb, m, r, dtype=torch.float64, device="cuda")
G = torch.randn(nb, n, r, dtype=torch.float64, device="cuda")
L = torch.linalg.cholesky(torch.eye(n, dtype=torch.float64, device="cuda").expand(nb, n, n) * 4 +
                          0.01 * torch.ones(n, n, dtype=torch.float64, device="cuda"))


def t(fn, flops, name, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    print(f"{name:28s} {ms:7.3f} ms  {flops / ms / 1e9:6.2f} TF/s")


t(lambda: torch.bmm(LO.transpose(1, 2), Om), 2.0 * nb * m * n * r, "cuBLAS L_O^T Om (bmm)")
t(lambda: torch.bmm(LO, G), 2.0 * nb * m * n * r, "cuBLAS L_O G (bmm)")
G64 = torch.randn(nb, n, 64, dtype=torch.float64, device="cuda")
t(lambda: torch.bmm(LO, G64), 2.0 * nb * m * n * 64, "cuBLAS L_O G64 (bmm, N=64)")
t(lambda: torch.linalg.solve_triangular(L, LO.transpose(1, 2), upper=False), 1.0 * nb * m * n * n,
  "cuBLAS TRSM L^-1 B^T", reps=2)
A = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
t(lambda: A @ A, 2.0 * 8192**3, "cuBLAS DGEMM 8192^3", reps=3)
