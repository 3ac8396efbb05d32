"""bench.py --config 0|2|3|4: factor + PCG to rel-res 1e-6 on a sparse config.

value   = device-timed numeric factorization + PCG (symbolic plan prepared, A and b
          resident in HBM) in seconds -- the BASELINE metric "factor+PCG time".  Each
          step drops the previous factor, so from the third step on the numeric sweep
          is the plan's recorded CUDA graph replayed on the matrix (refactorization).
e2e     = the public API end to end: factorize(A, config, coords) (host ordering +
          symbolic + plan upload + numeric) and pcg_solve(A, b) with host b in and
          host x out.
cpu_baseline = the oracle (the reference algorithm restated on scipy/LAPACK) on a
          bounded sample -- the same generator at a smaller grid -- with the time
          extrapolated to the full config by the ratio of modeled work.
"""

import json
import os
import time

import numpy as np

KNOBS = dict(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=256, power_iters=1, seed=0,
             interior_blocks=True, max_restarts=10)
METRIC = "factor+PCG time to rel-res 1e-6 (s); factor GFLOP/s as % of FP64 TC peak"
GRID = {0: 128, 2: 64, 3: 96, 4: 65}
SAMPLE_GRID = {0: 128, 2: 32, 3: 32, 4: 21}
NAMES = {0: "config[0] 2D Laplacian 128^2", 2: "config[2] 3D Laplacian 64^3",
         3: "config[3] 3D lognormal FV diffusion 96^3", 4: "config[4] 3D elasticity 64^3 elements (zeros stripped)"}


def _problem(cfg, grid):
    from paper_1507_05593_b200.problems import diffusion_fv_3d, elasticity_3d, laplacian_2d, laplacian_3d

    if cfg == 0:
        return laplacian_2d(grid)
    if cfg == 2:
        return laplacian_3d(grid)
    if cfg == 3:
        return diffusion_fv_3d(grid)
    return elasticity_3d(grid, strip_zeros=True)


def cpu_sample(cfg, grid):
    """Oracle factor+PCG on the sample grid; returns (seconds, n, iterations)."""
    try:
        import threadpoolctl

        # one BLAS thread: the reference's default (cli.py:23-32,48) and, for its many
        # small LAPACK calls, faster than a threaded BLAS
        threadpoolctl.threadpool_limits(limits=1)
    except Exception:
        pass
    from oracle import numeric as on

    A, coords = _problem(cfg, grid)
    b = np.random.default_rng(0).standard_normal(A.n)
    t0 = time.perf_counter()
    F = on.factorize(A, on.Config(**KNOBS), coords=coords)
    x, rep = on.pcg(A, b, F, tol=1e-6)
    return time.perf_counter() - t0, A.n, rep.iterations


def run_sparse(args, rank, world, torch, dist):
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E
    from paper_1507_05593_b200.distributed import factorize_distributed
    from paper_1507_05593_b200.factor import SolverConfig, factorize, prepare
    from paper_1507_05593_b200.pcg import pcg_solve, pcg_solve_device

    import bench as B

    cfg = args.config
    lib = _lib.load()
    A, coords = _problem(cfg, args.grid or GRID[cfg])
    n = A.n
    b = np.random.default_rng(0).standard_normal(n)
    conf = SolverConfig(**KNOBS)
    t_prep0 = time.perf_counter()
    prep = prepare(A, conf, coords)
    t_prep = time.perf_counter() - t_prep0
    bd = E.to_dev(b)
    A.device_csr()

    # N > 1: the factorization is sharded by nested-dissection subtree (each rank
    # sweeps its subtrees, the source panels are all-gathered, the top separators
    # run on every rank, the factor blocks are all-gathered); PCG then runs on
    # every rank with the whole factor (a replicated solve)
    fact = factorize_distributed if world > 1 else factorize

    def step():
        F = fact(A, prepared=prep)
        x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
        return F, rep

    F = None
    for _ in range(max(args.warmup, 1)):
        F = None  # a refactorization loop drops the previous factor (graph replay reuses its memory)
        F, rep = step()
    torch.cuda.synchronize()
    with B.ClockSampler(torch.cuda.current_device()) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        lib.rsc_launch_counter(1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tf = []
        ev0.record()
        for _ in range(args.steps):
            F = None
            F, rep = step()
            tf.append(F.stats.phase_times["numeric"])
        ev1.record()
        torch.cuda.synchronize()
        launches = int(lib.rsc_launch_counter(1))
        if dist is not None:
            dist.barrier()
    t = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    st = F.stats
    work = st.model_gflop
    graph_nodes = st.gpu_launches if getattr(F, "_entry", None) is not None else 0
    # dominant kernel: the grouped DMMA GEMM.  Its flops come from the launch
    # descriptors of an ordinary pass; its device time from CUPTI kernel records
    # (torch.profiler) of one timed-path step (the replayed graph) -- per-launch CUDA
    # events would also count the host issue gaps between launches
    import paper_1507_05593_b200.factor as FM
    from torch.profiler import ProfilerActivity, profile

    F = None
    g0, FM.GRAPH_REFACTOR = FM.GRAPH_REFACTOR, False
    E.PROFILE = E.KernelProfile()
    step()  # (N > 1: this rank's subtrees + the top separators)
    gemm_flops = E.PROFILE.summary()["flops"]
    E.PROFILE = None
    FM.GRAPH_REFACTOR = g0
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as kp:
        F = None
        F, _ = step()
        torch.cuda.synchronize()
    kev = [e for e in kp.events() if e.device_type.name == "CUDA"]
    gemm_s = sum(e.device_time for e in kev if "gemm_grouped_kernel" in e.name) / 1e6
    busy_s = sum(e.device_time for e in kev) / 1e6
    prof = {"flops": gemm_flops, "seconds": gemm_s}
    peak = B.fp64_peak_tflops(torch)
    # HBM-bound kernels of the PCG: the preconditioner apply (its replayed graph) and
    # the CSR SpMV, CUDA events around 20 back-to-back calls each.  Algorithmic bytes
    # (SURVEY §8(d)): apply = 16 B per stored factor scalar (read once in each sweep)
    # + 48 B per row of vectors; SpMV = 12 B per stored nonzero + 4(n+1) + 16n.
    hbm, hbm_src = B.hbm_peak()
    zd, yd = torch.empty_like(bd), torch.empty_like(bd)
    S = A.device_csr()

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3 / reps

    t_ap = timed(lambda: F.apply_device(bd, zd))
    t_sp = timed(lambda: E.spmv(S, bd, yd))
    b_ap = 16.0 * st.stored_scalars + 48.0 * n
    b_sp = 12.0 * S.nnz + 4.0 * (n + 1) + 16.0 * n
    hbm_line = {
        "bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": hbm_src,
        "apply": {"seconds": t_ap, "bytes": b_ap, "achieved": b_ap / t_ap / 1e9, "frac": b_ap / t_ap / 1e9 / hbm},
        "spmv": {"seconds": t_sp, "bytes": b_sp, "achieved": b_sp / t_sp / 1e9, "frac": b_sp / t_sp / 1e9 / hbm,
                 "l2_resident": bool(b_sp < 100e6)},
    }
    # end to end through the public API (host A, coords, b in; host x out)
    t0 = time.perf_counter()
    for _ in range(max(1, min(args.steps, 2))):
        F2 = fact(A, conf, coords=coords)
        x, rep2 = pcg_solve(A, b, preconditioner=F2, tol=1e-6)
    te = (time.perf_counter() - t0) / max(1, min(args.steps, 2))
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        sg = SAMPLE_GRID[cfg]
        ts, ns, its = cpu_sample(cfg, sg)
        # modeled-work ratio from the GPU work counter on both sizes
        if sg != (args.grid or GRID[cfg]):
            As, cs = _problem(cfg, sg)
            Fs = factorize(As, conf, coords=cs)
            ratio = work / max(Fs.stats.model_gflop, 1e-12)
        else:
            ratio = 1.0
        cpu = {"value": ts * ratio, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"oracle factor+PCG on grid {sg} (n={ns}, {its} PCG its) took {ts:.1f} s; scaled by the "
                         f"modeled-work ratio {ratio:.1f} to the full config"}
    line = {
        "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 1), "ms_per_step": 1e3 * t, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator; reference PCG64 sketches)",
        "config": {"workload": NAMES[cfg], "n": n,
                   "parallelism": "single GPU" if world == 1 else
                   f"{world} ranks: ND subtrees sharded, top separators and PCG replicated", "nnz_lower": A.nnz_lower, "knobs": KNOBS, "tol": 1e-6,
                   "pcg_iterations": rep.iterations, "final_relres": rep.relative_residual,
                   "numeric_factor_s": float(np.median(tf)), "symbolic_prepare_s": t_prep,
                   "modeled_gflop": work, "factor_gflops": work / float(np.median(tf)),
                   "restarts": st.restarts, "compressed_offdiag": st.compressed_offdiag,
                   "compressed_diag": st.compressed_diag, "stored_scalars": st.stored_scalars},
        "roofline": {"bound": "tensor", "achieved": prof["flops"] / max(prof["seconds"], 1e-12) / 1e12,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": prof["flops"] / max(prof["seconds"], 1e-12) / 1e12 / peak, "traffic": None,
                     "kernel": "gemm_grouped_kernel (all grouped GEMM launches of one factor+PCG)",
                     "kernel_seconds": prof["seconds"], "kernel_share_of_step": prof["seconds"] / t,
                     "all_kernels_seconds": busy_s,
                     "peak_source": "FP64 cuBLAS DGEMM 8192^3 measured in this run"},
        "hbm_roofline": hbm_line,
        "cpu_baseline": cpu,
        "e2e": {"value": te, "unit": "s", "h2d_bytes_per_step": int(8 * (A.nnz_lower * 2 + n)),
                "d2h_bytes_per_step": int(8 * n)},
        "gpu_launches": launches // args.steps + graph_nodes,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
