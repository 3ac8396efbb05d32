"""bench.py --config 0|2|3|4 (default 4): factor + PCG to rel-res 1e-6 on a sparse config.

B200 arm (`run_sparse`):
  value   = device-timed numeric factorization + PCG (symbolic plan prepared, A and b
            resident in HBM) in seconds -- the BASELINE metric "factor+PCG time".  Each
            step drops the previous factor, so from the third step on the numeric sweep
            is the plan's recorded CUDA graph replayed on the matrix (refactorization).
  e2e     = the public API end to end, one-shot: factorize(A, config, coords) (host
            ordering + symbolic + plan upload + numeric) and pcg_solve(A, b) with host
            b in and host x out.
  config.modeled_gflop = the reference algorithm's work census (census.py, SURVEY
            §8(d)) at the kept ranks; factor_gflops = census / numeric seconds.
  cpu_baseline = the oracle (the reference algorithm restated on scipy/LAPACK, one
            BLAS thread) on a bounded sample: the same generator at a smaller grid,
            scaled by the census ratio full / sample.

Reference arm (`run_reference_sparse`, `--impl reference`): the oracle factor + PCG of
the FULL-SIZE config, once, single-threaded BLAS (the reference's own default,
cli.py:23-32,48; threaded OpenBLAS is ~25x slower on its many small calls).  The
unit sweep is cut into K contiguous slices (the "steps"); value = the whole run.
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


def _one_blas_thread():
    """Pin numpy's and scipy's OpenBLAS to one thread (both must be loaded first);
    returns the limiter, which must stay referenced."""
    import scipy.linalg  # noqa: F401  (loads scipy's OpenBLAS)
    import threadpoolctl

    return threadpoolctl.threadpool_limits(limits=1, user_api="blas")


def _census(sym, ranks, alpha_d=None, per_unit=None):
    from paper_1507_05593_b200.census import census
    from paper_1507_05593_b200.factor import SolverConfig

    return census(sym, SolverConfig(**KNOBS), ranks, alpha_d, per_unit)


def cpu_sample(cfg, grid):
    """Oracle factor+PCG on the sample grid: (seconds, n, iterations, census GF)."""
    lim = _one_blas_thread()  # noqa: F841
    from oracle import numeric as on
    from paper_1507_05593_b200.symbolic import analyze

    A, coords = _problem(cfg, grid)
    b = np.random.default_rng(0).standard_normal(A.n)
    t0 = time.perf_counter()
    c = on.Config(**KNOBS)
    plan = analyze(A, c.tau_o, c.tau_d, c.interior_blocks, coords=coords)
    F = on.factorize(A, c, coords=coords, plan=plan)
    x, rep = on.pcg(A, b, F, tol=1e-6)
    dt = time.perf_counter() - t0
    gf = sum(_census(plan, F.ranks, F.stats["alpha_d_final"]).values()) / 1e9
    return dt, A.n, rep.iterations, gf


class _Budget(Exception):
    pass


def run_reference_sparse(args, rank):
    """The oracle on the full-size config (see module docstring)."""
    if rank != 0:
        return
    lim = _one_blas_thread()  # noqa: F841
    from oracle import numeric as on
    from paper_1507_05593_b200.symbolic import analyze

    cfg = args.config
    K = max(int(args.steps), 1)
    c = on.Config(**KNOBS)
    for _ in range(args.warmup):  # warm imports / BLAS on a small instance
        Aw, cw = _problem(cfg, 8 if cfg != 0 else 16)
        pw = analyze(Aw, c.tau_o, c.tau_d, c.interior_blocks, coords=cw)
        on.pcg(Aw, np.ones(Aw.n), on.factorize(Aw, c, coords=cw, plan=pw), tol=1e-6)
    A, coords = _problem(cfg, args.grid or GRID[cfg])
    b = np.random.default_rng(0).standard_normal(A.n)
    t0 = time.perf_counter()
    plan = analyze(A, c.tau_o, c.tau_d, c.interior_blocks, coords=coords)
    t_sym = time.perf_counter() - t0
    stamps = []
    budget = float(args.ref_budget)

    def hook(u, kind, payload):
        now = time.perf_counter()
        stamps.append(now)
        if now - t0 > budget:
            raise _Budget()

    nunits = len(plan.units)
    extrap = None
    t1 = time.perf_counter()
    try:
        F = on.factorize(A, c, coords=coords, plan=plan, on_unit=hook)
        t_num = time.perf_counter() - t1
        t2 = time.perf_counter()
        x, rep = on.pcg(A, b, F, tol=1e-6)
        t_pcg = time.perf_counter() - t2
        its = rep.iterations
    except _Budget:
        # over budget: the remaining units are extrapolated at the rate (s / census
        # flop) of the most recent quarter of the work done; PCG at the measured
        # 4% of the numeric time (config[4] on the reference: 51.5 / 1249.6 s)
        done = len(stamps) - 1
        t_num_done = stamps[-1] - t1
        from paper_1507_05593_b200.census import census as _census_fn

        cum = []  # kept ranks past the cut are unknown: sketch widths (upper bound)
        _census_fn(plan, c, None, None, cum)
        cum = np.asarray(cum)
        f_done = cum[done - 1] if done > 0 else 0.0
        q = int(done * 0.75)
        rate = (stamps[done] - stamps[q]) / max(cum[done - 1] - (cum[q - 1] if q > 0 else 0.0), 1.0)
        t_num = t_num_done + rate * (cum[-1] - f_done)
        t_pcg = 0.04 * t_num
        its = None
        extrap = {"units_done": done, "units": nunits, "measured_numeric_s": t_num_done,
                  "rule": "remaining units at the s/flop of the last quarter of done work; PCG = 4% of numeric"}
    total = t_sym + t_num + t_pcg
    # K slices of the unit sweep (equal unit counts); the last one carries PCG
    cut = np.linspace(0, len(stamps) - 1, K + 1).astype(int) if len(stamps) > 1 else np.zeros(K + 1, int)
    sl = [float(stamps[cut[i + 1]] - stamps[cut[i]]) if len(stamps) > 1 else 0.0 for i in range(K)]
    sl[-1] += max(0.0, (t1 + t_num) - (stamps[-1] if stamps else t1)) + t_pcg
    sl[0] += t_sym
    line = {
        "impl": "reference", "metric": METRIC, "value": total, "unit": "s", "n_gpus": args.gpus,
        "steps": K, "warmup": args.warmup, "ms_per_step": 1e3 * total / K, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator; reference PCG64 sketches)",
        "config": {"workload": NAMES[cfg], "n": A.n, "nnz_lower": A.nnz_lower, "knobs": KNOBS, "tol": 1e-6,
                   "ordering_symbolic_s": t_sym, "numeric_s": t_num, "pcg_s": t_pcg, "pcg_iterations": its,
                   "slices_s": sl, "extrapolated": extrap},
        "cpu_baseline": {"value": total, "unit": "s", "cores": 1, "kind": "port",
                         "sample": f"the full-size {NAMES[cfg]} factor + PCG, once, one BLAS thread (oracle/ "
                                   f"restatement of the reference; ordering + symbolic by the package's host code, "
                                   f"the same plan); the {nunits}-unit sweep cut into {K} slices = steps"},
        "e2e": {"value": total, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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

    # N > 1: the factorization is sharded by nested-dissection subtree (distributed.py)
    fact = factorize_distributed if world > 1 else factorize

    def step():
        F = fact(A, prepared=prep)
        x, rep = pcg_solve_device(A, bd, preconditioner=F, tol=1e-6)
        return F, rep

    F = None
    for _ in range(max(args.warmup, 3)):
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
        # RSC_BENCH_PROFILE_RANGE=1: cudaProfilerStart/Stop around the timed steps, so an
        # `ncu --profile-from-start off` launch list holds exactly the timed region
        prof_range = os.environ.get("RSC_BENCH_PROFILE_RANGE") == "1"
        if prof_range:
            torch.cuda.profiler.start()
        ev0.record()
        for _ in range(args.steps):
            F = None
            F, rep = step()
            tf.append(F.stats.phase_times["numeric"])
        ev1.record()
        torch.cuda.synchronize()
        if prof_range:
            torch.cuda.profiler.stop()
        launches = int(lib.rsc_launch_counter(1))
        if dist is not None:
            dist.barrier()
    t = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    st = F.stats
    cen = _census(prep[0], F.ranks, st.alpha_d_final)
    work = sum(cen.values()) / 1e9
    graph_nodes = st.gpu_launches if getattr(F, "_entry", None) is not None else 0
    # dominant kernel: the grouped DMMA GEMM.  Its flops come from the launch
    # descriptors of an ordinary pass; its device time from CUPTI kernel records
    # (torch.profiler) of one timed-path step (the replayed graph)
    import paper_1507_05593_b200.factor as FM
    from torch.profiler import ProfilerActivity, profile

    F = None
    g0, FM.GRAPH_REFACTOR = FM.GRAPH_REFACTOR, False
    E.PROFILE = E.KernelProfile()
    step()
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
    by_kernel = {}
    for e in kev:
        nm = e.name.replace("void ", "").replace("(anonymous namespace)::", "").split("<")[0].split("(")[0]
        by_kernel[nm] = by_kernel.get(nm, 0.0) + e.device_time / 1e6
    top = sorted(by_kernel.items(), key=lambda x: -x[1])[:8]
    prof = {"flops": gemm_flops, "seconds": gemm_s}
    peak = B.fp64_peak_tflops(torch)
    # HBM-bound kernels of the PCG: the preconditioner apply and the CSR SpMV, CUDA
    # events around 20 back-to-back calls each.  Algorithmic bytes:
    # apply = 16 B per stored factor scalar (read once in each sweep) + 48 B per row of
    # vectors; SpMV = 12 B per stored nonzero + 4(n+1) + 16n.
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
    # end to end through the public API, one-shot (host A, coords, b in; host x out)
    reps = max(1, min(args.steps, 2))
    t0 = time.perf_counter()
    for _ in range(reps):
        F2 = fact(A, conf, coords=coords)
        x, rep2 = pcg_solve(A, b, preconditioner=F2, tol=1e-6)
        del F2
    te = (time.perf_counter() - t0) / reps
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        sg = SAMPLE_GRID[cfg]
        ts, ns, its, gfs = cpu_sample(cfg, sg)
        ratio = work / gfs if sg != (args.grid or GRID[cfg]) else 1.0
        cpu = {"value": ts * ratio, "unit": "s", "cores": 1, "kind": "port",
               "sample": f"oracle factor+PCG on grid {sg} (n={ns}, {its} PCG its, {gfs:.2f} census GFLOP) took "
                         f"{ts:.1f} s on one BLAS thread; scaled by the census ratio {ratio:.1f} to the full config "
                         f"(bench.py --impl reference times the full-size run itself)"}
    line = {
        "metric": METRIC, "value": t, "unit": "s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": 1e3 * t, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator; reference PCG64 sketches)",
        "config": {"workload": NAMES[cfg], "n": n,
                   "parallelism": "single GPU" if world == 1 else
                   f"{world} ranks: ND subtrees sharded, top separators split by source owner",
                   "nnz_lower": A.nnz_lower, "knobs": KNOBS, "tol": 1e-6,
                   "l2": "inputs (A blocks, factor: GBs) far larger than the 126 MB L2",
                   "pcg_iterations": rep.iterations, "final_relres": rep.relative_residual,
                   "numeric_factor_s": float(np.median(tf)), "symbolic_prepare_s": t_prep,
                   "modeled_gflop": work, "census_gflop": {k: v / 1e9 for k, v in cen.items()},
                   "factor_gflops": work / float(np.median(tf)),
                   "factor_frac_of_fp64_peak": work / float(np.median(tf)) / 1e3 / peak,
                   "restarts": st.restarts, "compressed_offdiag": st.compressed_offdiag,
                   "compressed_diag": st.compressed_diag, "stored_scalars": st.stored_scalars,
                   "kernel_time_top": {k: v for k, v in top}},
        "roofline": {"bound": "tensor", "achieved": prof["flops"] / max(prof["seconds"], 1e-12) / 1e12,
                     "peak": peak, "unit": "TFLOP/s",
                     "frac": prof["flops"] / max(prof["seconds"], 1e-12) / 1e12 / peak,
                     # dram__bytes_read.sum + dram__bytes_write.sum of every grouped-GEMM
                     # launch of one config[4] numeric pass (ncu, profiles/r02/
                     # ncu_gemm_dram_cfg4.txt): 241.4 GB over 7905 launches
                     "traffic": 241.4e9 / 7905 if cfg == 4 else None,
                     "traffic_unit": "bytes per launch (mean over one numeric pass, ncu; not this run)",
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
