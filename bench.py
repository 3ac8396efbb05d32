"""Benchmark of the B200 rank-structured Cholesky hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config 4]

Default workload: BASELINE config[4] (3D linear elasticity, 64^3 hexahedral elements,
n = 811,200, stored zeros stripped) -- the largest single-GPU config by work and nnz.
A step is one numeric factorization + PCG to relative residual 1e-6; value = its
device-timed seconds (the BASELINE metric "factor+PCG time"), e2e = the one-shot
public API (ordering + symbolic + numeric + PCG, host buffers in and out).  The
reference arm times the full-size oracle factor + PCG on the host (bench_sparse.py).
`--config 2|3|0` selects the other sparse configs, `--config 1` the batched
supernode micro-benchmark (512 independent 256x256 supernodes: POTRF + TRSM + sketch
r=58 + pivoted-QR compression, GFLOP/s).

Multi-GPU: `--gpus N` without a torchrun environment relaunches itself under
`torch.distributed.run` with N processes (one per GPU).  The sparse configs shard by
nested-dissection subtree (distributed.py); config[1] by independent supernodes
(weak scaling, no data-path collective).  Time = max over ranks of the device-timed
region.
"""

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "factor+PCG time to rel-res 1e-6 (s); factor GFLOP/s as % of FP64 TC peak"
FP64_DATASHEET_TFLOPS = 40.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--config", type=int, default=4)
    p.add_argument("--nb", type=int, default=512)
    p.add_argument("--chunk", type=int, default=None, help="supernodes per grouped launch (default: all)")
    p.add_argument("--grid", type=int, default=None, help="grid size override for sparse configs")
    p.add_argument("--cpu-sample", type=int, default=128, help="blocks in the CPU baseline sample")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ref-budget", type=float, default=1560.0,
                   help="reference arm: wall seconds before the remaining sweep is extrapolated")
    return p.parse_args()


# ---------------------------------------------------------------------------
# helpers


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak_tflops(torch):
    """Measured FP64 ceiling on this GPU: cuBLAS DGEMM (torch float64 matmul), best of 5."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = a @ b
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = max(best, 2.0 * n**3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del a, b, c
    return best


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback B200_PROFILING.md"


# ---------------------------------------------------------------------------
# config[1]


def cfg1_inputs(nb):
    from paper_1507_05593_b200.problems import batched_supernodes

    return batched_supernodes(nb=nb)


def cpu_cfg1(D, B, sample, threads):
    """Oracle port of the reference composition on `sample` blocks, `threads` host
    threads (one BLAS thread each).  Returns (GFLOP/s, seconds, flops)."""
    try:
        import threadpoolctl

        limiter = threadpoolctl.threadpool_limits(limits=1)
    except Exception:
        limiter = None
    from oracle import kernels as ok
    from paper_1507_05593_b200.batched import model_flops

    def one(i):
        ok.cfg1_block(D[i], B[i], 58, 1, ok.block_seed(0, 0, i))

    t0 = time.perf_counter()
    if threads > 1:
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, range(sample)))
    else:
        for i in range(sample):
            one(i)
    dt = time.perf_counter() - t0
    if limiter is not None:
        limiter.unregister() if hasattr(limiter, "unregister") else None
    fl = model_flops(sample, 256, 2048, 58, 1)
    return fl / dt / 1e9, dt, fl


def run_reference(args, rank):
    if rank != 0:
        return
    nb = min(args.nb, args.cpu_sample)
    D, B = cfg1_inputs(nb)
    threads = os.cpu_count() or 1
    vals = []
    for _ in range(args.warmup):
        cpu_cfg1(D, B, nb, threads)
    t_all = 0.0
    for _ in range(args.steps):
        g, dt, _ = cpu_cfg1(D, B, nb, threads)
        vals.append(g)
        t_all += dt
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_all / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator of BASELINE config[1])",
        "config": {"workload": "config[1] batched supernode factor+compress", "blocks_per_step": nb,
                   "n": 256, "m": 2048, "sketch_rank": 58, "power_iters": 1},
        "cpu_baseline": {"value": v, "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": f"{nb} of 512 config[1] blocks per step, oracle/kernels.cfg1_block "
                                   f"(scipy LAPACK, 1 BLAS thread per worker)"},
        "e2e": {"value": v, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_cfg1(args, rank, world, torch, dist):
    from paper_1507_05593_b200 import _lib
    from paper_1507_05593_b200 import engine as E
    from paper_1507_05593_b200.batched import BatchedSupernodes, model_flops

    lib = _lib.load()
    nb, n, m, r, q = args.nb, 256, 2048, 58, 1
    D, B = cfg1_inputs(nb)
    bs = BatchedSupernodes(nb, n, m, r, q=q, chunk=args.chunk)
    D0 = torch.from_numpy(D).cuda()
    B0 = torch.from_numpy(B).cuda()

    def step():
        # POTRF is in place: restore D (268 MB); the TRSM reads B0 and writes L_O
        bs.D.copy_(D0)
        bs.run(master=0, B_src=B0)  # includes the device PCG64 sketch generation

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    bs.check_info()
    ranks = bs.rank.cpu().numpy()

    def barrier():
        if dist is not None:
            dist.barrier()

    with ClockSampler(torch.cuda.current_device()) as clk:
        barrier()
        torch.cuda.synchronize()
        lib.rsc_launch_counter(1)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        launches = int(lib.rsc_launch_counter(1))
        barrier()
    t = ev0.elapsed_time(ev1) * 1e-3
    if dist is not None:
        tt = torch.tensor([t], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = float(tt.item())
    flops = model_flops(nb, n, m, r, q)
    value = world * flops * args.steps / t / 1e9

    # roofline of the dominant kernel (the DMMA GEMM of the sketch products), timed
    # live on the launching stream with CUDA events
    LO, G, H, Omd = bs.B, bs.G, bs.H, bs.Om
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    reps = 3
    evs[0].record()
    for _ in range(reps):
        E.gemm_strided_batched(LO, Omd, G, transA=True, splitk=bs.splitk)
        E.gemm_strided_batched(LO, G, H)
    evs[1].record()
    torch.cuda.synchronize()
    gemm_t = evs[0].elapsed_time(evs[1]) * 1e-3 / (2 * reps)
    gemm_flops = 2.0 * nb * m * n * r
    peak = fp64_peak_tflops(torch)

    # end to end through the host API
    e2e = None
    if True:  # every rank measures its own e2e (max over ranks below)
        st = bs.pinned_staging()
        # the caller's host inputs live in page-locked memory (what a serving process
        # would allocate for a stream of factorizations)
        Dh = torch.from_numpy(D).pin_memory()
        Bh = torch.from_numpy(B).pin_memory()
        bs.factor_compress_host(Dh, Bh, pinned=st)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            bs.factor_compress_host(Dh, Bh, pinned=st)
        te = (time.perf_counter() - t0) / args.steps
        if dist is not None:
            tt = torch.tensor([te], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": world * flops / te / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": bs.h2d_bytes(),
               "d2h_bytes_per_step": bs.d2h_bytes(), "seconds_per_step": te}
        # the e2e pass is host-link bound: its roofline is the pinned H2D copy rate of
        # this box (one 1 GiB pinned -> device copy, CUDA events, best of 3)
        del Dh, Bh
        hb = torch.empty(1 << 27, dtype=torch.float64).pin_memory()
        db = torch.empty(1 << 27, dtype=torch.float64, device="cuda")
        best = 0.0
        for _ in range(3):
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            db.copy_(hb, non_blocking=True)
            s1.record()
            torch.cuda.synchronize()
            best = max(best, hb.numel() * 8 / (s0.elapsed_time(s1) * 1e-3) / 1e9)
        del hb, db
        ach = bs.h2d_bytes() / te / 1e9
        e2e["link_roofline"] = {"bound": "pcie_h2d", "achieved": ach, "peak": best, "unit": "GB/s",
                                "frac": ach / best, "peak_source": "pinned 1 GiB H2D copy measured in this run"}

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        sample = min(args.cpu_sample, nb)
        threads = os.cpu_count() or 1
        g, dt, _ = cpu_cfg1(D, B, sample, threads)
        cpu = {"value": g, "unit": "GFLOP/s", "cores": threads, "kind": "port",
               "sample": f"{sample} of {nb} config[1] blocks ({dt:.1f} s wall), oracle/kernels.cfg1_block, "
                         f"1 BLAS thread per worker"}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GFLOP/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": 1e3 * t / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded generator of BASELINE config[1]; reference PCG64 sketches, generated on "
                "the device bit-identically inside every step)",
        "config": {"workload": "config[1] batched supernode factor+compress", "blocks_per_gpu": nb, "n": 256,
                   "m": 2048, "true_rank": 48, "sketch_rank": r, "power_iters": q,
                   "factor_seconds_per_step": t / args.steps,
                   "fp64_tc_frac_of_step": value / world / 1e3 / peak,
                   "kept_ranks": sorted(set(int(x) for x in ranks)),
                   "l2": "inputs larger than L2 (2.4 GB/step); each step re-copies D from a pristine device copy "
                         "(in-place POTRF) and the TRSM reads B from its pristine copy"},
        "roofline": {"bound": "tensor", "achieved": gemm_flops / gemm_t / 1e12, "peak": peak, "unit": "TFLOP/s",
                     "frac": gemm_flops / gemm_t / 1e12 / peak,
                     # dram__bytes_read.sum + dram__bytes_write.sum per launch, mean of the two
                     # sketch-product kernels, from one ncu --set full capture of this pipeline
                     # (profiles/r01/ncu_full_bench_cfg1_gemm.txt: 3.59 GB and 2.68 GB per launch
                     # vs 2.69 GB algorithmic: L_O once + X in + product out)
                     "traffic": 3.131e9, "traffic_unit": "bytes per launch (ncu, not this run)",
                     "kernel": "gemm_grouped_kernel (sketch products L_O^T Omega, L_O G)",
                     "peak_source": "FP64 cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json has no FP64 "
                                    f"entry); datasheet {FP64_DATASHEET_TFLOPS} TF"},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def _relaunch(args):
    """--gpus N > 1 outside torchrun: run this script under torch.distributed.run."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if args.config == 1:
            run_reference(args, rank)
        else:
            from bench_sparse import run_reference_sparse

            run_reference_sparse(args, rank)
        return
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.config == 1:
            run_b200_cfg1(args, rank, world, torch, dist)
        else:
            from bench_sparse import run_sparse

            run_sparse(args, rank, world, torch, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
