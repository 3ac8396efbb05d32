"""Level-batched supernode factor + compression (the config[1] kernel pipeline).

For a batch of independent supernodes (diagonal block D_i, off-diagonal block B_i)
this runs, entirely on the device and batched across supernodes:

    Omega_i ~ PCG64(_block_seed(master, 0, i)) normals   rsc_normal_pcg64  (kernels.py:85-92)
    L_D = chol(D)                       rsc_potrf_batched      (factor.py:614)
    L_O = B L_D^{-T}                    rsc_trsm_batched        (factor.py:414,633)
    G   = L_O^T Omega                   grouped DMMA GEMM       (kernels.py:107)
    q x { H = L_O G ; G = L_O^T H }     grouped DMMA GEMM       (kernels.py:108-110)
    U   = orth(G)  (pivoted QR+cutoff)  rsc_qrcp_batched        (kernels.py:111)
    V   = L_O U                         grouped DMMA GEMM       (kernels.py:112)

which is the reference composition dense_cholesky -> tri_solve -> low_rank_approx
for every block.  Omega_i are the reference's own PCG64 sketches
(seed `_block_seed(seed, 0, i)`), generated on the device bit-identically to numpy
(rng.cu), so no sketch crosses PCIe.

The whole batch goes through each stage in one grouped launch (the products
stream L_O from HBM at ~8 flop/byte, above the FP64 ridge); `chunk` can cut the
batch to trade launch width for L2 residency.
"""

import concurrent.futures as cf
import math

import numpy as np
import torch

from . import engine as E
from .errors import IndefiniteError

FLOPS_NOTE = "POTRF n^3/3 + TRSM m n^2 + (2+2q) GEMMs 2 m n r + QRCP 4 n r^2"


def block_seed(master, *tags):
    """Seed of one sketch: SeedSequence((master,)+tags) -> first uint64 word
    (reference factor.py:324-326)."""
    ss = np.random.SeedSequence((int(master),) + tuple(int(t) for t in tags))
    return int(ss.generate_state(1, np.uint64)[0])


def sketch(m, r, seed):
    return np.random.Generator(np.random.PCG64(seed)).standard_normal((m, r))


def make_sketches(nb, m, r, master=0, threads=8, out=None):
    """Host PCG64 sketches for blocks 0..nb-1 (numpy releases the GIL while filling,
    so a thread pool scales across blocks)."""
    if out is None:
        out = np.empty((nb, m, r))
    seeds = [block_seed(master, 0, i) for i in range(nb)]

    def fill(i):
        out[i] = sketch(m, r, seeds[i])

    if threads <= 1:
        for i in range(nb):
            fill(i)
    else:
        with cf.ThreadPoolExecutor(threads) as ex:
            list(ex.map(fill, range(nb)))
    return out


def model_flops(nb, n, m, r, q):
    """Algorithmic FLOPs of the reference composition (SURVEY §8(d) work model)."""
    per = n**3 / 3 + m * n * n + (2 + 2 * q) * 2.0 * m * n * r + 4.0 * n * r * r
    return nb * per


class BatchedSupernodes:
    """Device workspace for a batch of `nb` supernodes of shape (n, m) with sketch width r."""

    def __init__(self, nb, n, m, r, q=1, chunk=None, splitk=None, pipeline=1):
        self.nb, self.n, self.m, self.r, self.q = nb, n, m, r, q
        self.chunk = nb if chunk is None else max(1, min(chunk, nb))
        self.pipeline = pipeline
        self._streams_side = None
        # split the tall K = m of L_O^T X so a launch has >= ~4 CTAs per SM
        self.splitk = splitk if splitk is not None else max(1, min(m // 256, 16))
        self.D = E.empty(nb, n, n)
        self.B = E.empty(nb, m, n)
        self.Om = E.empty(nb, m, r)
        self.Dinv = E.empty(nb, n, 64)
        self.G = E.empty(nb, n, r)
        self.H = E.empty(nb, m, r)
        self.U = E.empty(nb, n, r)
        self.V = E.empty(nb, m, r)
        self.info = E.zeros(nb, dtype=E.I32)
        self.rank = E.zeros(nb, dtype=E.I32)
        self._qr_work = []
        self._rng_n = np.full(nb, m * r, dtype=np.int64)
        lib = E.require_cuda()
        self._rng_work = E.empty(int(lib.rsc_normal_workspace_bytes(nb, self._rng_n.ctypes.data)) // 8 + 1)
        self._rng_ptrs = np.asarray([self.Om[i].data_ptr() for i in range(nb)], dtype=np.uint64)
        self._streams = None

    def sketch_states(self, master):
        """PCG64 states of the blocks' sketches (reference seeding, host integer work)."""
        keys = np.zeros((self.nb, 3), dtype=np.uint64)
        keys[:, 0] = master
        keys[:, 2] = np.arange(self.nb, dtype=np.uint64)
        return E.pcg64_block_states(keys)[1]

    def generate_sketches(self, master=0, lo=0, hi=None, states=None):
        """Omega_i = PCG64(_block_seed(master, 0, i)).standard_normal((m, r)) on the
        device, for blocks lo..hi-1."""
        hi = self.nb if hi is None else hi
        states = self.sketch_states(master) if states is None else states
        w = self._rng_work
        E.normal_pcg64(states[lo:hi], self._rng_n[lo:hi], self._rng_ptrs[lo:hi], alloc=lambda k: w[:k])

    def run(self, master=0, sketches=True, lo=0, hi=None, states=None, B_src=None):
        """Factor + compress blocks lo..hi-1 (inputs in self.D / self.B, or the
        off-diagonal blocks read from the device tensor B_src and L_O written to
        self.B).  The sketches are generated on the device unless `sketches` is False
        (then self.Om is used as the caller left it).

        Stream schedule: the sketch generator (integer-ALU bound) runs on a side
        stream under the latency-bound POTRF and the TRSM, and joins before the first
        sketch product.  With `pipeline` > 1 the chunks of the batch rotate over that
        many streams, so one chunk's latency-bound stages (POTRF, QRCP) overlap another
        chunk's DMMA-bound TRSM and products."""
        hi = self.nb if hi is None else hi
        main = torch.cuda.current_stream()
        rng_done = None
        if sketches:
            side = self._side_streams(1)[0]
            side.wait_stream(main)
            with torch.cuda.stream(side):
                self.generate_sketches(master, lo, hi, states)
            rng_done = torch.cuda.Event()
            rng_done.record(side)
        chunks = list(range(lo, hi, self.chunk))
        self._qr_work = []  # workspaces stay alive until the next run
        pipes = [main] if self.pipeline <= 1 or len(chunks) <= 1 else self._side_streams(1 + self.pipeline)[1:]
        for p in pipes:
            if p is not main:
                p.wait_stream(main)
        for ci, c0 in enumerate(chunks):
            with torch.cuda.stream(pipes[ci % len(pipes)]):
                self._run_chunk(c0, min(hi, c0 + self.chunk), rng_done, B_src)
        for p in pipes:
            if p is not main:
                main.wait_stream(p)
        if rng_done is not None:
            main.wait_event(rng_done)

    def _side_streams(self, k):
        if self._streams_side is None or len(self._streams_side) < k:
            self._streams_side = [torch.cuda.Stream() for _ in range(k)]
        return self._streams_side

    def _run_chunk(self, c0, c1, rng_done, B_src):
        n, m, r, q = self.n, self.m, self.r, self.q
        cnt = c1 - c0
        Dp, Ip, Bp = self._ptrs(self.D, c0, c1), self._ptrs(self.Dinv, c0, c1), self._ptrs(self.B, c0, c1)
        E.potrf_batched(Dp, [n] * cnt, [n] * cnt, Ip, self.info[c0:c1])
        Sp = None if B_src is None else self._ptrs(B_src, c0, c1)
        E.trsm_right(Dp, [n] * cnt, [n] * cnt, Ip, Sp, Bp, [m] * cnt, [n] * cnt)
        if rng_done is not None:
            torch.cuda.current_stream().wait_event(rng_done)
        LO, G, H, Om = self.B[c0:c1], self.G[c0:c1], self.H[c0:c1], self.Om[c0:c1]
        E.gemm_strided_batched(LO, Om, G, transA=True, splitk=self.splitk)
        for _ in range(q):
            E.gemm_strided_batched(LO, G, H)
            E.gemm_strided_batched(LO, H, G, transA=True, splitk=self.splitk)
        self._qr_work.append(E.qrcp_batched(self._ptrs(self.G, c0, c1), [n] * cnt, [r] * cnt,
                                            [r] * cnt, self._ptrs(self.U, c0, c1), [r] * cnt,
                                            self.rank[c0:c1]))
        E.gemm_strided_batched(LO, self.U[c0:c1], self.V[c0:c1])

    @staticmethod
    def _ptrs(T, lo, hi):
        """Device addresses of T[lo:hi] (3-D contiguous), computed arithmetically (no
        per-block tensor indexing on the host)."""
        step = T.stride(0) * T.element_size()
        return np.uint64(T.data_ptr()) + np.arange(lo, hi, dtype=np.uint64) * np.uint64(step)

    def check_info(self):
        info = self.info.cpu().numpy()
        bad = np.nonzero(info)[0]
        if bad.size:
            raise IndefiniteError(int(info[bad[0]]) - 1, f"block {int(bad[0])}: pivot {int(info[bad[0]]) - 1}")

    def factor_compress_host(self, D, B, master=0, pinned=None, pieces=16):
        """Public host-buffer entry point: H2D of D/B, the batched pipeline (sketches
        generated on the device), D2H of (L_D, V, U, ranks); returns host arrays.

        The batch is cut into `pieces` slices pipelined over three streams -- the
        copy engine uploads slice k+1 while the SMs factor slice k and the other copy
        engine downloads slice k-1 -- so the step costs about one PCIe pass of the
        inputs instead of upload + compute + download."""
        if pinned is None:
            pinned = self.pinned_staging()
        st = pinned
        # page-locked caller buffers go straight to the copy engine; pageable numpy
        # arrays are staged through the pinned buffers first
        src = {}
        for key, a in (("D", D), ("B", B)):
            if isinstance(a, torch.Tensor) and a.is_pinned():
                src[key] = a
            else:
                np.copyto(st[key].numpy(), np.asarray(a))
                src[key] = st[key]
        comp = torch.cuda.current_stream()
        if self._streams is None:
            self._streams = (torch.cuda.Stream(), torch.cuda.Stream())
        up, down = self._streams
        up.wait_stream(comp)  # device buffers are free once earlier work on comp is done
        states = self.sketch_states(master)
        k = max(1, min(pieces, self.nb))
        bounds = [self.nb * i // k for i in range(k + 1)]
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            if hi == lo:
                continue
            ev = torch.cuda.Event()
            with torch.cuda.stream(up):
                self.D[lo:hi].copy_(src["D"][lo:hi], non_blocking=True)
                self.B[lo:hi].copy_(src["B"][lo:hi], non_blocking=True)
                ev.record(up)
            comp.wait_event(ev)
            self.run(master, lo=lo, hi=hi, states=states)
            done = torch.cuda.Event()
            done.record(comp)
            down.wait_event(done)
            with torch.cuda.stream(down):
                st["LD"][lo:hi].copy_(self.D[lo:hi], non_blocking=True)
                st["V"][lo:hi].copy_(self.V[lo:hi], non_blocking=True)
                st["U"][lo:hi].copy_(self.U[lo:hi], non_blocking=True)
                st["rank"][lo:hi].copy_(self.rank[lo:hi], non_blocking=True)
        down.synchronize()
        comp.wait_stream(down)
        self.check_info()
        return st["LD"].numpy(), st["V"].numpy(), st["U"].numpy(), st["rank"].numpy()

    def pinned_staging(self):
        nb, n, m, r = self.nb, self.n, self.m, self.r

        def pin(*shape, dtype=torch.float64):
            return torch.empty(*shape, dtype=dtype, pin_memory=True)

        return {"D": pin(nb, n, n), "B": pin(nb, m, n), "LD": pin(nb, n, n),
                "V": pin(nb, m, r), "U": pin(nb, n, r), "rank": pin(nb, dtype=torch.int32)}

    def h2d_bytes(self):
        return 8 * self.nb * (self.n * self.n + self.m * self.n)

    def d2h_bytes(self):
        return 8 * self.nb * (self.n * self.n + self.m * self.r + self.n * self.r) + 4 * self.nb

    def results(self, i):
        """Host copies (L_D, L_O, V, U) of block i, ranks applied."""
        k = int(self.rank[i].item())
        return (self.D[i].cpu().numpy(), self.B[i].cpu().numpy(), self.V[i, :, :k].cpu().numpy(),
                self.U[i, :, :k].cpu().numpy())
