"""Preconditioner application z = P^T (L L^T)^{-1} P r on the device
(reference factor.py:175-218).

Forward sweep: per unit, a diagonal solve of its columns, then the coupling update
y[R] -= L_O w (dense panel, materialized interior coupling Y_B, or V (U^T w));
backward sweep mirrored.  With Y_B materialized the interior branch (two in-block
solves + sparse coupling, factor.py:189-194,206-210) is the same operator as the
dense branch, so every unit runs the same kernels.

Level scheduling: a unit depends only on the units whose rows reach into its
columns (its update sources), so units are grouped by height in that DAG.  Each
level is a few *phases* of the mixed-mode GEMV: the diagonal solves (explicit
inverses, row-parallel), then the dense couplings together with the first factor of
every low-rank coupling, then the second low-rank factor; diagonal trees of the
level advance in lock-step waves (Alg. 4 flattened), two phases per wave.  Each
phase is ONE launch of rsc_gemv_multi (mode and alpha per problem).  (A persistent
single-launch executor with grid barriers between phases measured no faster: the
phases are latency-bound, not launch-bound.)  Two vectors alternate roles instead of
copying: in the forward sweep the right-hand sides accumulate in `y` and every
solved block is written to `y2` (couplings read solved values from `y2`); the
backward sweep starts from `y2` and writes `y`.  All low-rank intermediates live in
one buffer zeroed once per apply.  Descriptors are static after factorization and
built once; after a few eager applies the whole sweep is replayed from a CUDA graph.

Flattened tree inverses (TREE_INV, default): the block substitution of a diagonal
tree (Alg. 4, diagblocks.py:192-273) is a chain of 3 L - 2 dependent phases for L
leaves.  The inverse of a block triangle [[D1, 0], [V U^T, D2]] is
[[D1^{-1}, 0], [-(D2^{-1} V)(D1^{-T} U)^T, D2^{-1}]]: the same tree with the same
ranks.  So once per factorization every coupling is carried through its sibling
subtrees' solves (V' = D2^{-1} V, U' = D1^{-T} U; dense couplings D2^{-1} B D1^{-1}),
all in lock-step batched Alg. 4 waves, and every application of a tree is two
phases: all leaf inverses and all U'^T r at once, then all V' t.
"""

import os

import numpy as np
import torch

from . import _lib
from . import engine as E
from ._lib import int_array, ptr_array
from .factor import DenseTri, DeviceTree, DevLR



class _Phase:
    """Problems of one phase of the apply program (no dependencies among them):
    (M ptr, rows, cols, ldm, x ptr, xidx ptr|0, y ptr, yidx ptr|0, mode, alpha)."""

    def __init__(self):
        self.items = []
        self.lr = []  # (item index, U data_ptr) of the low-rank factor items: cols = rank

    def add(self, *item, lr=None):
        if lr is not None:  # kept even at rank 0: a later refactorization may raise it
            if item[1] > 0:
                self.lr.append((len(self.items), lr))
                self.items.append(item)
        elif item[1] > 0 and item[2] > 0:
            self.items.append(item)


class _ClusterTasks:
    """One launch of cluster tasks (rsc_apply_cluster_tasks): the Alg. 4 op list of
    every diagonal block tree of a level, one thread-block cluster per tree."""

    items = ()
    lr = ()

    def __init__(self, ops):
        self.ops = ops  # [_Phase]: one ordered op list per tree


def _cap(lr):
    """Column capacity of a low-rank block: its U / V are views of the sketch-padded
    buffers (numeric._finalize_ranks), so a refactorization's rank fits this."""
    U = lr.U
    return U.stride(0) if U.dim() == 2 and U.stride(1) == 1 else lr.k


class DeviceApply:
    """The apply program of a factor.  For a factor sharded by ND subtree
    (distributed.factorize_distributed, F.dist set) every rank holds its own subtree
    units plus the replicated top separators: the program runs the local units'
    forward sweep, sums the top separators' right-hand sides over the ranks (one
    all-reduce of the top rows; rank 0 contributes r there, the others only their
    coupling updates), runs the top units' forward and backward sweeps (identical on
    every rank), then the local backward sweep.  The result is exact on the rank's
    own rows and the top rows (pcg combines the ranks' rows)."""

    def __init__(self, F):
        # no strong reference back to the factor (it owns this program): a cycle would
        # keep the factor's device arena alive until the cyclic GC runs
        self.n = F.n
        self.nunits = len(F.dunits)
        plan = F.plan
        self.fwd = E.to_dev(np.asarray(F.perm.forward, dtype=np.int32))
        self.inv = E.to_dev(np.asarray(F.perm.inverse, dtype=np.int32))
        self.y = E.empty(self.n, 1)
        self.y2 = E.empty(self.n, 1)
        self.zbuf = E.empty(self.n)
        self.r_in = E.empty(self.n)
        units = F.dunits
        self._build_inverses(units)
        # every low-rank block is used once per sweep: 2 * sum(k) intermediates
        ksum = 0
        for u in units:
            if isinstance(u.off, DevLR):
                ksum += _cap(u.off)
            if isinstance(u.diag, DeviceTree):
                ksum += sum(_cap(b) for b in u.diag.blocks.values() if isinstance(b, DevLR))
        self.tall = E.empty(max(2 * ksum, 1))
        self._toff = 0
        uidx = {un.u: i for i, un in enumerate(units)}
        self.dist = getattr(F, "dist", None)
        shared = set(self.dist["top_units"]) if self.dist else set()
        self.flow = self.FLOW and not self.dist
        task_of = self._subtree_tasks(units, plan) if not (self.dist or self.flow) else \
            np.full(len(units), -1, dtype=np.int64)

        def levels(members):
            lv = {}
            for i in members:
                un = units[i]
                v = 0
                if un.kind == "node":
                    for ps in plan.tarr[un.j]["s"].tolist():
                        su = uidx.get(plan.sources[ps].unit)
                        if su is not None and su in lv:  # sources outside `members` run before
                            v = max(v, lv[su] + 1)
                lv[i] = v
            n = max(lv.values(), default=-1) + 1
            return [[units[i] for i in members if lv[i] == k] for k in range(n)]

        local = [i for i in range(len(units)) if task_of[i] < 0 and units[i].u not in shared]
        top = [i for i in range(len(units)) if units[i].u in shared]
        g_local, g_top = levels(local), levels(top)
        self.phases = []
        yb, y2b = self.y.data_ptr(), self.y2.data_ptr()
        self.tasks = {False: self._task_ops(units, task_of, plan, yb, y2b, False),
                      True: self._task_ops(units, task_of, plan, y2b, yb, True)}
        for us in g_local:
            self._level(us, plan, yb, y2b, backward=False)
        self.n_local_fwd = len(self.phases)  # the top rows are all-reduced here (sharded factor)
        for us in g_top:
            self._level(us, plan, yb, y2b, backward=False)
        self.n_fwd = len(self.phases)
        for us in reversed(g_top):
            self._level(us, plan, y2b, yb, backward=True)
        for us in reversed(g_local):
            self._level(us, plan, y2b, yb, backward=True)
        if self.dist:
            cols = np.concatenate([np.arange(units[i].c0, units[i].c1) for i in top]) if top else \
                np.zeros(0, np.int64)
            self.top_cols = E.to_dev(cols.astype(np.int32))
            self.top_buf = E.empty(max(cols.size, 1), 1)
            own = np.concatenate([np.arange(units[i].c0, units[i].c1) for i in local]) if local else \
                np.zeros(0, np.int64)
            # rows (in the permuted order) this rank's result is exact on: its own + the top
            self.exact_cols = np.concatenate([own, cols]).astype(np.int64)
        self._pack()
        self._idx = plan.idx
        if self.flow:
            self._build_flow()
        self.graph = None
        self.calls = 0

    # -- the dataflow program ------------------------------------------------------
    # The whole apply as one persistent launch (rsc_apply_flow): the level phases
    # above give a valid sequential order of the GEMV ops; rsc_flow_deps turns it into
    # the op graph (hazards on the vectors), and the kernel runs every op as soon as
    # the ops feeding it are done.  Off by default (RSC_APPLY_FLOW=1 turns it on): on
    # config[4] it measured 10.2 ms against 8.4 ms for the level phases + subtree
    # tasks (profiles/r02/apply_flow_cfg4.txt).  Its trace shows why: the critical
    # path is 898 dependent ops long (the top separators' unit chain, three GEMVs per
    # low-rank unit), 1.7 us of signal latency plus ~6 us per op -- the same chain the
    # phases walk, with a per-item cost the launch-per-phase path does not pay.
    FLOW = os.environ.get("RSC_APPLY_FLOW", "0") == "1"

    def _build_flow(self):
        lib = _lib.load()
        items = [it for ph in self.phases for it in ph.items]
        nops = len(items)
        self.flow_nops = nops
        if nops == 0:
            self.flow_dev = None
            return
        c = list(zip(*items))
        M, rows, cols, ld = ptr_array(c[0]), int_array(c[1]), int_array(c[2]), int_array(c[3])
        x, xi, y, yi = ptr_array(c[4]), ptr_array(c[5]), ptr_array(c[6]), ptr_array(c[7])
        modes = int_array(c[8])
        alphas = np.ascontiguousarray(np.asarray(c[9], dtype=np.float64))
        trans = (modes & 1).astype(bool)
        xlen = np.where(trans, rows, cols).astype(np.int32)
        ylen = np.where(trans, cols, rows).astype(np.int32)
        asg = ((modes & 4) != 0).astype(np.int32)
        bases = np.array([self.y.data_ptr(), self.y2.data_ptr(), self.tall.data_ptr()], dtype=np.int64)
        lens = np.array([self.n, self.n, self.tall.numel()], dtype=np.int64)
        idx = self._idx
        need = np.empty(nops, dtype=np.int32)
        sptr = np.empty(nops + 1, dtype=np.int32)
        cap = 8 * nops
        while True:
            succ = np.empty(max(cap, 1), dtype=np.int32)
            ne = lib.rsc_flow_deps(nops, x.ctypes.data, xi.ctypes.data, xlen.ctypes.data, y.ctypes.data,
                                   yi.ctypes.data, ylen.ctypes.data, asg.ctypes.data, 3, bases.ctypes.data,
                                   lens.ctypes.data, idx.host.ctypes.data, idx.dev.data_ptr(), idx.host.size,
                                   need.ctypes.data, sptr.ctypes.data, succ.ctypes.data, cap)
            if ne < 0:
                raise RuntimeError(f"rsc_flow_deps failed ({ne})")
            if ne <= cap:
                break
            cap = ne
        args = [M.ctypes.data, rows.ctypes.data, cols.ctypes.data, ld.ctypes.data, x.ctypes.data, xi.ctypes.data,
                y.ctypes.data, yi.ctypes.data, modes.ctypes.data, alphas.ctypes.data]
        db = lib.rsc_gemv_desc_bytes()
        desc = np.empty(nops * db, dtype=np.uint8)
        total = lib.rsc_flow_describe(nops, *args, desc.ctypes.data, None)
        item_op = np.empty(total, dtype=np.int32)
        total = lib.rsc_flow_describe(nops, *args, desc.ctypes.data, item_op.ctypes.data)
        self.flow_edges = int(ne)
        self.flow_items = int(total)
        self.flow_dev = (E.to_dev(desc), E.to_dev(item_op), E.to_dev(need), E.to_dev(sptr),
                         E.to_dev(succ[:max(int(ne), 1)]), torch.zeros(1 + 2 * nops, dtype=torch.int32,
                                                                       device="cuda"))

    # -- subtree tasks -------------------------------------------------------------
    TASK_BYTES = int(float(os.environ.get("RSC_APPLY_TASK_MB", "1")) * (1 << 20))  # subtree tasks up to 1 MB (measured 3-5% faster applies on config[4])

    def _subtree_tasks(self, units, plan):
        """Unit forest (parent = the unit holding the first row of a unit's row
        structure, i.e. its first update target) and the maximal subtrees of at most
        TASK_BYTES factor bytes: task_of[i] = index of the task's root unit, or -1
        for the top units that run as level phases."""
        part = plan.sym.partition
        owner = np.full(part.count, -1, dtype=np.int64)
        for i, un in enumerate(units):
            if un.kind == "node":
                owner[un.j] = i
            else:
                owner[np.asarray(un.members)] = i
        nb = np.zeros(len(units))
        parent = np.full(len(units), -1, dtype=np.int64)
        for i, un in enumerate(units):
            nc = un.ncols
            b = nc * (nc + 1) / 2.0
            if isinstance(un.off, DevLR):
                b += (un.rows.size + nc) * un.off.k
            elif un.off is not None:
                b += un.off.numel()
            if isinstance(un.diag, DeviceTree):
                b = 1e30  # diagonal trees stay in the level phases (their waves are wide)
            nb[i] = 8.0 * b
            if un.rows.size:
                parent[i] = owner[part.supernode_of(int(un.rows[0]))]
        sub = nb.copy()
        for i in range(len(units)):  # units are in post-order: children first
            if parent[i] >= 0:
                sub[parent[i]] += sub[i]
        small = sub <= self.TASK_BYTES
        task_of = np.full(len(units), -1, dtype=np.int64)
        for i in range(len(units) - 1, -1, -1):
            if not small[i]:
                continue
            p = parent[i]
            task_of[i] = task_of[p] if (p >= 0 and small[p]) else i
        self.n_tasks = int(np.sum(small & ((parent < 0) | ~small[np.maximum(parent, 0)])))
        return task_of

    def _task_ops(self, units, task_of, plan, rhs, out, backward):
        """Op lists of every subtree task (forward: units in sweep order; backward:
        reversed), each op a _Phase item; returns [(task root, _Phase)] largest first."""
        cols_task = np.full(self.n, -1, dtype=np.int64)
        for i, un in enumerate(units):
            if task_of[i] >= 0:
                cols_task[un.c0:un.c1] = task_of[i]
        tasks = {}
        order = range(len(units)) if not backward else range(len(units) - 1, -1, -1)
        for i in order:
            t = task_of[i]
            if t < 0:
                continue
            ph = tasks.setdefault(t, _Phase())
            un = units[i]
            own = bool(un.rows.size == 0 or np.all(cols_task[un.rows] == t))
            if not backward:
                self._solve(ph, un.diag, rhs + 8 * un.c0, out + 8 * un.c0, False)
                if un.rows.size and un.off is not None:
                    self._couplings_into(ph, ph, un, plan, rhs, out, False, 16 if own else 0)
            else:
                if un.rows.size and un.off is not None:
                    self._couplings_into(ph, ph, un, plan, rhs, out, True, 16)
                self._solve(ph, un.diag, rhs + 8 * un.c0, out + 8 * un.c0, True)
        lst = sorted(tasks.items(), key=lambda kv: -sum(it[1] * it[2] for it in kv[1].items))
        return lst

    def _emit(self, ph):
        if ph.items:
            self.phases.append(ph)

    def _pack(self):
        """Every phase -> one prebuilt rsc_gemv_multi launch (host arrays kept)."""
        lib = _lib.load()
        self.launches = []
        self._lr_index = []  # (launch, item, U ptr): the items whose cols is a rank
        for ph in self.phases:
            if isinstance(ph, _ClusterTasks):
                self.launches.append((0, None, None))
                continue
            self._lr_index.extend((len(self.launches), i, key) for i, key in ph.lr)
            c = list(zip(*ph.items))
            arrs = [ptr_array(c[0]), int_array(c[1]), int_array(c[2]), int_array(c[3]), ptr_array(c[4]),
                    ptr_array(c[5]), ptr_array(c[6]), ptr_array(c[7]), int_array(c[8]),
                    np.ascontiguousarray(np.asarray(c[9], dtype=np.float64))]
            self.launches.append((len(ph.items), arrs, [a.ctypes.data for a in arrs]))
        self._fn = lib.rsc_gemv_multi
        self._build_dev()
        self._build_tasks()
        self._build_cluster_tasks()

    def _build_cluster_tasks(self):
        """Device descriptors of every cluster-task launch (rsc_gemv_describe over all
        ops of the launch's trees plus one sentinel, per-tree op offsets)."""
        lib = _lib.load()
        db = lib.rsc_gemv_desc_bytes()
        self.ctask_dev = {}
        self._ctask_lr = []  # (phase index, tree index, item index, U ptr)
        for li, ph in enumerate(self.phases):
            if not isinstance(ph, _ClusterTasks):
                continue
            items, ptr = [], [0]
            for ti, op in enumerate(ph.ops):
                self._ctask_lr.extend((li, ti, i, key) for i, key in op.lr)
                items.extend(op.items)
                ptr.append(len(items))
            items = items + [(items[0][0], 0, 0, 1, items[0][4], 0, items[0][6], 0, 0, 0.0)]  # sentinel
            c = list(zip(*items))
            arrs = [ptr_array(c[0]), int_array(c[1]), int_array(c[2]), int_array(c[3]), ptr_array(c[4]),
                    ptr_array(c[5]), ptr_array(c[6]), ptr_array(c[7]), int_array(c[8]),
                    np.ascontiguousarray(np.asarray(c[9], dtype=np.float64))]
            n = len(items)
            desc = np.empty(n * db, dtype=np.uint8)
            blocks = np.empty(n, dtype=np.int64)
            _lib.check(lib.rsc_gemv_describe(n, *[a.ctypes.data for a in arrs], desc.ctypes.data,
                                             blocks.ctypes.data), "rsc_gemv_describe")
            self.ctask_dev[li] = (E.to_dev(desc), E.to_dev(np.asarray(ptr, dtype=np.int32)), len(ph.ops))

    def _build_tasks(self):
        """Device descriptors of the subtree tasks of both sweeps (rsc_apply_tasks)."""
        lib = _lib.load()
        db = lib.rsc_gemv_desc_bytes()
        self.task_dev = {}
        self._task_lr = []  # (direction, op index, U ptr)
        for bw, lst in self.tasks.items():
            items, ptr = [], [0]
            for _, ph in lst:
                base = len(items)
                self._task_lr.extend((bw, base + i, key) for i, key in ph.lr)
                items.extend(ph.items)
                ptr.append(len(items))
            if not lst:
                continue
            items = items + [(items[0][0], 0, 0, 1, items[0][4], 0, items[0][6], 0, 0, 0.0)]  # sentinel
            c = list(zip(*items))
            arrs = [ptr_array(c[0]), int_array(c[1]), int_array(c[2]), int_array(c[3]), ptr_array(c[4]),
                    ptr_array(c[5]), ptr_array(c[6]), ptr_array(c[7]), int_array(c[8]),
                    np.ascontiguousarray(np.asarray(c[9], dtype=np.float64))]
            n = len(items)
            desc = np.empty(n * db, dtype=np.uint8)
            blocks = np.empty(n, dtype=np.int64)
            _lib.check(lib.rsc_gemv_describe(n, *[a.ctypes.data for a in arrs], desc.ctypes.data,
                                             blocks.ctypes.data), "rsc_gemv_describe")
            self.task_dev[bw] = (E.to_dev(desc), E.to_dev(np.asarray(ptr, dtype=np.int32)), len(lst), arrs)

    DEV_MIN = 225  # phases with more problems than one parameter block (GMAXP = 224)

    def _build_dev(self):
        """Large phases run from device-resident descriptors: one launch per phase
        (rsc_gemv_multi_dev) instead of one per 224 problems."""
        lib = _lib.load()
        db = lib.rsc_gemv_desc_bytes()
        self.dev = {}
        for li, (n, _, args) in enumerate(self.launches):
            if n < self.DEV_MIN:
                continue
            desc = np.empty(n * db, dtype=np.uint8)
            blocks = np.empty(n, dtype=np.int64)
            _lib.check(lib.rsc_gemv_describe(n, *args, desc.ctypes.data, blocks.ctypes.data), "rsc_gemv_describe")
            b2p = np.repeat(np.arange(n, dtype=np.int32), blocks)
            self.dev[li] = (E.to_dev(desc), E.to_dev(b2p), int(b2p.size))

    def rekey(self, F):
        """Adopt a refactorization whose kept ranks differ from this program's (the
        QRCP cutoff sits on rounding-level |R_ii|, so FP64 atomic sums move a few ranks
        between replays).  Same memory (graph replay), same block structure: only the
        rank dimension of the low-rank items changes -- patch it in the packed launch
        arrays and re-capture the graph instead of rebuilding the program (0.2-0.4 s
        on config[4]).  False if the blocks do not match (caller rebuilds)."""
        ks = {}
        for u in F.dunits:
            if isinstance(u.off, DevLR):
                ks[u.off.U.data_ptr()] = u.off.k
            if isinstance(u.diag, DeviceTree):
                for b in u.diag.blocks.values():
                    if isinstance(b, DevLR):
                        ks[b.U.data_ptr()] = b.k
        have = ({key for _, _, key in self._lr_index} | {key for _, _, key in self._task_lr}
                | {key for _, _, _, key in self._ctask_lr})
        if set(ks) != have or len(F.dunits) != self.nunits:
            return False
        self._tree_inverse_buffers(F.dunits, old=self.tinv)  # the solves read the new ranks
        self._refresh_graph = None
        for li, ii, key in self._lr_index:
            self.launches[li][1][2][ii] = ks[key]
        for ph in self.phases:  # the flow program is rebuilt from the phase items
            for i, key in ph.lr:
                it = list(ph.items[i])
                it[2] = ks[key]
                ph.items[i] = tuple(it)
        if self.flow:
            self._build_flow()
        self._build_dev()  # the device descriptors carry the ranks too
        for bw, lst in self.tasks.items():  # task ops: rebuild with the new ranks
            for _, ph in lst:
                for i, key in ph.lr:
                    it = list(ph.items[i])
                    it[2] = ks[key]
                    ph.items[i] = tuple(it)
        self._build_tasks()
        for li, ti, ii, key in self._ctask_lr:
            op = self.phases[li].ops[ti]
            it = list(op.items[ii])
            it[2] = ks[key]
            op.items[ii] = tuple(it)
        self._build_cluster_tasks()
        self.graph = None
        self.calls = min(self.calls, self.GRAPH_AFTER)
        return True

    def _run_program(self):
        s = E.stream_handle()
        lib = _lib.load()
        if self.flow:
            if self.flow_dev is not None:
                d, io, nd, sp, sc, st = self.flow_dev
                _lib.check(lib.rsc_apply_flow(d.data_ptr(), io.data_ptr(), nd.data_ptr(), sp.data_ptr(),
                                              sc.data_ptr(), st.data_ptr(), self.flow_nops, self.flow_items, s),
                           "rsc_apply_flow")
            return
        dev, fdev = self.dev, lib.rsc_gemv_multi_dev

        def tasks(bw):
            t = self.task_dev.get(bw)
            if t is not None:
                _lib.check(lib.rsc_apply_tasks(t[0].data_ptr(), t[1].data_ptr(), t[2], s), "rsc_apply_tasks")

        tasks(False)  # forward: the subtrees first, then the top levels
        for li, (n, _, args) in enumerate(self.launches):
            if li == self.n_local_fwd and self.dist:
                self._reduce_top()
            if li in self.ctask_dev:
                d, ptr, nt = self.ctask_dev[li]
                _lib.check(lib.rsc_apply_cluster_tasks(d.data_ptr(), ptr.data_ptr(), nt, self.CLUSTER, s),
                           "rsc_apply_cluster_tasks")
            elif n == 0:
                continue
            elif li in dev:
                d, b2p, tot = dev[li]
                _lib.check(fdev(d.data_ptr(), b2p.data_ptr(), tot, s), "rsc_gemv_multi_dev")
            else:
                _lib.check(self._fn(n, *args, s), "rsc_gemv_multi")
        if self.dist and self.n_local_fwd >= len(self.launches):
            self._reduce_top()
        tasks(True)  # backward: the top levels first, then the subtrees

    def _reduce_top(self):
        """Sum the top separators' forward right-hand sides over the ranks."""
        import torch.distributed as dist

        if self.top_cols.numel() == 0:
            return
        E.gather_rows(self.top_cols, self.y, self.top_buf)
        grp = self.dist["group"]
        if dist.get_backend(grp) == "gloo":
            h = self.top_buf.cpu()
            dist.all_reduce(h, group=grp)
            self.top_buf.copy_(h)
        else:
            dist.all_reduce(self.top_buf, group=grp)
        # y[top] = sum: scatter-add onto zeroed rows
        self.y[self.top_cols.long()] = 0.0
        E.scatter_add_rows(self.top_cols, self.top_buf, self.y)

    # -- program construction ------------------------------------------------------
    def _build_inverses(self, units):
        """Linv = L^{-1} (one batched TRSM against identities) and LinvT for every dense
        diagonal triangle and tree leaf: O(n^3/3) once per factor, after which every
        apply's diagonal solves are bandwidth-bound GEMVs.  The buffers hang on the
        triangles and are rewritten in place, so refresh_inverses() re-derives them
        after a graph replay has overwritten the factor with new values."""
        tris = []
        for u in units:
            if isinstance(u.diag, DenseTri):
                tris.append(u.diag)
            elif isinstance(u.diag, DeviceTree):
                tris.extend(b for s_, b in u.diag.blocks.items() if u.diag.shape.nodes[s_].is_leaf)
        self.tris = [t for t in tris if t.n]
        self._sq = None
        if any(t.Linv is None for t in self.tris):
            self.mem = E.Arena()
            for t in self.tris:
                if t.Linv is None:
                    t.Linv = self.mem.empty(t.n, t.n)
                    t.LinvT = self.mem.empty(t.n, t.n)
                    t.inv_mem = self.mem  # a later program may reuse these views
        self._tree_inverse_buffers(units)
        self.refresh_inverses()

    # Flattened inverses of the diagonal block trees (module docstring).
    # RSC_APPLY_TREE_INV=0 keeps the lock-step Alg. 4 waves.
    TREE_INV = os.environ.get("RSC_APPLY_TREE_INV", "1") == "1"

    def _tree_inverse_buffers(self, units, old=None):
        """tree.inv[s] of every internal block s: (V', U') at the coupling's column
        capacity, or (Y, W) for a dense coupling B (Y = D2^{-1} B, then
        W = (Y D1^{-1})^T).  `old`: the tree units of the program being re-keyed,
        whose buffers the new factor's trees adopt (same memory, same structure)."""
        self.tinv = []
        if not self.TREE_INV:
            return
        trees = [u for u in units if isinstance(u.diag, DeviceTree)]
        if old is not None:
            for u, uo in zip(trees, old):
                u.diag.inv, u.diag.inv_mem = uo.diag.inv, uo.diag.inv_mem
        for u in trees:
            tree = u.diag
            if getattr(tree, "inv", None) is None:
                mem = getattr(self, "mem", None)
                if mem is None:
                    mem = self.mem = E.Arena()
                tree.inv, tree.inv_mem = {}, mem
                for s, b in tree.blocks.items():
                    nd = tree.shape.nodes[s]
                    if nd.is_leaf:
                        continue
                    n1, n2 = nd.split - nd.lo, nd.hi - nd.split
                    if isinstance(b, DevLR):
                        cap = _cap(b)
                        tree.inv[s] = (mem.empty(n2, cap), mem.empty(n1, cap))
                    else:
                        tree.inv[s] = (mem.empty(n2, n1), mem.empty(n1, n2))
            self.tinv.append(u)
        self._tinv_key = None

    def _refresh_tree_inverses(self):
        from .numeric import diag_solve_many

        if not self.tinv:
            return
        lib = E.ensure_gemm_workspace()
        cp, tp, it1, it2 = [], [], [], []
        for u in self.tinv:
            tree = u.diag
            for s, (A0, A1) in tree.inv.items():
                nd, b = tree.shape.nodes[s], tree.blocks[s]
                if isinstance(b, DevLR):
                    k = b.k
                    if k == 0:
                        continue
                    Vi, Ui = A0[:, :k], A1[:, :k]
                    cp.append((b.V, Vi))
                    cp.append((b.U, Ui))
                    it1.append((u, Vi, False, nd.right.s))
                    it1.append((u, Ui, True, nd.left.s))
                else:
                    cp.append((b, A0))
                    it1.append((u, A0, False, nd.right.s))
                    tp.append((A0, A1))
                    it2.append((u, A1, True, nd.left.s))

        def copies(pairs, trans):
            if not pairs:
                return
            arrs = [ptr_array([a.data_ptr() for a, _ in pairs]), ptr_array([d.data_ptr() for _, d in pairs]),
                    int_array([a.shape[0] for a, _ in pairs]), int_array([a.shape[1] for a, _ in pairs]),
                    int_array([E.ld(a) for a, _ in pairs]), int_array([E.ld(d) for _, d in pairs])]
            _lib.check(lib.rsc_copy2d_batched(len(pairs), *[x.ctypes.data for x in arrs], trans,
                                              E.stream_handle()), "rsc_copy2d_batched")

        copies(cp, 0)
        diag_solve_many(it1, E.empty)
        copies(tp, 1)
        diag_solve_many(it2, E.empty)

    def refresh_inverses(self):
        """Re-derive every explicit inverse from the factor's current values.  A
        refactorization loop calls this once per factorization with unchanged
        structure, so from the second call it is replayed from a CUDA graph (the
        tree solves are ~400 small launches: host-bound when issued eagerly)."""
        if not self.tris:
            return
        self._refresh_calls = getattr(self, "_refresh_calls", 0) + 1
        g = getattr(self, "_refresh_graph", None)
        if g is None and self._refresh_calls > 1 and self.REFRESH_GRAPH:
            try:
                E.ensure_gemm_workspace()
                g = E.capture_graph(self._refresh_body)
            except Exception:
                g = False
            self._refresh_graph = g
        if g:
            g.replay()
        else:
            self._refresh_body()

    REFRESH_GRAPH = os.environ.get("RSC_APPLY_REFRESH_GRAPH", "1") == "1"

    def _refresh_body(self):
        tris = self.tris
        lib = _lib.load()
        if self._sq is None:
            ns = [t.n for t in tris]
            self._sq = (int_array(ns), ptr_array([t.Linv.data_ptr() for t in tris]),
                        ptr_array([t.LinvT.data_ptr() for t in tris]), int_array([E.ld(t.Linv) for t in tris]),
                        int_array([E.ld(t.LinvT) for t in tris]))
        n_, li, lt, ldi, ldt = self._sq
        s = E.stream_handle()
        _lib.check(lib.rsc_identity_batched(len(tris), li.ctypes.data, n_.ctypes.data, ldi.ctypes.data, s),
                   "rsc_identity_batched")
        E.trsm_batched("left", 0, [t.L.data_ptr() for t in tris], [t.n for t in tris], [E.ld(t.L) for t in tris],
                       [t.Dinv.data_ptr() for t in tris], [t.Linv.data_ptr() for t in tris], [t.n for t in tris],
                       [t.n for t in tris])
        _lib.check(lib.rsc_transpose_batched(len(tris), li.ctypes.data, lt.ctypes.data, n_.ctypes.data,
                                             ldi.ctypes.data, ldt.ctypes.data, s), "rsc_transpose_batched")
        self._refresh_tree_inverses()

    def _rows_ptr(self, plan, un):
        key = ("int", un.u) if un.kind == "interior" else un.j
        return plan.idx.ptr(plan.rows_off[key])

    def _t(self, k):
        p = self.tall.data_ptr() + 8 * self._toff
        self._toff += k
        return p

    @staticmethod
    def _solve(ph, tri, xp, yp, backward):
        """out = L^{-1} rhs (forward, Linv lower) or L^{-T} rhs (backward, LinvT upper)."""
        M = tri.LinvT if backward else tri.Linv
        ph.add(M.data_ptr(), tri.n, tri.n, E.ld(M), xp, 0, yp, 0, 12 if backward else 6, 1.0)

    def _level(self, us, plan, rhs, out, backward):
        """One level of a sweep; right-hand sides accumulate in `rhs`, solved blocks are
        written to `out` (base addresses of y / y2)."""
        dense = [u for u in us if isinstance(u.diag, DenseTri)]
        trees = [u for u in us if isinstance(u.diag, DeviceTree)]
        cpl = [u for u in us if u.rows.size and u.off is not None]
        if not backward:
            first = _Phase()
            for u in dense:
                self._solve(first, u.diag, rhs + 8 * u.c0, out + 8 * u.c0, False)
            small, big = self._split_trees(trees)
            first = self._tree_phases(big, rhs, out, False, first)
            self._emit(first)
            self._tree_cluster_tasks(small, rhs, out, False)
            self._couplings(cpl, plan, rhs, out, False)
        else:
            self._couplings(cpl, plan, rhs, out, True)
            first = _Phase()
            for u in dense:
                self._solve(first, u.diag, rhs + 8 * u.c0, out + 8 * u.c0, True)
            small, big = self._split_trees(trees)
            first = self._tree_phases(big, rhs, out, True, first)
            self._emit(first)
            self._tree_cluster_tasks(small, rhs, out, True)

    def _couplings(self, cpl, plan, rhs, out, backward):
        a, b = _Phase(), _Phase()
        for u in cpl:
            self._couplings_into(a, b, u, plan, rhs, out, backward, 0)
        self._emit(a)
        self._emit(b)

    def _couplings_into(self, a, b, u, plan, rhs, out, backward, excl):
        """Coupling update of unit u: items of the first factor into `a`, second into
        `b` (the same list for a subtree task, whose ops run in order).  `excl` = 16
        when the target rows belong to the caller alone (plain accumulate)."""
        rows = self._rows_ptr(plan, u)
        c0 = 8 * u.c0
        if isinstance(u.off, DevLR):
            k, t = u.off.k, self._t(_cap(u.off))
            U, V = u.off.U, u.off.V
            key = U.data_ptr()
            own_t = 16 if a is b else 0  # t is private: exclusive when the ops are ordered
            if not backward:  # t = U^T w ; y[R] -= V t
                a.add(U.data_ptr(), u.ncols, k, E.ld(U), out + c0, 0, t, 0, 1 | own_t, 1.0, lr=key)
                b.add(V.data_ptr(), u.rows.size, k, E.ld(V), t, 0, rhs, rows, 0 | excl, -1.0, lr=key)
            else:  # t = V^T y[R] ; w -= U t
                a.add(V.data_ptr(), u.rows.size, k, E.ld(V), out, rows, t, 0, 1 | own_t, 1.0, lr=key)
                b.add(U.data_ptr(), u.ncols, k, E.ld(U), t, 0, rhs + c0, 0, 0 | excl, -1.0, lr=key)
        elif not backward:  # y[R] -= L_O w
            a.add(u.off.data_ptr(), u.rows.size, u.ncols, E.ld(u.off), out + c0, 0, rhs, rows, 0 | excl, -1.0)
        else:  # w -= L_O^T y[R]
            a.add(u.off.data_ptr(), u.rows.size, u.ncols, E.ld(u.off), out, rows, rhs + c0, 0, 1 | excl, -1.0)

    # Alg. 4 of the diagonal trees as cluster tasks (one cluster per tree, its ops in
    # order) instead of lock-step waves of dependent launches.  Off by default: on
    # config[4] the apply measured 8.57 ms with waves, 8.9-9.2 ms with cluster tasks
    # for the trees under 0.25-2 MB per op and 18.2 ms for all trees
    # (profiles/r02/apply_tree_cluster_cfg4.txt): one 8-CTA cluster streams a tree's
    # ops no faster than a dependent launch over the whole GPU.
    TREE_CLUSTER = os.environ.get("RSC_APPLY_TREE_CLUSTER", "0") == "1"  # measured slower on config[4] (below)
    CLUSTER = 8
    # trees whose largest op moves more than this run as lock-step waves over the
    # whole GPU (one cluster's bandwidth is too low for them)
    TREE_CLUSTER_OP_BYTES = int(float(os.environ.get("RSC_APPLY_TREE_CLUSTER_MB", "0.5")) * (1 << 20))

    def _split_trees(self, trees):
        """(cluster-task trees, wave trees) by the bytes of each tree's largest op."""
        if not self.TREE_CLUSTER or self.flow:
            return [], trees
        small, big = [], []
        for u in trees:
            mx = 0
            for b in u.diag.blocks.values():
                if isinstance(b, DevLR):
                    mx = max(mx, 8 * max(b.V.shape[0], b.U.shape[0]) * _cap(b))
                elif isinstance(b, DenseTri):
                    mx = max(mx, 4 * b.n * b.n)  # the explicit inverse's triangle
                else:
                    mx = max(mx, 8 * b.numel())
            (small if mx <= self.TREE_CLUSTER_OP_BYTES else big).append(u)
        return small, big

    def _tree_cluster_tasks(self, trees, rhs, out, backward):
        from .numeric import tree_ops

        ybase = self.y.data_ptr()
        off = lambda v: v.data_ptr() - ybase  # tree_ops hands out views of self.y
        lists = []
        for u in trees:
            ph = _Phase()
            for op in tree_ops(u.diag, None, self.y[u.c0:u.c1], backward):
                if op[0] == "leaf":
                    if op[1].n:
                        self._solve(ph, op[1], rhs + off(op[2]), out + off(op[2]), backward)
                    continue
                _, b, Xs, Yd, tr = op
                xp, yp = out + off(Xs), rhs + off(Yd)
                if isinstance(b, DevLR):
                    t = self._t(_cap(b))
                    P1, P2 = (b.V, b.U) if tr else (b.U, b.V)
                    key = b.U.data_ptr()
                    # t = P1^T x: column sums over row slabs dealt to several CTAs (atomic)
                    ph.add(P1.data_ptr(), P1.shape[0], b.k, E.ld(P1), xp, 0, t, 0, 1, 1.0, lr=key)
                    # y -= P2 t: rows partitioned over the CTAs (exclusive)
                    ph.add(P2.data_ptr(), P2.shape[0], b.k, E.ld(P2), t, 0, yp, 0, 0 | 16, -1.0, lr=key)
                elif tr:  # Y -= B^T X: column sums (atomic)
                    ph.add(b.data_ptr(), b.shape[0], b.shape[1], E.ld(b), xp, 0, yp, 0, 1, -1.0)
                else:  # Y -= B X: rows (exclusive)
                    ph.add(b.data_ptr(), b.shape[0], b.shape[1], E.ld(b), xp, 0, yp, 0, 0 | 16, -1.0)
            if ph.items:
                lists.append(ph)
        if lists:
            self.phases.append(_ClusterTasks(lists))

    def _tree_phases(self, trees, rhs, out, backward, first):
        if self.TREE_INV and trees:
            return self._tree_flat(trees, rhs, out, backward, first)
        return self._tree_waves(trees, rhs, out, backward, first)

    def _tree_flat(self, trees, rhs, out, backward, first):
        """out = D^{-1} rhs (or D^{-T} rhs) of every tree through its flattened inverse:
        `first` gets every leaf inverse and the first factor of every coupling (all
        read rhs), a second phase accumulates the couplings' second factors into out."""
        second = _Phase()
        for u in trees:
            tree, base = u.diag, 8 * u.c0
            for s in tree.shape.order:
                nd, b = tree.shape.nodes[s], tree.blocks[s]
                if nd.is_leaf:
                    if b.n:
                        self._solve(first, b, rhs + base + 8 * nd.lo, out + base + 8 * nd.lo, backward)
                    continue
                A0, A1 = tree.inv[s]
                x1, x2 = base + 8 * nd.lo, base + 8 * nd.split
                n1, n2 = nd.split - nd.lo, nd.hi - nd.split
                if isinstance(b, DevLR):
                    t, key = self._t(_cap(b)), b.U.data_ptr()
                    if not backward:  # out[X2] -= V' (U'^T rhs[X1])
                        first.add(A1.data_ptr(), n1, b.k, E.ld(A1), rhs + x1, 0, t, 0, 1, 1.0, lr=key)
                        second.add(A0.data_ptr(), n2, b.k, E.ld(A0), t, 0, out + x2, 0, 0, -1.0, lr=key)
                    else:  # out[X1] -= U' (V'^T rhs[X2])
                        first.add(A0.data_ptr(), n2, b.k, E.ld(A0), rhs + x2, 0, t, 0, 1, 1.0, lr=key)
                        second.add(A1.data_ptr(), n1, b.k, E.ld(A1), t, 0, out + x1, 0, 0, -1.0, lr=key)
                elif not backward:  # out[X2] -= W^T rhs[X1], W = (D2^{-1} B D1^{-1})^T
                    second.add(A1.data_ptr(), n1, n2, E.ld(A1), rhs + x1, 0, out + x2, 0, 1, -1.0)
                else:  # out[X1] -= W rhs[X2]
                    second.add(A1.data_ptr(), n1, n2, E.ld(A1), rhs + x2, 0, out + x1, 0, 0, -1.0)
        self._emit(first)
        self._emit(second)
        return _Phase()

    def _tree_waves(self, trees, rhs, out, backward, first):
        """Alg. 4 of every tree in `trees`, in lock-step waves; wave w's leaf solves,
        dense couplings and first low-rank factors share one launch, the second
        low-rank factors a second one.  `first` (the level's own first phase) is
        merged into wave 0; returns the phase still to be launched."""
        from .numeric import tree_ops

        ybase = self.y.data_ptr()
        off = lambda v: v.data_ptr() - ybase  # tree_ops hands out views of self.y
        seqs = [tree_ops(u.diag, None, self.y[u.c0:u.c1], backward) for u in trees]
        seqs = [s for s in seqs if s]
        if not seqs:
            return first
        cur = first
        for w in range(max(len(s) for s in seqs)):
            second = _Phase()
            for s in seqs:
                if w >= len(s):
                    continue
                op = s[w]
                if op[0] == "leaf":
                    if op[1].n:
                        self._solve(cur, op[1], rhs + off(op[2]), out + off(op[2]), backward)
                    continue
                _, b, Xs, Yd, tr = op
                xp, yp = out + off(Xs), rhs + off(Yd)
                if isinstance(b, DevLR):
                    t = self._t(_cap(b))
                    P1, P2 = (b.V, b.U) if tr else (b.U, b.V)
                    key = b.U.data_ptr()
                    cur.add(P1.data_ptr(), P1.shape[0], b.k, E.ld(P1), xp, 0, t, 0, 1, 1.0, lr=key)
                    second.add(P2.data_ptr(), P2.shape[0], b.k, E.ld(P2), t, 0, yp, 0, 0, -1.0, lr=key)
                else:  # Y -= B X (forward) or Y -= B^T X (transposed)
                    cur.add(b.data_ptr(), b.shape[0], b.shape[1], E.ld(b), xp, 0, yp, 0, 1 if tr else 0, -1.0)
            self._emit(cur)
            self._emit(second)
            cur = _Phase()
        return cur

    # -- execution ---------------------------------------------------------------
    def _body(self):
        n = self.n
        self.tall.zero_()
        E.gather_rows(self.inv, self.r_in.reshape(n, 1), self.y)
        if self.dist and self.dist["rank"] != 0 and self.top_cols.numel():
            self.y[self.top_cols.long()] = 0.0  # rank 0 alone brings r to the top rows' sum
        self._run_program()
        E.gather_rows(self.fwd, self.y, self.zbuf.reshape(n, 1))

    # eager applies before the sweep is captured into a CUDA graph (capture costs
    # about two eager applies; PCG with 1-3 iterations never amortises it)
    GRAPH_AFTER = 3

    def __call__(self, r_dev, out=None):
        self.r_in.copy_(r_dev.reshape(-1))
        self.calls += 1
        if self.graph is None and self.calls > self.GRAPH_AFTER and not self.dist:
            try:
                self.graph = E.capture_graph(self._body)
            except Exception:
                self.graph = False
        if self.graph:
            self.graph.replay()
        else:
            self._body()
        z = out if out is not None else E.empty(self.n)
        z.copy_(self.zbuf)
        return z
