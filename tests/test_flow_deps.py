"""rsc_flow_deps (host): the op graph of the dataflow apply must order every pair of
conflicting accesses of the sequential program (read-after-write, write-after-read,
write-after-write unless both are accumulations), and nothing it reports may point
forward.  Random op lists over three vectors, contiguous and indexed accesses."""

import numpy as np
import pytest

from paper_1507_05593_b200 import _lib


def _random_program(rng, nops, lens, idx_host):
    bases = np.array([1 << 20, 1 << 24, 1 << 28], dtype=np.int64)  # fake device addresses
    ops = []
    for _ in range(nops):
        acc = []
        for _side in range(2):
            b = int(rng.integers(3))
            if rng.random() < 0.35 and idx_host.size > 8:  # indexed access into buffer b
                ln = int(rng.integers(1, 8))
                off = int(rng.integers(0, idx_host.size - ln))
                acc.append((b, int(bases[b]), off, ln))
            else:
                ln = int(rng.integers(1, 12))
                st = int(rng.integers(0, lens[b] - ln))
                acc.append((b, int(bases[b]) + 8 * st, -1, ln))
        ops.append((acc[0], acc[1], int(rng.random() < 0.3)))
    return bases, ops


def _elements(acc, idx_host):
    b, addr, off, ln = acc
    base = (addr - [1 << 20, 1 << 24, 1 << 28][b]) // 8
    if off < 0:
        return {(b, base + k) for k in range(ln)}
    return {(b, base + int(idx_host[off + k])) for k in range(ln)}


@pytest.mark.parametrize("seed", range(6))
def test_flow_deps_orders_every_conflict(seed):
    lib = _lib.load()
    rng = np.random.default_rng(seed)
    lens = np.array([40, 40, 60], dtype=np.int64)
    idx_host = rng.integers(0, 38, size=200).astype(np.int32)
    idx_dev = 1 << 40
    nops = 120
    bases, ops = _random_program(rng, nops, lens, idx_host)
    xa = np.array([o[0][1] for o in ops], dtype=np.int64)
    xi = np.array([0 if o[0][2] < 0 else idx_dev + 4 * o[0][2] for o in ops], dtype=np.int64)
    xl = np.array([o[0][3] for o in ops], dtype=np.int32)
    ya = np.array([o[1][1] for o in ops], dtype=np.int64)
    yi = np.array([0 if o[1][2] < 0 else idx_dev + 4 * o[1][2] for o in ops], dtype=np.int64)
    yl = np.array([o[1][3] for o in ops], dtype=np.int32)
    asg = np.array([o[2] for o in ops], dtype=np.int32)
    need = np.empty(nops, np.int32)
    sptr = np.empty(nops + 1, np.int32)
    cap = 100000
    succ = np.empty(cap, np.int32)
    ne = lib.rsc_flow_deps(nops, xa.ctypes.data, xi.ctypes.data, xl.ctypes.data, ya.ctypes.data, yi.ctypes.data,
                           yl.ctypes.data, asg.ctypes.data, 3, bases.ctypes.data, lens.ctypes.data,
                           idx_host.ctypes.data, idx_dev, idx_host.size, need.ctypes.data, sptr.ctypes.data,
                           succ.ctypes.data, cap)
    assert 0 <= ne <= cap
    succ = succ[:ne]
    # edges point forward; need = in-degree
    indeg = np.zeros(nops, np.int64)
    reach = np.zeros((nops, nops), dtype=bool)
    for p in range(nops):
        for o in succ[sptr[p]:sptr[p + 1]]:
            assert o > p
            indeg[o] += 1
            reach[p, o] = True
    assert np.array_equal(indeg, need)
    for p in range(nops - 1, -1, -1):  # transitive closure (edges point forward)
        for o in np.nonzero(reach[p])[0]:
            reach[p] |= reach[o]
    R = [_elements(o[0], idx_host) for o in ops]
    Wr = [_elements(o[1], idx_host) for o in ops]
    for a in range(nops):
        for b in range(a + 1, nops):
            raw = Wr[a] & R[b]
            war = R[a] & Wr[b]
            waw = (Wr[a] & Wr[b]) and (asg[a] or asg[b])
            if raw or war or waw:
                assert reach[a, b], (a, b, raw, war, waw)


def test_flow_deps_grows_capacity():
    lib = _lib.load()
    bases = np.array([1 << 20], dtype=np.int64)
    lens = np.array([16], dtype=np.int64)
    n = 5  # op k reads what op k-1 wrote: a chain of 4 edges
    xa = np.array([bases[0] + 8 * (k % 2) * 8 for k in range(n)], dtype=np.int64)
    ya = np.array([bases[0] + 8 * ((k + 1) % 2) * 8 for k in range(n)], dtype=np.int64)
    z = np.zeros(n, np.int64)
    ln = np.full(n, 8, np.int32)
    asg = np.ones(n, np.int32)
    idx = np.zeros(1, np.int32)
    need = np.empty(n, np.int32)
    sptr = np.empty(n + 1, np.int32)
    succ = np.empty(1, np.int32)
    args = (n, xa.ctypes.data, z.ctypes.data, ln.ctypes.data, ya.ctypes.data, z.ctypes.data, ln.ctypes.data,
            asg.ctypes.data, 1, bases.ctypes.data, lens.ctypes.data, idx.ctypes.data, 1 << 40, 1)
    ne = lib.rsc_flow_deps(*args, need.ctypes.data, sptr.ctypes.data, succ.ctypes.data, 1)
    assert ne > 1
    succ = np.empty(ne, np.int32)
    assert lib.rsc_flow_deps(*args, need.ctypes.data, sptr.ctypes.data, succ.ctypes.data, ne) == ne
    assert need[0] == 0 and all(need[1:] >= 1)
