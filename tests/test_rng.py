"""Device Gaussian sketches vs the reference's own host stream.

The reference draws every sketch as
np.random.Generator(np.random.PCG64(_block_seed(seed, *tags))).standard_normal((m, r))
(kernels.py:85-92, factor.py:324-326).  The product generates them on the GPU
(rng.cu); the checker here is numpy itself, bit for bit.
"""
import math
import random

import numpy as np
import pytest

from paper_1507_05593_b200 import _lib
from paper_1507_05593_b200 import engine as E


def _numpy_states(seed):
    st = np.random.PCG64(seed).state["state"]
    m = (1 << 64) - 1
    return [st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m]


def test_block_seed_and_pcg64_state_match_numpy():
    keys = [(0, 0, j) for j in range(64)] + [(0, 1, 17, 3), (5, 1, 2**33, 0), (2**63 + 5, 0, 7),
                                             (123456789,), (0,), (1, 0)]
    seeds, states = E.pcg64_block_states(keys)
    for k, s, row in zip(keys, seeds, states):
        ref = int(np.random.SeedSequence(k).generate_state(1, np.uint64)[0])
        assert int(s) == ref, k
        assert [int(v) for v in row] == _numpy_states(ref), k
    direct = E.pcg64_seed_states(seeds)
    assert np.array_equal(direct, states)


def _host_has_fma():
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return False
    return " fma" in flags and " avx2" in flags


@pytest.mark.skipif(not _host_has_fma(), reason="libm picks its non-FMA log1p on this CPU")
def test_log1p_restatement_matches_libm():
    lib = _lib.load()
    rnd = random.Random(11)
    xs = [-(rnd.getrandbits(53) / 9007199254740992.0) for _ in range(200000)]
    xs += [math.ldexp(rnd.random(), -rnd.randrange(0, 70)) * rnd.choice((-1, 1)) for _ in range(100000)]
    xs += [0.0, -0.0, -1e-300, 1e-17, -0.5, 0.41421, -0.29289, 0.25, 1e300, 3.0]
    bad = [x for x in xs if lib.rsc_log1p_fdlibm(x) != math.log1p(x)]
    assert not bad, bad[:5]


def test_ziggurat_tables_come_from_numpy():
    import importlib.util
    import os

    from conftest import ROOT

    path = os.path.join(ROOT, "paper_1507_05593_b200", "csrc", "gen_ziggurat.py")
    spec = importlib.util.spec_from_file_location("gen_ziggurat", path)
    gz = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(gz)
    wi, ki, fi = gz.extract()
    # the quick-accept branch of numpy's ziggurat reproduces its first outputs
    raw = np.random.PCG64(99).random_raw(4096)
    z = np.random.Generator(np.random.PCG64(99)).standard_normal(3000)
    idx = (raw & np.uint64(0xFF)).astype(np.int64)
    r = raw >> np.uint64(8)
    rabs = (r >> np.uint64(1)) & np.uint64(0x000FFFFFFFFFFFFF)
    x = rabs.astype(np.float64) * wi[idx]
    x = np.where((r & np.uint64(1)) == 1, -x, x)
    quick = rabs < ki[idx]
    # the leading run of quick accepts maps draw i -> normal i
    lead = int(np.argmin(quick)) if not quick.all() else quick.size
    assert lead > 10
    assert np.array_equal(x[:lead], z[:lead])
    assert fi[0] == 1.0 and ki[1] == 0


SIZES = [1, 2, 31, 4095, 4096, 4097, 8191, 58 * 2048, 100003, 1]


def _gpu_normals(ns, states):
    import torch

    outs = [torch.full((max(n, 1),), float("nan"), dtype=torch.float64, device="cuda") for n in ns]
    work = E.normal_pcg64(states, ns, [o.data_ptr() for o in outs])
    torch.cuda.synchronize()
    del work
    return [o.cpu().numpy()[:n] for o, n in zip(outs, ns)]


@pytest.mark.gpu
def test_device_normals_bit_identical(cuda):
    keys = [(0, 0, j) for j in range(len(SIZES))]
    seeds, states = E.pcg64_block_states(keys)
    got = _gpu_normals(SIZES, states)
    for n, s, g in zip(SIZES, seeds, got):
        ref = np.random.Generator(np.random.PCG64(int(s))).standard_normal(n)
        assert np.array_equal(g.view(np.uint64), ref.view(np.uint64)), n


@pytest.mark.gpu
def test_device_normals_many_streams(cuda):
    """More streams than one launch group (400), mixed and zero sizes."""
    rng = np.random.default_rng(5)
    ns = [int(v) for v in rng.integers(0, 20000, 900)]
    ns[3] = 0
    keys = [(7, 1, j, j % 3) for j in range(len(ns))]
    seeds, states = E.pcg64_block_states(keys)
    got = _gpu_normals(ns, states)
    for n, s, g in zip(ns, seeds, got):
        ref = np.random.Generator(np.random.PCG64(int(s))).standard_normal(n)
        assert np.array_equal(g, ref)


@pytest.mark.gpu
def test_device_normals_sequential_fallbacks(cuda):
    """Force both exact fallbacks: chunk overflow and scanning too few draws."""
    lib = _lib.load()
    ns = [5000, 70000, 9000, 1]
    seeds, states = E.pcg64_block_states([(3, 0, j) for j in range(len(ns))])
    try:
        for cap, slack in ((40, 1), (160, 0), (0, 0)):
            assert lib.rsc_normal_debug_limits(cap, slack) == 0
            got = _gpu_normals(ns, states)
            for n, s, g in zip(ns, seeds, got):
                ref = np.random.Generator(np.random.PCG64(int(s))).standard_normal(n)
                assert np.array_equal(g, ref), (cap, slack, n)
    finally:
        lib.rsc_normal_debug_limits(160, 1)


@pytest.mark.gpu
def test_cfg1_sketches_bit_identical(cuda):
    """All 512 config[1] sketches (2048 x 58 each, 60.8 M normals)."""
    import torch

    from paper_1507_05593_b200.batched import block_seed

    nb, m, r = 512, 2048, 58
    seeds, states = E.pcg64_block_states([(0, 0, i) for i in range(nb)])
    assert [int(s) for s in seeds[:4]] == [block_seed(0, 0, i) for i in range(4)]
    Om = torch.empty(nb, m, r, dtype=torch.float64, device="cuda")
    work = E.normal_pcg64(states, [m * r] * nb, [Om[i].data_ptr() for i in range(nb)])
    torch.cuda.synchronize()
    del work
    host = Om.cpu().numpy()
    for i in range(nb):
        ref = np.random.Generator(np.random.PCG64(int(seeds[i]))).standard_normal((m, r))
        assert np.array_equal(host[i], ref), i
