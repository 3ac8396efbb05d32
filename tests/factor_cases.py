"""Instances of tests/golden/factor_*.npz (mirrors make_golden.FACTOR_CASES)."""
INF = float("inf")
KNOBS = dict(tau_o=32, oversample=10, alpha_o=1.0, alpha_d=0.5, tau_d=256, power_iters=1, seed=0,
             interior_blocks=True, max_restarts=10)
CASES = {
    "l2d16_exact": ("laplacian_2d", (16,), False, dict(tau_o=INF), True),
    "l3d8_small": ("laplacian_3d", (8,), False, dict(tau_o=16, tau_d=32, oversample=4), True),
    "l3d12": ("laplacian_3d", (12,), False, dict(tau_d=64), True),
    "l3d16": ("laplacian_3d", (16,), False, dict(tau_d=64), False),
    "el5": ("elasticity_3d", (5,), True, dict(tau_o=16, tau_d=32, oversample=4), True),
    "el7": ("elasticity_3d", (7,), True, dict(tau_d=64), False),
    "cfg0": ("laplacian_2d", (128,), False, dict(), False),
    "l3d24": ("laplacian_3d", (24,), False, dict(), False),
    "l3d16_noint": ("laplacian_3d", (16,), False, dict(tau_d=64, interior_blocks=False), False),
    "l3d20_td32": ("laplacian_3d", (20,), False, dict(tau_o=16, tau_d=32, oversample=4), False),
    "el9_td48": ("elasticity_3d", (9,), True, dict(tau_o=24, tau_d=48, oversample=6), False),
}


def load_case(name):
    from paper_1507_05593_b200 import problems as P

    gen, args, strip, over, keep_dense = CASES[name]
    kw = {"strip_zeros": True} if strip else {}
    A, coords = getattr(P, gen)(*args, **kw)
    return A, coords, dict(KNOBS, **over), keep_dense
