"""The work census (paper_1507_05593_b200/census.py) against the
oracle restatement instrumented operation by operation (oracle/numeric.py COUNT):
equal per category on exact, compressed, diagonal-tree and elasticity instances."""
import pytest

from factor_cases import load_case


@pytest.mark.parametrize("name", ["l3d8_small", "l3d12", "el5", "el7"])
def test_census_matches_instrumented_oracle(name):
    from oracle import numeric as on
    from paper_1507_05593_b200.census import census
    from paper_1507_05593_b200.symbolic import analyze

    A, coords, knobs, _ = load_case(name)
    cfg = on.Config(**knobs)
    plan = analyze(A, cfg.tau_o, cfg.tau_d, cfg.interior_blocks, coords=coords)
    on.COUNT = {}
    try:
        F = on.factorize(A, cfg, coords=coords, plan=plan)
        ref = dict(on.COUNT)
    finally:
        on.COUNT = None
    C = census(plan, cfg, F.ranks, F.stats["alpha_d_final"])
    for k, v in C.items():
        assert abs(ref.get(k, 0.0) - v) <= 1e-9 * max(1.0, abs(v)), (k, ref.get(k), v)
    assert set(ref) <= set(C)


def test_census_cfg0_total_matches_survey():
    """Config[0] (nothing compressed): 1.44 GFLOP in SURVEY §8(d)."""
    from oracle import numeric as on
    from paper_1507_05593_b200.census import census
    from paper_1507_05593_b200.symbolic import analyze

    A, coords, knobs, _ = load_case("cfg0")
    cfg = on.Config(**knobs)
    plan = analyze(A, cfg.tau_o, cfg.tau_d, cfg.interior_blocks, coords=coords)
    tot = sum(census(plan, cfg, {}).values())
    assert abs(tot / 1e9 - 1.44) < 0.01 * 1.44
