"""Scaling-study metric definitions against the reference's own test values
(tests/test_bench.cpp:12-130, acceptance.cpp:278-304)."""
import pytest

from paper_2007_06048_b200 import scaling as S
from paper_2007_06048_b200._lib import ConfigError


def test_cd_cost_matches_reference_hand_count():
    c = S.count_stencil_cost("acoustic_iso_cd", 1)          # test_bench.cpp:12-19
    assert c.flops_per_point == 3 * 5 + 2 + 6
    assert c.bytes_per_point == 16
    assert c.arithmetic_intensity == pytest.approx(23.0 / 16.0, rel=1e-12)
    r4 = S.count_stencil_cost("acoustic_iso_cd", 4)
    assert r4.flops_per_point - c.flops_per_point == 3 * 3 * 5   # test_bench.cpp:21-26
    assert r4.flops_per_point == 68
    assert S.count_stencil_cost("acoustic_iso", 4).bytes_per_point == 40
    assert (S.count_stencil_cost("acoustic_iso", 4).flops_per_point >
            S.count_stencil_cost("acoustic_iso", 2).flops_per_point)
    with pytest.raises(ConfigError):
        S.count_stencil_cost("acoustic_iso_cd", 0)


def test_weak_scaling_plans():
    ideal = S.weak_scaling_plan(1000, [1, 2, 4], "ideal")         # test_bench.cpp:50-66
    assert [n for _, n in ideal] == [(1000, 1000, 1000), (2000, 1000, 1000), (4000, 1000, 1000)]
    prac = S.weak_scaling_plan(1000, [1, 2, 4, 6], "practical")
    assert [n[0] for _, n in prac] == [1000, 1280, 1600, 1856]
    with pytest.raises(ConfigError):
        S.weak_scaling_plan(0, [1, 2])
    with pytest.raises(ConfigError):
        S.weak_scaling_plan(1000, [1, 0])


def _run(r, n, t):
    return S.ScalingRun(ranks=r, n=n, nsteps=10, kernel_s=t, modeling_s=1.1 * t,
                        points_per_s=n[0] * n[1] * n[2] * 10 / t)


def test_strong_and_weak_efficiency():
    res = S.ScalingResult("strong", [_run(8, (1000,) * 3, 80.0), _run(256, (1000,) * 3, 4.0)])
    S.compute_efficiency(res)                                       # test_bench.cpp:84-92
    assert res.runs[0].efficiency_pct == pytest.approx(100.0, rel=1e-9)
    assert res.runs[1].efficiency_pct == pytest.approx(62.5, rel=1e-9)
    w = S.ScalingResult("weak_practical", [_run(1, (1000, 1000, 1000), 50.0),
                                          _run(2, (2000, 1000, 1000), 50.0),
                                          _run(4, (4000, 1000, 1000), 62.5)])
    S.compute_efficiency(w)                                         # test_bench.cpp:94-106
    assert [r.efficiency_pct for r in w.runs] == pytest.approx([100.0, 100.0, 80.0], rel=1e-9)


def test_failed_runs_and_executor():
    res = S.ScalingResult("strong", [_run(1, (64,) * 3, 8.0), _run(2, (64,) * 3, 4.0)])
    res.runs[1].ok = False
    res.runs[1].kernel_s = 0.0
    S.compute_efficiency(res)                                       # test_bench.cpp:118-127
    assert res.runs[0].efficiency_pct == pytest.approx(100.0)
    assert res.runs[1].efficiency_pct == 0.0
    seen = []

    def ex(n, ranks):
        seen.append((ranks, n))
        if ranks == 4:
            raise RuntimeError("boom")
        return 8.0 / ranks, 9.0 / ranks

    out = S.run_scaling([(1, (32,) * 3), (2, (32,) * 3), (4, (32,) * 3)], 7, "strong", ex)
    assert seen == [(1, (32,) * 3), (2, (32,) * 3), (4, (32,) * 3)]
    assert out.runs[1].efficiency_pct == pytest.approx(100.0)
    assert not out.runs[2].ok and out.runs[2].error == "boom"
