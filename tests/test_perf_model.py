"""SPEC perf module and acceptance criteria 1-2:
the paper's cost model and Amdahl numbers."""

import math

import pytest

from paper_1801_02362_b200 import perf
from paper_1801_02362_b200.errors import ConfigError


def test_cost_model_paper_numbers():
    m = perf.CostModel(N=2120, M=50, L=50, K=3000)
    assert perf.original_cost(m) == pytest.approx(91.4, abs=1e-12)
    assert perf.close_cost(m) == pytest.approx(1.7067, abs=1e-4)
    assert perf.msd_speedup(m) == pytest.approx(53.6, abs=0.1)
    m2 = perf.CostModel(N=512, M=0, L=1, K=10000)
    assert perf.original_cost(m2) == 512 and perf.close_cost(m2) == pytest.approx(1.0512)
    assert perf.msd_speedup(m2) == pytest.approx(487.1, abs=0.5)
    r = perf.model_report(2120, 50, 50, 3000, p=0.43)
    assert r["amdahl"] == pytest.approx(1.73, abs=0.02) and r["accelerates"]


def test_amdahl_table1():
    assert perf.amdahl(0.93, 488) == pytest.approx(13.9, abs=0.1)
    assert perf.amdahl(0.43, 54) == pytest.approx(1.73, abs=0.02)
    assert perf.amdahl(0.0, 7.0) == 1.0
    assert perf.amdahl(0.6, 1e9) == pytest.approx(1.0 / 0.4, rel=1e-6)
    with pytest.raises(ConfigError):
        perf.amdahl(0.5, 0.0)


def test_acceleration_condition_and_monotonicity():
    assert perf.accelerates(perf.CostModel(N=100, M=0, L=1, K=1000))
    assert not perf.accelerates(perf.CostModel(N=100, M=1, L=10 ** 6, K=1))
    # equality is not acceleration: M + (N - M)/L == 1 + N/K
    assert not perf.accelerates(perf.CostModel(N=10, M=0, L=5, K=10))  # 2 vs 2
    prev = 0.0
    for K in (1, 10, 100, 1000):
        s = perf.msd_speedup(perf.CostModel(N=500, M=20, L=10, K=K))
        assert s > prev
        prev = s
    prev = math.inf
    for L in (1, 5, 50):
        s = perf.msd_speedup(perf.CostModel(N=500, M=20, L=L, K=100))
        assert s < prev
        prev = s
    with pytest.raises(ConfigError):
        perf.CostModel(N=10, M=11)


def test_measured_vs_model_identity():
    class Rep:
        steps, mode, expensive_count, reassign_count, measured_K = 400, "close", 400 + 7 * 16, 7, 400 / 7

    d = perf.measured_vs_model(Rep, N=16)
    assert d["difference"] == 0.0

    class Orig:
        steps, mode, expensive_count, reassign_count, measured_K = 400, "original", 400 * 16, 0, math.inf

    assert perf.measured_vs_model(Orig, N=16)["difference"] == 0.0
