"""Spearman on the B200 vs the CPU oracle (reference continuous.py:128-203).

rho is bit-exact (exact integer rank sums, survey Appendix B); p within 1e-6
relative or 1e-12 absolute; identical NaN pattern.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps


def _check(res, ref):
    for name in ("stat", "p", "rho"):
        assert same_nan(res[name], ref[name]), name
    assert bitwise_equal(res["stat"], ref["stat"])
    assert bitwise_equal(res["rho"], ref["rho"])
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("F,S", [(17, 200), (40, 1000), (33, 5000)])
def test_spearman_matches_oracle(oracle, F, S, na):
    raw = workloads.simulate(F, S, "continuous", na_ratio=na, seed=F + S + int(na * 100))
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("spearman", ("stat", "p", "rho"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


@pytest.mark.parametrize("S", [300, 2500, 12000, 25000, 40000, 50000])
def test_spearman_ties_and_blocks(oracle, S):
    rng = np.random.default_rng(S)
    x = workloads.config_spearman_like(rng, 24, S)
    x[3] = np.round(x[3])          # heavy ties
    x[4, :] = 1.5                  # constant -> NaN row
    x[5, : S // 2] = -0.0          # signed zeros tie with +0.0
    x[5, S // 2:] = 0.0
    x[6] = np.where(rng.random(S) < 0.5, 1.0, 2.0)  # two huge tie groups
    mat = ps.make_matrix(x, "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("spearman", ("stat", "p", "rho"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


def test_spearman_small_degenerate(oracle):
    nan = np.nan
    raw = np.array([
        [0.0, 1.0, nan, nan, nan],
        [5.0, 3.0, nan, nan, nan],
        [1.0, 2.0, 3.0, 4.0, 5.0],
        [2.0, 4.0, 5.0, 7.0, 9.0],
        [nan, nan, nan, nan, 1.0],
        [3.0, 3.0, 3.0, 3.0, 3.0],
    ])
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("spearman", ("stat", "p", "rho"))
    res = ps.run(req, mat)
    _check(res, oracle.oracle_run(req, mat))
    assert res["stat"][0, 1] == -1.0 and np.isnan(res["p"][0, 1])   # two samples
    assert res["stat"][2, 3] == 1.0 and res["p"][2, 3] == 0.0       # perfect monotone


def test_spearman_numeric_sentinel_with_nan_data(oracle):
    """NaN data under a numeric sentinel is present and never ties (quirk)."""
    rng = np.random.default_rng(5)
    x = rng.normal(size=(6, 50))
    x[0, [3, 9]] = np.nan
    x[x > 1.8] = -99.0
    mat = ps.make_matrix(x, "continuous", na_sentinel=-99.0)
    req = ps.TestRequest("spearman", ("stat", "rho"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    assert bitwise_equal(res["stat"], ref["stat"])


def test_spearman_config2_slice(oracle):
    c = workloads.config(2, scale=0.12)
    mat = ps.make_matrix(c["a"], "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("spearman", ("stat", "p", "p_bh", "rho"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    _check(res, ref)
    assert same_nan(res["p_bh"], ref["p_bh"])
    assert p_close(res["p_bh"], ref["p_bh"], rtol=2e-6)
    assert bitwise_equal(res["p_bh"], oracle.adjust(res["p"], "bh", True))


@pytest.mark.parametrize("S", [500, 6000, 20000])
def test_spearman_keys_equal_in_high_bits(oracle, S):
    """Values that agree in their high 32 bits but differ below: the presort
    orders on the high half first, then repairs short colliding runs and
    re-sorts features with long ones on the full key."""
    rng = np.random.default_rng(S + 7)
    x = workloads.config_spearman_like(rng, 10, S)
    x[1] = 1.0 + rng.integers(0, 1000, S) * 2.0**-40        # one long colliding run
    x[2] = np.round(x[2], 1) + rng.integers(0, 3, S) * 2.0**-45  # many short runs
    x[3] = -1.0 - rng.integers(0, 50, S) * 2.0**-38          # negative keys
    x[4, ::3] = 0.0
    x[4, 1::3] = -0.0
    x[5, ::7] = np.nan                                      # NaN values as data
    mat = ps.make_matrix(x, "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("spearman", ("stat", "p", "rho"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))
