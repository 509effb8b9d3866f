"""Pearson on the B200 vs the CPU oracle (reference continuous.py:29-103).

Tolerances (north star): |dr| <= 1e-9 * max(|r|, 1e-3); p within 1e-6 relative
or 1e-12 absolute; identical NaN pattern; r2 follows r.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import max_rel, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps


def _check(res, ref):
    for name in ("stat", "p", "r2"):
        assert same_nan(res[name], ref[name]), name
    r, rr = res["stat"], ref["stat"]
    m = ~np.isnan(rr)
    assert np.all(np.abs(r[m] - rr[m]) <= 1e-9 * np.maximum(np.abs(rr[m]), 1e-3))
    assert p_close(res["p"], ref["p"])
    np.testing.assert_array_equal(res["stat"], res["stat"].T)


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("F,S", [(17, 200), (70, 333), (130, 1000)])
def test_pearson_matches_oracle(oracle, F, S, na):
    raw = workloads.simulate(F, S, "continuous", na_ratio=na, seed=F * 7 + S + int(na * 10))
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p", "r2"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    _check(res, ref)


def test_pearson_degenerate_rows(oracle):
    rng = np.random.default_rng(3)
    raw = rng.normal(size=(12, 40))
    raw[0] = 0.1                      # constant whose mean does not round back to 0.1
    raw[1] = 3.0                      # exact constant
    raw[2, 2:] = np.nan               # n = 2 with everyone
    raw[3, :] = np.nan                # all missing
    raw[4, 1:] = np.nan               # single sample
    raw[5] = raw[6]                   # perfectly correlated pair
    raw[7] = -raw[6] * 2 + 1          # perfectly anti-correlated
    raw[8, ::2] = 5.0                 # constant on half the samples
    raw[9, 1::2] = np.nan
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p", "r2"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    _check(res, ref)
    # diagonal of a non-constant variable: r = 1, p = 0 (test_engine.py:137-144)
    assert res["stat"][6, 6] == 1.0 and res["p"][6, 6] == 0.0


def test_pearson_numeric_sentinel_and_orientation(oracle):
    rng = np.random.default_rng(11)
    raw = rng.normal(size=(300, 25))  # samples x features
    raw[rng.random(raw.shape) < 0.2] = -99.0
    mat = ps.make_matrix(raw, "continuous", na_sentinel=-99.0, features_on_rows=False)
    req = ps.TestRequest("pearson", ("stat", "p", "p_bonferroni", "p_bh", "p_by", "r2"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    _check(res, ref)
    for name in ("p_bonferroni", "p_bh", "p_by"):
        assert same_nan(res[name], ref[name])
        # adjusted values differ from the oracle's only through the raw p
        assert max_rel(res[name], ref[name]) <= 2e-6


def test_pearson_config1(oracle):
    c = workloads.config(1)
    mat = ps.make_matrix(c["a"], "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("pearson", ("stat", "p", "p_bonferroni", "p_bh"))
    res = ps.run(req, mat)
    ref = oracle.oracle_run(req, mat)
    assert same_nan(res["stat"], ref["stat"])
    r, rr = res["stat"], ref["stat"]
    m = ~np.isnan(rr)
    assert np.all(np.abs(r[m] - rr[m]) <= 1e-9 * np.maximum(np.abs(rr[m]), 1e-3))
    assert p_close(res["p"], ref["p"])


def test_pearson_config5_recipe_full_sample_count(oracle):
    """Config-5 generator and missingness at its FULL sample count (10^5):
    300 features x 10^5 samples, every pair checked against the oracle (the
    k-loop length is what stresses the fp64 contraction's summation order)."""
    import workloads as wl

    rng = np.random.default_rng([wl.SEED_BASE, 5, 1])
    x = wl._mcar(rng, wl._latent(rng, 300, 100000), 0.30)
    mat = ps.make_matrix(x, "continuous", na_sentinel=wl.SENTINEL)
    req = ps.TestRequest("pearson", ("stat", "p", "r2"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


@pytest.mark.parametrize("mode", ["0", "2"])
def test_operand_modes_bit_identical(monkeypatch, mode):
    """Pre-centred operands (default: x' computed once per element) are the
    tile loop's own fp64 subtraction done ahead: every output bit equals the
    other variants (PS_PEARSON_MODE=0 raw values, 2 x' and x'^2 precomputed)."""
    x = workloads.simulate(300, 2000, "continuous", na_ratio=0.2, seed=123)
    x[5] = 7.25  # constant row: replay path
    mat = ps.make_matrix(x, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p", "r2", "p_bh"))
    want = ps.run(req, mat)
    monkeypatch.setenv("PS_PEARSON_MODE", mode)
    got = ps.run(req, mat)
    for n in req.outputs:
        assert np.array_equal(got[n].view(np.uint64), want[n].view(np.uint64)), n
