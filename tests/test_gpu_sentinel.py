"""Missing-value sentinel edge cases (reference datamodel.py:86-104),
pinned to the reference's own outputs (tests/golden/edge_fixtures.npz, made by
tests/golden/make_edge_golden.py from pairstat.run):

* ``na_sentinel=-0.0``: presence is a BIT comparison, so -0.0 cells are
  missing while +0.0 cells (and label 0) are present -- all 7 tests;
* NaN *data* under a numeric sentinel is present data: the rank tests sort it
  after every number (ranking.py:47) and answer normally; the reference's
  Pearson feeds NaN into beta_sym_sf, whose continued fraction raises
  NonConvergence (specfun.py:108) -- the device path raises the same.

The CPU oracle is checked against the same fixtures (not marked gpu).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from conftest import bitwise_equal, max_rel, p_close, same_nan

import paper_2505_00448_b200 as ps

GOLDEN = Path(__file__).resolve().parent / "golden" / "edge_fixtures.npz"
EXACT = {"spearman": ("stat", "rho"), "chi2": ("stat", "phi", "cramers_v"), "kruskal": ("stat", "eta2"),
         "mwu": ("stat", "r")}


def _cases():
    return [str(c) for c in np.load(GOLDEN)["cases"]]


def _load(case):
    d = np.load(GOLDEN)
    test = case.split("_", 1)[1]
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    sent = float(d[f"{case}__sentinel"])
    ma = ps.make_matrix(d[f"{case}__a"], kind_a, na_sentinel=sent)
    mb = ps.make_matrix(d[f"{case}__b"], kind_b, na_sentinel=sent) if kind_b else None
    names = ("stat", "p") + ps.EFFECTS_BY_TEST[test] + ("p_bh",)
    return test, ps.TestRequest(test, names), ma, mb, {n: d[f"{case}__{n}"] for n in names}


def _compare(test, got, want, exact_all=False):
    for n, w in want.items():
        g = got[n]
        assert same_nan(g, w), (test, n)
        if exact_all or n in EXACT.get(test, ()):
            assert bitwise_equal(g, w), (test, n)
        elif n.startswith("p"):
            assert p_close(g, w), (test, n)
        else:
            assert max_rel(g, w, floor=1e-3) <= 1e-9, (test, n)


def test_fixture_sentinel_semantics():
    d = np.load(GOLDEN)
    a = d["negzero_pearson__a"]
    m = ps.make_matrix(a, "continuous", na_sentinel=-0.0)
    assert not m.present[np.signbit(a) & (a == 0)].any()
    assert m.present[~np.signbit(a) & (a == 0)].all() and (~np.signbit(a) & (a == 0)).any()


@pytest.mark.parametrize("case", _cases())
def test_oracle_matches_reference_edge(oracle, case):
    test, req, ma, mb, want = _load(case)
    _compare(test, oracle.oracle_run(req, ma, mb), want, exact_all=True)


@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases())
def test_device_matches_reference_edge(case):
    test, req, ma, mb, want = _load(case)
    _compare(test, ps.run(req, ma, mb), want)


@pytest.mark.gpu
def test_nan_data_under_numeric_sentinel_pearson_raises(oracle):
    rng = np.random.default_rng(1)
    x = rng.normal(size=(6, 80))
    x[rng.random(x.shape) < 0.1] = -99.0
    x[2, 7] = np.nan  # present data (the sentinel is -99)
    m = ps.make_matrix(x, "continuous", na_sentinel=-99.0)
    with pytest.raises(ps.NonConvergence):
        ps.run(ps.TestRequest("pearson", ("stat", "p")), m)
    with pytest.raises(oracle.OracleError):
        oracle.oracle_run(ps.TestRequest("pearson", ("stat", "p")), m)
    # the library recovers: the next call runs normally
    x = x.copy()  # make_matrix froze the array (datamodel.py:181-188)
    x[2, 7] = 0.5
    m2 = ps.make_matrix(x, "continuous", na_sentinel=-99.0)
    req = ps.TestRequest("pearson", ("stat", "p"))
    ref = oracle.oracle_run(req, m2)
    _compare("pearson", ps.run(req, m2), ref)


@pytest.mark.gpu
@pytest.mark.parametrize("test", ["ttest", "anova"])
def test_nan_data_under_numeric_sentinel_group_tests_raise(oracle, test):
    """The reference's t-test / ANOVA also reach t_sf / f_sf with a NaN
    statistic and raise NonConvergence (checked with pairstat.run)."""
    import workloads

    kind_a, _ = ps.KINDS_BY_TEST[test]
    rng = np.random.default_rng(3)
    lab = workloads.simulate(3, 60, kind_a, categories=3, na_ratio=0.1, seed=4)
    lab[np.isnan(lab)] = -99.0
    val = rng.normal(size=(4, 60))
    val[1, 5] = np.nan
    ma = ps.make_matrix(lab, kind_a, na_sentinel=-99.0)
    mb = ps.make_matrix(val, "continuous", na_sentinel=-99.0)
    req = ps.TestRequest(test, ("stat", "p"))
    with pytest.raises(oracle.OracleError):
        oracle.oracle_run(req, ma, mb)
    with pytest.raises(ps.NonConvergence):
        ps.run(req, ma, mb)
