"""Chi-squared on the B200 vs the CPU oracle (reference categorical.py:31-94).

Contingency tables are exact int8 tensor-core counts; chi2, phi and V replay
the reference's fp64 operation order and are bit-exact; p within 1e-6
relative or 1e-12 absolute; identical NaN pattern.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps

OUTS = ("stat", "p", "phi", "cramers_v")


def _check(res, ref):
    for name in OUTS:
        assert same_nan(res[name], ref[name]), name
    for name in ("stat", "phi", "cramers_v"):
        assert bitwise_equal(res[name], ref[name]), name
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("F,S,c", [(17, 200, 3), (40, 1000, 6), (25, 3000, 12)])
def test_chi2_matches_oracle(oracle, F, S, c, na):
    raw = workloads.simulate(F, S, "categorical", categories=c, na_ratio=na, seed=F * S + c)
    mat = ps.make_matrix(raw, "categorical")
    req = ps.TestRequest("chi2", OUTS)
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


def test_chi2_mixed_level_counts_and_degenerate(oracle):
    rng = np.random.default_rng(4)
    S = 500
    rows = []
    for k in [1, 2, 2, 3, 5, 8, 10, 4]:
        rows.append(rng.integers(0, k, size=S).astype(float))
    raw = np.array(rows)
    raw[rng.random(raw.shape) < 0.2] = np.nan
    raw[3, :] = np.nan          # empty feature: c = 0
    raw[4, raw[4] == 2] = 3     # level 2 never observed -> empty declared level
    mat = ps.make_matrix(raw, "categorical")
    req = ps.TestRequest("chi2", OUTS)
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


def test_chi2_dichotomous_input(oracle):
    raw = workloads.simulate(30, 400, "dichotomous", na_ratio=0.2, seed=9)
    mat = ps.make_matrix(raw, "dichotomous")
    req = ps.TestRequest("chi2", OUTS)
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


def test_chi2_label_out_of_range():
    raw = np.array([[0.0, 1.0, 2.0, 1.0], [1.0, 0.0, 1.0, 0.0]])
    good = ps.make_matrix(raw, "categorical")
    bad = ps.DataMatrix(values=good.values, na_sentinel=good.na_sentinel, kind="categorical",
                        category_counts=np.array([2, 2]), present=good.present)
    with pytest.raises(ps.LabelOutOfRange, match="category range"):
        ps.run(ps.TestRequest("chi2", ("stat",)), bad)


def test_chi2_config3_slice(oracle):
    c = workloads.config(3, scale=0.1)
    mat = ps.make_matrix(c["a"], "categorical", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("chi2", OUTS)
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


@pytest.mark.parametrize("mc,phases", [("1", None), ("1", "3"), ("0", None)])
@pytest.mark.parametrize("F", [150, 200])
def test_chi2_cluster_pairs(oracle, monkeypatch, mc, phases, F):
    """Contingency tables from the 2-CTA cluster GEMM (tile pairs sharing a
    multicast operand, an unpaired tile with a dummy partner) equal the
    single-CTA stream-K GEMM's and the oracle's, for any number of K phases.
    10 levels per feature: F = 150 -> 6 tile rows (three leftover tiles: one
    column pair, one dummy partner), F = 200 -> 8 tile rows (two column pairs)."""
    monkeypatch.setenv("PS_CHI2_MC", mc)
    if phases:
        monkeypatch.setenv("PS_CHI2_PHASES", phases)
    raw = workloads.simulate(F, 3000, "categorical", categories=10, na_ratio=0.15, seed=F + 1)
    mat = ps.make_matrix(raw, "categorical")
    req = ps.TestRequest("chi2", OUTS)
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))
