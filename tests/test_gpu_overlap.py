"""run() with compute overlapped with the input upload vs the upload-then-compute
order (PS_NO_OVERLAP=1), on inputs large enough to be staged in several
chunks.  The incremental launches change only which CTA computes a cell and
when, so Pearson, Spearman, Kruskal-Wallis and Mann-Whitney are bitwise equal;
ANOVA / t-test moments are split over K per uploaded column window, so they
agree to the floating-point tolerance of the parity bar (and with the oracle).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, max_rel, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps

OUTS = {
    "pearson": ("stat", "p", "r2", "p_bh"),
    "spearman": ("stat", "p", "rho", "p_bonferroni", "p_bh"),
    "kruskal": ("stat", "p", "eta2", "p_bh"),
    "mwu": ("stat", "p", "r"),
    "anova": ("stat", "p", "partial_eta2", "p_bh"),
    "ttest": ("stat", "p", "cohens_d"),
}


def _inputs(test):
    if test == "pearson":
        a = workloads.simulate(3200, 1500, "continuous", na_ratio=0.1, seed=41)
        a[7] = np.round(a[7], 2)
        return ps.make_matrix(a, "continuous"), None
    if test == "spearman":
        a = workloads.simulate(520, 6000, "continuous", na_ratio=0.15, seed=42)
        a[3] = np.round(a[3], 1)  # ties
        return ps.make_matrix(a, "continuous"), None
    kind = "dichotomous" if test in ("mwu", "ttest") else "categorical"
    lab = workloads.simulate(24, 6000, kind, categories=5, na_ratio=0.1, seed=43)
    val = workloads.simulate(700, 6000, "continuous", na_ratio=0.1, seed=44)
    val[5] = np.round(val[5], 1)
    return ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")


@pytest.mark.parametrize("test", sorted(OUTS))
def test_overlapped_run_matches_sequential(test, monkeypatch):
    ma, mb = _inputs(test)
    req = ps.TestRequest(test, OUTS[test])
    monkeypatch.delenv("PS_NO_OVERLAP", raising=False)
    got = ps.run(req, ma, mb)
    monkeypatch.setenv("PS_NO_OVERLAP", "1")
    want = ps.run(req, ma, mb)
    exact = test not in ("anova", "ttest")
    for name in OUTS[test]:
        g, w = got[name], want[name]
        assert same_nan(g, w), (test, name)
        if exact:
            assert bitwise_equal(g, w), (test, name)
        elif name.startswith("p"):
            assert p_close(g, w), (test, name)
        else:
            assert max_rel(g, w, floor=1e-300) <= 1e-9, (test, name)
