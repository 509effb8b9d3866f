"""Parity at the FULL BASELINE sizes (configs 1-4 and the config-5 Spearman leg).

The device computes the whole config through ``run``; the CPU oracle
recomputes sampled row ranges of it (the oracle takes the reference's
(lo, hi) partitions, so a few triangle rows / label rows / continuous
features cost seconds), and the full matrices are checked for the
size-independent properties of the outputs: symmetry, value ranges, NaN
diagonal of adjusted matrices, Bonferroni = min(1, m p) and BH monotone
(p <= p_bh <= p_bonferroni).  The adjusted matrices are compared by VALUE:
bit for bit with the oracle's adjustment of the device p, and (configs 1-4,
where the whole oracle run takes seconds) within the p tolerance of the
oracle's own end-to-end adjusted matrices.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, max_rel, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps

EXACT = {"spearman": ("stat", "rho"), "chi2": ("stat", "phi", "cramers_v"), "kruskal": ("stat", "eta2"),
         "mwu": ("stat", "r")}
OUTS = {"pearson": ("stat", "p", "r2", "p_bonferroni", "p_bh"), "spearman": ("stat", "p", "rho", "p_bonferroni", "p_bh"),
        "chi2": ("stat", "p", "phi", "cramers_v"), "anova": ("stat", "p", "partial_eta2", "p_bh"),
        "ttest": ("stat", "p", "cohens_d"), "kruskal": ("stat", "p", "eta2", "p_bh"),
        "mwu": ("stat", "p", "r")}


def _inputs(cfg_key, test):
    cfg = workloads.config(cfg_key)
    a, b = cfg["a"], cfg["b"]
    kind_a, kind_b = cfg["kind_a"], cfg["kind_b"]
    if test in ("ttest", "mwu"):
        a = np.ascontiguousarray(a[cfg["two_level_rows"]])
        kind_a = "dichotomous"
    ma = ps.make_matrix(a, kind_a, na_sentinel=workloads.SENTINEL)
    mb = ps.make_matrix(b, kind_b, na_sentinel=workloads.SENTINEL) if b is not None else None
    return ma, mb


def _rows(n, k=3):
    return sorted({0, n // 2, n - 1})[:k]


@pytest.mark.parametrize("cfg_key,test", [(1, "pearson"), (2, "spearman"), (3, "chi2"), (4, "anova"),
                                          (4, "ttest"), (4, "kruskal"), (4, "mwu"), ("5s", "spearman")])
def test_full_size_against_oracle_rows(oracle, cfg_key, test):
    ma, mb = _inputs(cfg_key, test)
    req = ps.TestRequest(test, OUTS[test])
    res = ps.run(req, ma, mb)
    homog = mb is None
    shape = res.shape
    # sampled ranges: triangle rows (homogeneous), label rows (ttest/anova: flat
    # cells of a row), continuous features (mwu/kruskal)
    if homog:
        ranges = [(r, r + 1) for r in _rows(shape[0])]
    elif test in ("ttest", "anova"):
        ranges = [(g * shape[1], (g + 1) * shape[1]) for g in _rows(shape[0])]
    else:
        ranges = [(h, h + 1) for h in _rows(shape[1])]
    canonical = ("stat", "p") + ps.EFFECTS_BY_TEST[test]
    want_names = [n for n in canonical if n in req.outputs]
    for lo, hi in ranges:
        ref = oracle.compute(test, ma, mb, wanted=set(want_names), lo=lo, hi=hi)
        if homog:
            sel = (slice(lo, hi), slice(lo, None))
        elif test in ("ttest", "anova"):
            g = lo // shape[1]
            sel = (slice(g, g + 1), slice(None))
        else:
            sel = (slice(None), slice(lo, hi))
        for name in want_names:
            got, exp = res[name][sel], ref[name][sel]
            assert same_nan(got, exp), (test, name, lo)
            if name in EXACT.get(test, ()):
                assert bitwise_equal(got, exp), (test, name, lo)
            elif name == "p":
                assert p_close(got, exp), (test, name, lo)
            else:
                assert max_rel(got, exp, floor=1e-300) <= 1e-9, (test, name, lo)
    # size-independent properties of the full matrices
    stat, p = res["stat"], res["p"]
    fin = ~np.isnan(p)
    assert ((p[fin] >= 0.0) & (p[fin] <= 1.0)).all()
    if homog:
        assert bitwise_equal(stat, stat.T) and bitwise_equal(p, p.T)
    if test in ("pearson", "spearman"):
        s = stat[~np.isnan(stat)]
        assert ((s >= -1.0) & (s <= 1.0)).all()
    if "p_bonferroni" in req.outputs:
        pb = res["p_bonferroni"]
        iu = np.triu_indices(shape[0], 1)
        fam = p[iu]
        m = np.count_nonzero(~np.isnan(fam))
        exp_b = np.minimum(1.0, m * fam)
        assert bitwise_equal(pb[iu], exp_b)
        assert np.isnan(np.diag(pb)).all()
    # adjusted matrices: bit for bit the oracle's adjust (adjust.py:46-87) of
    # the device p, and -- where the whole oracle run takes seconds -- within
    # the p-value tolerance of the oracle's end-to-end adjusted matrices
    adj_names = [n for n in ("p_bonferroni", "p_bh") if n in req.outputs]
    for n in adj_names:
        method = {"p_bonferroni": "bonferroni", "p_bh": "bh"}[n]
        assert bitwise_equal(res[n], oracle.adjust(p, method, homog)), (test, n)
    if adj_names and cfg_key != "5s":
        ref_p = oracle.compute(test, ma, mb, wanted={"p"})["p"]
        for n in adj_names:
            method = {"p_bonferroni": "bonferroni", "p_bh": "bh"}[n]
            want = oracle.adjust(ref_p, method, homog)
            assert same_nan(res[n], want), (test, n)
            assert p_close(res[n], want, rtol=2e-6), (test, n)
    if "p_bh" in req.outputs:
        bh = res["p_bh"]
        if homog:
            iu = np.triu_indices(shape[0], 1)
            q, pp = bh[iu], p[iu]
        else:
            q, pp = bh.ravel(), p.ravel()
        ok = ~np.isnan(pp)
        assert same_nan(q, pp)
        assert (q[ok] >= pp[ok]).all() and (q[ok] <= 1.0).all()
        # monotone in p: sorting by p sorts the adjusted values
        order = np.argsort(pp[ok], kind="stable")
        assert (np.diff(q[ok][order]) >= 0).all()
