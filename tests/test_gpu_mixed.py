"""ANOVA / t-test (moment contraction) and Kruskal-Wallis / Mann-Whitney U
(label-filtered rank walks) on the B200 vs the CPU oracle
(reference mixed.py:121-663).

ANOVA F / eta^2 and t / d: |rel| <= 1e-9; KW H, MWU U and r: bit-exact (exact
rank sums replayed in the reference's op order); p within 1e-6 relative or
1e-12 absolute; identical NaN pattern.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, max_rel, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps


def _inputs(test, Fc, Fq, S, na, seed, c=4):
    kind = ps.KINDS_BY_TEST[test][0]
    a = workloads.simulate(Fc, S, kind, categories=c, na_ratio=na, seed=seed)
    b = workloads.simulate(Fq, S, "continuous", na_ratio=na, seed=seed + 1)
    return ps.make_matrix(a, kind), ps.make_matrix(b, "continuous")


def _check_moment(res, ref, names):
    for name in names:
        assert same_nan(res[name], ref[name]), name
    assert max_rel(res["stat"], ref["stat"], floor=1e-300) <= 1e-9
    assert max_rel(res[names[-1]], ref[names[-1]], floor=1e-300) <= 1e-9
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("variant", ["student", "welch"])
def test_ttest_matches_oracle(oracle, na, variant):
    a, b = _inputs("ttest", 12, 70, 300, na, seed=int(na * 100) + 3)
    req = ps.TestRequest("ttest", ("stat", "p", "cohens_d"), t_variant=variant)
    _check_moment(ps.run(req, a, b), oracle.oracle_run(req, a, b), ("stat", "p", "cohens_d"))


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("c", [2, 3, 7, 30])
def test_anova_matches_oracle(oracle, na, c):
    a, b = _inputs("anova", 12, 90, 400, na, seed=int(na * 100) + c, c=c)
    req = ps.TestRequest("anova", ("stat", "p", "partial_eta2"))
    _check_moment(ps.run(req, a, b), oracle.oracle_run(req, a, b), ("stat", "p", "partial_eta2"))


def test_moment_degenerate_cases(oracle):
    nan = np.nan
    lab = np.array([
        [0, 0, 1, 1, 0, 1, nan, 0],
        [0, 0, 0, 0, 1, 1, 1, 1],
        [0, 1, 0, 1, 0, 1, 0, 1],
    ], dtype=float)
    val = np.array([
        [2.0, 2.0, 5.0, 5.0, 2.0, 5.0, 1.0, 2.0],    # zero within-group variance, unequal means
        [3.0, 3.0, 3.0, 3.0, 3.0, 3.0, 3.0, 3.0],    # all equal
        [0.1, 0.1, 0.1, 0.2, 0.1, 0.2, 0.1, 0.2],    # near-degenerate, rounding-sensitive
        [1.0, 2.0, 4.0, 7.0, nan, nan, nan, 3.0],
    ])
    for test, kind in (("anova", "categorical"), ("ttest", "dichotomous")):
        a = ps.make_matrix(lab, kind)
        b = ps.make_matrix(val, "continuous")
        outs = ("stat", "p", ps.EFFECTS_BY_TEST[test][0])
        for variant in ("student", "welch"):
            req = ps.TestRequest(test, outs, t_variant=variant)
            res = ps.run(req, a, b)
            ref = oracle.oracle_run(req, a, b)
            for name in outs:
                assert same_nan(res[name], ref[name]), (test, name)
                m = ~np.isnan(ref[name])
                np.testing.assert_allclose(res[name][m], ref[name][m], rtol=1e-9)


def test_anova_config4_slice(oracle):
    c = workloads.config(4, scale=0.05)
    a = ps.make_matrix(c["a"], "categorical", na_sentinel=workloads.SENTINEL)
    b = ps.make_matrix(c["b"], "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("anova", ("stat", "p", "partial_eta2", "p_bh"))
    res = ps.run(req, a, b)
    ref = oracle.oracle_run(req, a, b)
    _check_moment(res, ref, ("stat", "p", "partial_eta2"))
    assert same_nan(res["p_bh"], ref["p_bh"])
    assert p_close(res["p_bh"], ref["p_bh"], rtol=2e-6)
    assert bitwise_equal(res["p_bh"], oracle.adjust(res["p"], "bh", False))


def test_anova_label_out_of_range():
    lab = np.array([[0.0, 1.0, 2.0, 1.0]])
    val = np.array([[1.0, 2.0, 3.0, 4.0]])
    good = ps.make_matrix(lab, "categorical")
    bad = ps.DataMatrix(values=good.values, na_sentinel=good.na_sentinel, kind="categorical",
                        category_counts=np.array([2]), present=good.present)
    with pytest.raises(ps.LabelOutOfRange, match="category range"):
        ps.run(ps.TestRequest("anova", ("stat",)), bad, ps.make_matrix(val, "continuous"))


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("c", [2, 3, 8, 13, 20, 60])
def test_kruskal_matches_oracle(oracle, na, c):
    a, b = _inputs("kruskal", 12, 60, 400, na, seed=int(na * 100) + c, c=c)
    req = ps.TestRequest("kruskal", ("stat", "p", "eta2"))
    res = ps.run(req, a, b)
    ref = oracle.oracle_run(req, a, b)
    for name in ("stat", "p", "eta2"):
        assert same_nan(res[name], ref[name]), name
    assert bitwise_equal(res["stat"], ref["stat"])
    assert bitwise_equal(res["eta2"], ref["eta2"])
    assert p_close(res["p"], ref["p"])


def test_kruskal_mixed_level_counts(oracle):
    """Label features with 2..200 levels in one matrix (k > 16 takes the
    shared-accumulator walk for every feature)."""
    rows = [workloads.simulate(1, 600, "categorical", categories=c, na_ratio=0.2, seed=c)
            for c in (2, 5, 17, 40, 200)]
    a = ps.make_matrix(np.vstack(rows), "categorical")
    b = ps.make_matrix(workloads.simulate(40, 600, "continuous", na_ratio=0.2, seed=5), "continuous")
    req = ps.TestRequest("kruskal", ("stat", "p", "eta2"))
    res = ps.run(req, a, b)
    ref = oracle.oracle_run(req, a, b)
    for name in ("stat", "p", "eta2"):
        assert same_nan(res[name], ref[name]), name
    assert bitwise_equal(res["stat"], ref["stat"])
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("na", [0.0, 0.1, 0.3, 0.5])
@pytest.mark.parametrize("mode", ["auto", "asymptotic"])
def test_mwu_matches_oracle(oracle, na, mode):
    a, b = _inputs("mwu", 12, 60, 400, na, seed=int(na * 100) + 17)
    req = ps.TestRequest("mwu", ("stat", "p", "r"), u_mode=mode)
    res = ps.run(req, a, b)
    ref = oracle.oracle_run(req, a, b)
    for name in ("stat", "p", "r"):
        assert same_nan(res[name], ref[name]), name
    assert bitwise_equal(res["stat"], ref["stat"])
    assert bitwise_equal(res["r"], ref["r"])
    assert p_close(res["p"], ref["p"])


def test_rank_tests_with_ties(oracle):
    rng = np.random.default_rng(8)
    S = 3000
    lab = rng.integers(0, 4, size=(9, S)).astype(float)
    lab[rng.random(lab.shape) < 0.1] = np.nan
    val = np.round(rng.normal(size=(20, S)), 1)   # heavy ties
    val[3] = 1.0                                    # all tied -> NaN rows
    val[rng.random(val.shape) < 0.15] = np.nan
    a = ps.make_matrix(lab, "categorical")
    b = ps.make_matrix(val, "continuous")
    req = ps.TestRequest("kruskal", ("stat", "p", "eta2"))
    res, ref = ps.run(req, a, b), oracle.oracle_run(req, a, b)
    assert bitwise_equal(res["stat"], ref["stat"]) and same_nan(res["p"], ref["p"])
    assert p_close(res["p"], ref["p"])
    dich = ps.make_matrix(np.where(np.isnan(lab), np.nan, (lab > 1).astype(float)), "dichotomous")
    req = ps.TestRequest("mwu", ("stat", "p", "r"))
    res, ref = ps.run(req, dich, b), oracle.oracle_run(req, dich, b)
    assert bitwise_equal(res["stat"], ref["stat"]) and bitwise_equal(res["r"], ref["r"])
    assert same_nan(res["p"], ref["p"]) and p_close(res["p"], ref["p"])


def test_mwu_exact_small_groups(oracle):
    """Exact U distribution (mixed.py:231-247) on tie-free small groups."""
    rng = np.random.default_rng(12)
    S = 40
    lab = np.zeros((6, S))
    for i, n0 in enumerate([1, 3, 5, 7, 7, 20]):
        lab[i, rng.permutation(S)[:n0]] = 1.0
    val = rng.permutation(S * 3)[: S * 4].reshape(1, -1)[:, :S].astype(float)
    val = np.vstack([val, rng.normal(size=(3, S))])
    a = ps.make_matrix(lab, "dichotomous")
    b = ps.make_matrix(val, "continuous")
    for mode in ("auto", "exact"):
        req = ps.TestRequest("mwu", ("stat", "p", "r"), u_mode=mode)
        res, ref = ps.run(req, a, b), oracle.oracle_run(req, a, b)
        assert bitwise_equal(res["stat"], ref["stat"])
        # exact p-values are ratios of exact integer counts: bit-exact; in
        # auto mode the larger groups take the normal approximation (erfc ulps)
        if mode == "exact":
            assert bitwise_equal(res["p"], ref["p"])
        else:
            assert p_close(res["p"], ref["p"])


def test_mwu_exact_errors():
    lab = np.array([[0, 0, 1, 1, 0, 1.0]])
    tied = np.array([[1.0, 1.0, 2.0, 3.0, 4.0, 5.0]])
    a = ps.make_matrix(lab, "dichotomous")
    with pytest.raises(ps.ExactModeWithTies, match="tie-free"):
        ps.run(ps.TestRequest("mwu", ("p",), u_mode="exact"), a, ps.make_matrix(tied, "continuous"))
    big_lab = (np.arange(70) % 2).astype(float).reshape(1, -1)
    big_val = np.arange(70, dtype=float).reshape(1, -1)
    with pytest.raises(ps.TableTooLarge, match="cap"):
        ps.run(ps.TestRequest("mwu", ("p",), u_mode="exact"), ps.make_matrix(big_lab, "dichotomous"),
               ps.make_matrix(big_val, "continuous"))


def test_kruskal_config4_slice(oracle):
    c = workloads.config(4, scale=0.05)
    a = ps.make_matrix(c["a"], "categorical", na_sentinel=workloads.SENTINEL)
    b = ps.make_matrix(c["b"], "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("kruskal", ("stat", "p", "eta2", "p_bh"))
    res, ref = ps.run(req, a, b), oracle.oracle_run(req, a, b)
    assert bitwise_equal(res["stat"], ref["stat"])
    assert p_close(res["p"], ref["p"]) and same_nan(res["p_bh"], ref["p_bh"])
    assert p_close(res["p_bh"], ref["p_bh"], rtol=2e-6)
    assert bitwise_equal(res["p_bh"], oracle.adjust(res["p"], "bh", False))


@pytest.mark.parametrize("test", ["kruskal", "mwu"])
def test_rank_tests_large_sample_count(oracle, test):
    """S = 50,000 (the config-5 Spearman sample count): 16-bit orders, the
    walk's shared-memory plan at its largest."""
    a, b = _inputs(test, 3, 8, 50000, 0.15, seed=77, c=5)
    req = ps.TestRequest(test, ("stat", "p"))
    res = ps.run(req, a, b)
    ref = oracle.oracle_run(req, a, b)
    assert same_nan(res["stat"], ref["stat"])
    assert bitwise_equal(res["stat"], ref["stat"])
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("test", ["anova", "ttest"])
@pytest.mark.parametrize("offset,spread", [(1000.0, 1.4), (1e4, 3.0), (50.0, 0.01)])
def test_group_moments_large_offset_large_groups(oracle, test, offset, spread):
    """Values with a large offset relative to their spread and groups of
    ~10^4 samples: the reference's one-pass ssq - sum*mean carries a rounding
    error ~sqrt(n_j) eps raw / gs, which the device must either match by
    replay or stay within 1e-9 of (advisor finding, ps_group.cu replay rule)."""
    rng = np.random.default_rng(int(offset) + 7)
    S = 30000
    kind = "categorical" if test == "anova" else "dichotomous"
    lab = workloads.simulate(6, S, kind, categories=3, na_ratio=0.05, seed=int(offset) + 1)
    val = offset + spread * rng.standard_normal((40, S))
    val[::4] += spread * 0.05 * np.nan_to_num(lab[0])  # small real group effects on some columns
    val[rng.random(val.shape) < 0.05] = np.nan
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    eff = ps.EFFECTS_BY_TEST[test]
    req = ps.TestRequest(test, ("stat", "p") + eff)
    res, ref = ps.run(req, ma, mb), oracle.oracle_run(req, ma, mb)
    for n in req.outputs:
        assert same_nan(res[n], ref[n]), n
        if n == "p":
            assert p_close(res[n], ref[n]), n
        else:
            assert max_rel(res[n], ref[n], floor=1e-300) <= 1e-9, (n, max_rel(res[n], ref[n], floor=1e-300))


@pytest.mark.parametrize("test", ["anova", "ttest"])
@pytest.mark.parametrize("S", [1000, 9000, 33001])
def test_group_replay_everywhere_bitwise(oracle, test, S):
    """Data where every cell fails the conditioning rules (offset 1e4 over
    spread 3): every statistic comes from the exact replay kernel (staged bit
    walk, ps_group.cu), which must equal the reference's one-pass order bit
    for bit -- S not a multiple of the 1024-sample round, and > 2^15."""
    rng = np.random.default_rng(91 + S)
    kind = "categorical" if test == "anova" else "dichotomous"
    lab = workloads.simulate(4, S, kind, categories=5, na_ratio=0.05, seed=92)
    val = 1e4 + 3.0 * rng.standard_normal((9, S))
    val[rng.random(val.shape) < 0.05] = np.nan
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    req = ps.TestRequest(test, ("stat", "p") + ps.EFFECTS_BY_TEST[test])
    res, ref = ps.run(req, ma, mb), oracle.oracle_run(req, ma, mb)
    assert same_nan(res["stat"], ref["stat"])
    assert bitwise_equal(res["stat"], ref["stat"])
    assert p_close(res["p"], ref["p"])
