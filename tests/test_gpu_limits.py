"""Inputs at the edges of the device path's size classes.

The reference has no size limits (int64 tables, categorical.py:84-93; any
sample count, ranking.py:30-53), so the device path must answer there too:

* chi-squared with S >= 2^24 samples: table counts above 2^24 (no longer
  exact in fp32) accumulate as u32 -- bit-exact statistics vs the oracle;
  the u32 path forced at small S equals the fp32 path bit for bit;
* chi-squared tables in row bands (PS_CHI2_BAND_MB): scratch bounded for wide
  matrices, results bit-identical to one band.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps

CHI2 = ("stat", "p", "phi", "cramers_v")


def _same(a, b, names):
    for n in names:
        assert bitwise_equal(a[n], b[n]), n


def test_chi2_counts_above_2_pow_24(oracle):
    S = (1 << 24) + (1 << 20)
    rng = np.random.default_rng(24)
    x = np.zeros((3, S))
    x[0, rng.random(S) < 0.01] = 1.0      # (0, 0) cell of (0, 1): ~0.98 S > 2^24
    x[1, rng.random(S) < 0.005] = 1.0
    x[2] = rng.integers(0, 3, S)
    x[2, rng.random(S) < 0.02] = np.nan
    mat = ps.make_matrix(x, "categorical")
    req = ps.TestRequest("chi2", CHI2)
    res, ref = ps.run(req, mat), oracle.oracle_run(req, mat)
    for n in CHI2:
        assert same_nan(res[n], ref[n]), n
    for n in ("stat", "phi", "cramers_v"):
        assert bitwise_equal(res[n], ref[n]), n
    assert p_close(res["p"], ref["p"])


def test_chi2_u32_tables_equal_fp32(monkeypatch):
    raw = workloads.simulate(60, 5000, "categorical", categories=7, na_ratio=0.2, seed=9)
    mat = ps.make_matrix(raw, "categorical")
    req = ps.TestRequest("chi2", CHI2 + ("p_bh",))
    want = ps.run(req, mat)
    monkeypatch.setenv("PS_CHI2_U32", "1")
    _same(ps.run(req, mat), want, req.outputs)


def test_chi2_row_bands_equal_one_band(monkeypatch, oracle):
    c = workloads.config(3, scale=0.6)  # 300 features, k in 2..10 (Rp ~ 1900)
    mat = ps.make_matrix(c["a"], "categorical", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("chi2", CHI2)
    want = ps.run(req, mat)
    monkeypatch.setenv("PS_CHI2_BAND_MB", "1")  # 1 MiB of tables per band: many bands
    got = ps.run(req, mat)
    _same(got, want, CHI2)
    ref = oracle.compute("chi2", mat, None, wanted={"stat"}, lo=0, hi=5)
    assert bitwise_equal(got["stat"][:5], ref["stat"][:5])


@pytest.mark.parametrize("test", ["anova", "ttest"])
def test_group_replay_beyond_list_capacity(oracle, test):
    """More than 2^22 (the replay list's capacity) ill-conditioned cells:
    200 label rows x 20,990 constant continuous columns (every group mean
    equal: SSW = 0 / zero variance, decided by the exact replay).  The
    reference answers every cell (mixed.py:453-495); so does the device, by
    finishing the range again in list-sized chunks."""
    S = 96
    kind = "categorical" if test == "anova" else "dichotomous"
    lab = workloads.simulate(200, S, kind, categories=4, na_ratio=0.1, seed=5)
    rng = np.random.default_rng(6)
    val = np.repeat(rng.normal(size=(20990, 1)), S, axis=1)  # constant columns
    val = np.concatenate([val, rng.normal(size=(10, S))])
    val[rng.random(val.shape) < 0.05] = np.nan
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    eff = ps.EFFECTS_BY_TEST[test]
    req = ps.TestRequest(test, ("stat", "p") + eff)
    res, ref = ps.run(req, ma, mb), oracle.oracle_run(req, ma, mb)
    assert 200 * 20990 > 1 << 22  # constant-column cells: all take the exact replay
    for n in req.outputs:
        assert same_nan(res[n], ref[n]), n
        m = ~np.isnan(ref[n])
        if n == "p":
            assert p_close(res[n], ref[n]), n
        else:
            np.testing.assert_allclose(res[n][m], ref[n][m], rtol=1e-9, atol=0)


@pytest.mark.parametrize("test", ["anova", "ttest"])
def test_group_replay_chunked_equals_single_list(monkeypatch, test):
    kind = "categorical" if test == "anova" else "dichotomous"
    lab = workloads.simulate(12, 800, kind, categories=5, na_ratio=0.1, seed=7)
    val = workloads.simulate(90, 800, "continuous", na_ratio=0.1, seed=8)
    val[::3] = np.where(np.isnan(val[::3]), np.nan, 0.5)  # constant columns: replay cells
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    req = ps.TestRequest(test, ("stat", "p") + ps.EFFECTS_BY_TEST[test] + ("p_bh",))
    want = ps.run(req, ma, mb)
    monkeypatch.setenv("PS_REPLAY_CAP", "7")
    _same(ps.run(req, ma, mb), want, req.outputs)


@pytest.mark.parametrize("S", [55000, 70000])
def test_spearman_wide_sample_counts(oracle, S):
    """Beyond the shared-memory walk: S = 55,000 (16-bit tables, wide walk)
    and S = 70,000 (32-bit presort + wide walk).  rho bit-exact."""
    rng = np.random.default_rng(S)
    x = workloads.config_spearman_like(rng, 7, S)
    x[2, ::5] = np.nan   # NaN data under the numeric sentinel: present, sorts last
    x[3] = np.round(x[3])  # heavy ties
    mat = ps.make_matrix(x, "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("spearman", ("stat", "p", "rho", "p_bh"))
    res, ref = ps.run(req, mat), oracle.oracle_run(req, mat)
    for n in req.outputs:
        assert same_nan(res[n], ref[n]), n
    assert bitwise_equal(res["stat"], ref["stat"]) and bitwise_equal(res["rho"], ref["rho"])
    assert p_close(res["p"], ref["p"]) and p_close(res["p_bh"], ref["p_bh"], rtol=2e-6)


@pytest.mark.parametrize("test", ["kruskal", "mwu"])
@pytest.mark.parametrize("S", [70000])
def test_rank_mixed_wide_sample_counts(oracle, test, S):
    kind = "categorical" if test == "kruskal" else "dichotomous"
    lab = workloads.simulate(4, S, kind, categories=5, na_ratio=0.1, seed=S + 1)
    val = workloads.simulate(6, S, "continuous", na_ratio=0.2, seed=S + 2)
    val[1] = np.round(val[1], 2)  # ties
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    eff = ps.EFFECTS_BY_TEST[test]
    req = ps.TestRequest(test, ("stat", "p") + eff)
    res, ref = ps.run(req, ma, mb), oracle.oracle_run(req, ma, mb)
    for n in req.outputs:
        assert same_nan(res[n], ref[n]), n
    assert bitwise_equal(res["stat"], ref["stat"]) and bitwise_equal(res[eff[0]], ref[eff[0]])
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("host_labels", [True, False])
@pytest.mark.parametrize("test", ["chi2", "anova", "kruskal"])
def test_more_than_254_levels(oracle, test, host_labels):
    """c = 300 levels (16-bit label codes; the reference's c_f = max label + 1
    has no bound, datamodel.py:199-235).  Host labels are staged as codes by
    the host threads; device-resident labels are coded by prep_rows."""
    from paper_2505_00448_b200 import blocks
    import torch

    S = 4000
    lab = workloads.simulate(5, S, "categorical", categories=300, na_ratio=0.1, seed=300)
    lab[1] = np.where(np.isnan(lab[1]), np.nan, lab[1] % 7)  # a small-level row next to the wide ones
    ma = ps.make_matrix(lab, "categorical")
    assert int(ma.category_counts.max()) == 300
    mb = None
    if test != "chi2":
        val = workloads.simulate(9, S, "continuous", na_ratio=0.1, seed=301)
        val[2] = np.round(val[2], 2)
        mb = ps.make_matrix(val, "continuous")
    eff = ps.EFFECTS_BY_TEST[test]
    names = ("stat", "p") + eff
    req = ps.TestRequest(test, names)
    if test == "chi2":
        # the 300 x 300 diagonal tables have dof = 89,401: the reference's
        # chi2_sf does not converge there and raises (specfun.py:188) -- so
        # must the device; then a matrix whose wide feature leaves levels
        # empty (NaN cells) next to small-level features, compared by value
        with pytest.raises(oracle.OracleError):
            oracle.oracle_run(req, ma, mb)
        with pytest.raises(ps.NonConvergence):
            ps.run(req, ma, mb)
        lab = workloads.simulate(6, S, "categorical", categories=5, na_ratio=0.1, seed=302)
        lab[0] = np.where(np.isnan(lab[0]), np.nan, np.where(lab[0] == 4, 299.0, lab[0]))  # c_f = 300, 295 empty
        ma = ps.make_matrix(lab, "categorical")
        assert int(ma.category_counts.max()) == 300
    ref = oracle.oracle_run(req, ma, mb)
    if host_labels:
        res = ps.run(req, ma, mb)
    else:  # device-resident labels through the block API
        shape = ref["stat"].shape
        xa = torch.zeros((lab.shape[0], 4000), dtype=torch.float64, device="cuda")
        xa[:, :S] = torch.from_numpy(np.array(ma.values))
        da = blocks.DeviceMatrix(xa, "categorical", ma.na_sentinel, ma.category_counts, n_samples=S)
        db = blocks.DeviceMatrix(mb.values, "continuous", mb.na_sentinel, presort=test == "kruskal") if mb else None
        outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in names]
        lo, hi = blocks.full_range(test, da, db)
        blocks.block(test, da, db, lo, hi, outs)
        blocks.sync()
        res = {n: o.cpu().numpy() for n, o in zip(names, outs)}
    exact = {"chi2": ("stat", "phi", "cramers_v"), "kruskal": ("stat", "eta2")}.get(test, ())
    for n in names:
        assert same_nan(res[n], ref[n]), n
        if n in exact:
            assert bitwise_equal(res[n], ref[n]), n
        elif n == "p":
            assert p_close(res[n], ref[n]), n
        else:
            m = ~np.isnan(ref[n])
            np.testing.assert_allclose(res[n][m], ref[n][m], rtol=1e-9, atol=0)


def test_spearman_row_chunks_bound_scratch(monkeypatch):
    """Pair sums live in a chunk of rows x F (not F x F): forcing 7-row
    chunks (PS_SPEARMAN_ROWS) gives the one-chunk result bit for bit."""
    x = workloads.config_spearman_like(np.random.default_rng(8), 90, 3000)
    mat = ps.make_matrix(x, "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("spearman", ("stat", "p", "p_bh"))
    want = ps.run(req, mat)
    monkeypatch.setenv("PS_SPEARMAN_ROWS", "7")
    monkeypatch.setenv("PS_NO_OVERLAP", "1")
    _same(ps.run(req, mat), want, req.outputs)
