"""Pearson with the masked moments on the int8 tensor cores (ps_moments.cu).

Large-F Pearson computes Sx = X' M^T and Sxx = X'^2 M^T (and, by default, Sxy
and the pair counts) from exact int8 digit contractions (PS_PEARSON_SXY=dmma:
Sxy on the FP64 tensor tiles).  These tests force the
path on (PS_PEARSON_MOMENTS=1) at oracle-sized shapes and check it against the
CPU oracle (continuous.py:29-103) at the north-star tolerances, against the
FP64-moment path, on degenerate rows (constants, large offsets, NaN data under
a numeric sentinel, all-missing rows), and bit-for-bit across launch ranges.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import blocks


def _check(res, ref):
    for name in ("stat", "p"):
        assert same_nan(res[name], ref[name]), name
    r, rr = res["stat"], ref["stat"]
    m = ~np.isnan(rr)
    assert np.all(np.abs(r[m] - rr[m]) <= 1e-9 * np.maximum(np.abs(rr[m]), 1e-3))
    assert p_close(res["p"], ref["p"])


@pytest.mark.parametrize("sxy", ["int8", "dmma"])
@pytest.mark.parametrize("na", [0.0, 0.3])
@pytest.mark.parametrize("F,S", [(70, 333), (300, 1000), (260, 5000)])
def test_moments_match_oracle(oracle, monkeypatch, F, S, na, sxy):
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    monkeypatch.setenv("PS_PEARSON_SXY", sxy)
    raw = workloads.simulate(F, S, "continuous", na_ratio=na, seed=F * 11 + S + int(na * 10))
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


@pytest.mark.parametrize("sxy", ["int8", "dmma"])
def test_moments_degenerate_rows(oracle, monkeypatch, sxy):
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    monkeypatch.setenv("PS_PEARSON_SXY", sxy)
    rng = np.random.default_rng(5)
    raw = rng.normal(size=(40, 700))
    raw[0] = 0.1                        # constant
    raw[1] = 1e6 + rng.normal(size=700) * 1e-3   # large offset, small spread
    raw[2, 3:] = np.nan                 # n = 3 with everyone
    raw[3, :] = np.nan                  # all missing
    raw[4] = raw[5] * 1e-200            # tiny scale
    raw[6] = raw[7] * 1e150             # huge scale
    raw[8] = -raw[9]
    raw[10, rng.random(700) < 0.5] = np.nan
    raw[11, ::7] = 1e4                  # outliers
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


def test_moments_nan_data_raises_like_fp64_path(monkeypatch):
    """NaN data under a numeric sentinel is present data: the reference's tail
    raises NonConvergence; both moment paths must agree."""
    raw = workloads.simulate(30, 300, "continuous", na_ratio=0.1, seed=9)
    raw[4, 17] = np.nan
    mat = ps.make_matrix(raw, "continuous", na_sentinel=workloads.SENTINEL)
    req = ps.TestRequest("pearson", ("stat", "p"))
    outcomes = []
    for flag in ("0", "1"):
        monkeypatch.setenv("PS_PEARSON_MOMENTS", flag)
        try:
            ps.run(req, mat)
            outcomes.append("ok")
        except ps.NonConvergence:
            outcomes.append("NonConvergence")
    assert outcomes[0] == outcomes[1]


def test_moments_close_to_fp64_moments(monkeypatch):
    raw = workloads.simulate(2100, 1500, "continuous", na_ratio=0.3, seed=21)
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "0")
    a = ps.run(req, mat)
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    b = ps.run(req, mat)
    assert same_nan(a["stat"], b["stat"])
    m = ~np.isnan(a["stat"])
    assert np.max(np.abs(a["stat"][m] - b["stat"][m])) <= 1e-12
    assert p_close(b["p"], a["p"], rtol=1e-9)


def test_moments_range_independent(monkeypatch):
    """Block ranges compute the moments of rows / columns [lo, F) only: every
    pair is bitwise identical to the whole-matrix launch."""
    import torch

    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    F, S = 600, 900
    raw = workloads.simulate(F, S, "continuous", na_ratio=0.2, seed=4)
    dm = blocks.DeviceMatrix(raw, "continuous", np.nan, None)
    whole = [torch.full((F, F), float("nan"), dtype=torch.float64, device="cuda") for _ in range(2)]
    blocks.block("pearson", dm, None, 0, F, whole)
    parts = [torch.full((F, F), float("nan"), dtype=torch.float64, device="cuda") for _ in range(2)]
    for lo, hi in ((0, 137), (137, 400), (400, F)):
        blocks.block("pearson", dm, None, lo, hi, parts)
    blocks.sync()
    for w, p in zip(whole, parts):
        assert bitwise_equal(w.cpu().numpy(), p.cpu().numpy())
    dm.close()


def test_moments_outlier_exponent_replayed(oracle, monkeypatch):
    """A row whose digit scale is set by one outlier: for partners missing at
    the outlier the expansion's error bound exceeds 1e-12 of the centred sums,
    so those pairs are replayed exactly (without the check r would be off by
    ~1e-5 here)."""
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    rng = np.random.default_rng(8)
    F, S = 48, 20000
    raw = rng.normal(size=(F, S))
    raw[3, 0] = 1e5                     # mean shift ~5: mild cancellation, huge row exponent
    raw[7, 1] = -3e4
    raw[rng.random(F) < 0.5, 0] = np.nan
    raw[rng.random((F, S)) < 0.1] = np.nan
    raw[3, 0] = 1e5
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))


@pytest.mark.parametrize("F,S", [(600, 900), (1100, 2500)])
def test_cta_pair_gemms_bitwise_equal_multicast(monkeypatch, F, S):
    """PS_GEMM_2SM=1 runs the int8 contractions as tcgen05 cta_group::2 pair
    MMAs (M = 256 across the two SMs of a cluster): same units, K order and
    int32 sums as the multicast kernels, so every output bit agrees -- on the
    block path (odd tile-row counts leave a dummy partner CTA) and through
    ps_run's incremental column blocks."""
    import torch

    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    raw = workloads.simulate(F, S, "continuous", na_ratio=0.25, seed=12)
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("PS_GEMM_2SM", mode)
        dm = blocks.DeviceMatrix(raw, "continuous", np.nan, None)
        outs = [torch.full((F, F), float("nan"), dtype=torch.float64, device="cuda") for _ in range(2)]
        for lo, hi in ((0, 300), (300, F)):
            blocks.block("pearson", dm, None, lo, hi, outs)
        blocks.sync()
        dm.close()
        full = ps.run(ps.TestRequest("pearson", ("stat", "p")), ps.make_matrix(raw, "continuous"))
        res[mode] = [o.cpu().numpy() for o in outs] + [full["stat"], full["p"]]
    for a, b in zip(res["0"], res["1"]):
        assert bitwise_equal(a, b)


def test_symmetric_sxy_matches_digit_products(oracle, monkeypatch):
    """Sxy from 16 sum-plane products (D_s + D_t)(D_s + D_t)^T and the 8 squares
    (default for S < 2^17) is the same exact integer sum as the 36 digit products
    (PS_SXY_SYM=0); only the fp64 fold order differs: r within 1e-13, p within
    1e-9, both inside the oracle tolerances (range / upload-order independence of
    the default form: test_moments_range_independent, test_gpu_overlap.py)."""
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    F, S = 700, 3000
    raw = workloads.simulate(F, S, "continuous", na_ratio=0.3, seed=21)
    raw[5] = raw[5] * 1e6 + 3e6   # large scale, offset of a few sigma
    raw[9, ::7] = 0.0
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    monkeypatch.setenv("PS_SXY_SYM", "0")
    plain = ps.run(req, mat)
    monkeypatch.setenv("PS_SXY_SYM", "1")
    sym = ps.run(req, mat)
    assert same_nan(plain["stat"], sym["stat"])
    m = ~np.isnan(plain["stat"])
    assert np.max(np.abs(plain["stat"][m] - sym["stat"][m])) <= 1e-13
    assert p_close(sym["p"], plain["p"], rtol=1e-9)
    _check(sym, oracle.oracle_run(req, mat))


@pytest.mark.parametrize("b256", ["0", "1"])
def test_moment_plane_bases_match_oracle(oracle, monkeypatch, b256):
    """The moments from balanced base-256 planes (default: 6 for Sx, 7 for Sxx,
    one guard bit) and from the base-128 planes (PS_MOMENTS_B256=0: 7 + 8) both
    meet the oracle tolerances, on rows with large offsets / scales and values
    at the top of a row's binade (the most significant digit's range)."""
    monkeypatch.setenv("PS_PEARSON_MOMENTS", "1")
    monkeypatch.setenv("PS_MOMENTS_B256", b256)
    F, S = 300, 4000
    raw = workloads.simulate(F, S, "continuous", na_ratio=0.25, seed=33)
    raw[2] = raw[2] * 1e-7 - 3e-7
    raw[4] = np.where(np.isnan(raw[4]), np.nan, np.sign(raw[4]) * (1.0 - 2.0 ** -40))  # |x| just under 2^0
    raw[6, :50] = 1.9999999 * np.nanmax(np.abs(raw[6]))
    mat = ps.make_matrix(raw, "continuous")
    req = ps.TestRequest("pearson", ("stat", "p"))
    _check(ps.run(req, mat), oracle.oracle_run(req, mat))
