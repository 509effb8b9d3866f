"""Device BH / BY / Bonferroni vs the restated reference adjust (adjust.py:23-87).

Given the same p matrix the device result is bit-identical (survey Appendix B).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps


@pytest.mark.parametrize("method", ["bonferroni", "bh", "by"])
def test_adjust_vector_families(oracle, method):
    rng = np.random.default_rng(55)
    for size in [1, 2, 3, 7, 100, 1000, 4097, 20000, 24577, 200001, 1000003]:
        v = rng.random(size)
        ties = rng.random(size) < 0.3
        v[ties] = np.round(v[ties], 1)
        v[rng.random(size) < 0.1] = np.nan
        got = ps.adjust(v.reshape(1, -1), method, symmetric=False).ravel()
        want = oracle.adjust_family(v, method)
        assert bitwise_equal(got, want), (method, size)


@pytest.mark.parametrize("method", ["bonferroni", "bh", "by"])
def test_adjust_low_bit_collisions(oracle, method):
    """p-values equal in their high 32 bits (the small-family sort orders the
    high halves first, then repairs or fully re-sorts colliding runs)."""
    rng = np.random.default_rng(3)
    for size in [500, 20000]:
        v = 0.5 + rng.integers(0, 40, size) * 2.0**-45     # long colliding runs
        w = rng.random(size)
        w[::5] = 0.25 + rng.integers(0, 3, w[::5].size) * 2.0**-50  # short runs
        for x in (v, w):
            got = ps.adjust(x.reshape(1, -1), method, symmetric=False).ravel()
            assert bitwise_equal(got, oracle.adjust_family(x, method)), (method, size)


@pytest.mark.parametrize("method", ["bh", "by"])
def test_adjust_large_family_runs(oracle, method):
    """Families above the single-CTA size take the high-half radix with
    run repair: short colliding runs are repaired in place, long runs of
    differing keys fall back to the 64-bit sort, long runs of one value need
    neither."""
    rng = np.random.default_rng(11)
    size = 150001
    cases = []
    w = rng.random(size)
    w[::3] = 0.25 + rng.integers(0, 5, w[::3].size) * 2.0**-50       # short runs
    cases.append(w)
    v = rng.random(size)
    v[: size // 2] = 0.5 + rng.integers(0, 1000, size // 2) * 2.0**-45  # long mixed runs
    cases.append(v)
    u = rng.random(size)
    u[rng.random(size) < 0.4] = 1.0                                    # one long run of 1.0
    u[rng.random(size) < 0.05] = np.nan
    cases.append(u)
    t = rng.random(size) ** 8                                          # many binades
    cases.append(t)
    z = rng.random(size)
    z[:9000] = rng.integers(0, 900, 9000) * 2.0**-1074                  # a long run of subnormals
    z[9000:12000] = 0.0
    cases.append(z)
    y = rng.random(size)
    y[:40000] = rng.integers(0, 300, 40000) * 2.0**-1074                # too long for the CTA sort
    cases.append(y)
    x = rng.random(size)
    x[:5000] = 0.5 + rng.integers(0, 5000, 5000) * 2.0**-40             # CTA bitonic (wide low halves)
    x[5000:7000] = 0.25 + rng.integers(0, 2000, 2000) * 2.0**-54        # CTA counting sort
    cases.append(x)
    for x in cases:
        got = ps.adjust(x.reshape(1, -1), method, symmetric=False).ravel()
        assert bitwise_equal(got, oracle.adjust_family(x, method)), method


@pytest.mark.parametrize("method", ["bonferroni", "bh", "by"])
@pytest.mark.parametrize("n", [150, 301])
def test_adjust_symmetric(oracle, method, n):
    rng = np.random.default_rng(7)
    up = rng.random(n * (n - 1) // 2) ** 3
    up[rng.random(up.size) < 0.1] = np.nan
    m = np.zeros((n, n))
    r, c = np.triu_indices(n, 1)
    m[r, c] = up
    m[c, r] = up
    np.fill_diagonal(m, 0.0)
    got = ps.adjust(m, method, symmetric=True)
    want = oracle.adjust(m, method, symmetric=True)
    assert bitwise_equal(got, want)
    assert np.isnan(np.diag(got)).all()


def test_adjust_all_nan_and_errors():
    m = np.full((4, 4), np.nan)
    assert np.isnan(ps.adjust(m, "bh", symmetric=True)).all()
    with pytest.raises(ps.UnknownMethod, match="holm"):
        ps.adjust(m, "holm", symmetric=True)
    with pytest.raises(ps.NonSquareSymmetric, match="square"):
        ps.adjust(np.zeros((2, 3)), "bh", symmetric=True)
