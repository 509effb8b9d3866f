"""Config 5 (the 1/2/4/8-GPU scale run) at FULL size: Pearson 20,000 x 10^5,
30% MCAR, P = 1.9999e8 pairs, global BH over m ~ 2e8 p-values.

* r and p of three sampled triangle rows (0, the middle one, the last but
  one: 39,998 pairs x 10^5 samples) against the C oracle (the reference's
  two-pass loop restated, continuous.py:29-103): |dr| <= 1e-9 max(|r|, 1e-3),
  p within 1e-6 relative or 1e-12 absolute, identical NaN pattern.
* The device BH and Bonferroni of the full family -- m > 2^26, the 64-bit
  radix path of ps_adjust.cu -- bit for bit against the oracle's restatement
  of adjust.py:23-43 (numpy stable argsort) applied to the same p.
"""

from __future__ import annotations

import threading

import numpy as np
import pytest

from conftest import bitwise_equal, p_close, same_nan
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps


def _upper(m: np.ndarray) -> np.ndarray:
    """Row-major strict upper triangle (the reference's family order)."""
    F = m.shape[0]
    return np.concatenate([m[g, g + 1:] for g in range(F)])


def test_config5_full_size(oracle):
    cfg = workloads.config(5)
    mat = ps.make_matrix(cfg["a"], "continuous", na_sentinel=workloads.SENTINEL)
    F = mat.n_features
    req = ps.TestRequest("pearson", ("stat", "p", "p_bonferroni", "p_bh"))
    res = ps.run(req, mat)
    # three sampled triangle rows on the oracle, concurrently (one thread each)
    prep, run = oracle.block_runner("pearson", mat, None, wanted=("stat", "p"))
    rows = [0, F // 2, F - 2]
    threads = [threading.Thread(target=run, args=(g, g + 1)) for g in rows]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    ref = run.outs
    for g in rows:
        got_r, want_r = res["stat"][g, g:], ref["stat"][g, g:]
        assert same_nan(got_r, want_r), g
        m = ~np.isnan(want_r)
        assert np.all(np.abs(got_r[m] - want_r[m]) <= 1e-9 * np.maximum(np.abs(want_r[m]), 1e-3)), g
        assert same_nan(res["p"][g, g:], ref["p"][g, g:]), g
        assert p_close(res["p"][g, g:], ref["p"][g, g:]), g
    # global adjustment of the whole family, bit for bit given the device p
    fam = _upper(res["p"])
    m_def = int(np.count_nonzero(~np.isnan(fam)))
    assert m_def > 2 ** 26
    assert bitwise_equal(_upper(res["p_bh"]), oracle.adjust_family(fam, "bh"))
    assert bitwise_equal(_upper(res["p_bonferroni"]), oracle.adjust_family(fam, "bonferroni"))
    assert np.isnan(np.diag(res["p_bh"])).all()
    assert bitwise_equal(res["p_bh"], res["p_bh"].T)
