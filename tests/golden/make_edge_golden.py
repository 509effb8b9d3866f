#!/usr/bin/env python3
"""Golden vectors for the missing-value sentinel edge cases (builder container).

Outputs of the REFERENCE (``pairstat.run`` from /root/reference/pkg/src) on:

* ``negzero_<test>``: every test with ``na_sentinel=-0.0`` -- -0.0 cells are
  missing, +0.0 cells (and label 0) present (datamodel.py:86-104 compares
  bits);
* ``nandata_<test>`` (spearman / kruskal / mwu): NaN *data* under the
  numeric sentinel -99 -- present values that sort after every number
  (ranking.py:47).  (Pearson on such data raises NonConvergence in the
  reference; tests/test_gpu_sentinel.py checks that exception.)

Usage:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_edge_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import workloads  # noqa: E402


def _with_zeros(raw, kind, rng):
    x = raw.copy()
    if kind == "continuous":
        x[rng.random(x.shape) < 0.05] = 0.0
    x[np.isnan(x)] = -0.0  # the sentinel
    x[rng.random(x.shape) < 0.03] = -0.0
    return x


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    import pairstat  # the reference

    out: dict[str, np.ndarray] = {}
    cases = []

    def record(key, test, mats, sentinel):
        names = ("stat", "p") + pairstat.EFFECTS_BY_TEST[test] + ("p_bh",)
        ref = [pairstat.make_matrix(x, k, na_sentinel=sentinel) for x, k in mats]
        res = pairstat.run(pairstat.TestRequest(test, names), *ref)
        out[f"{key}__a"] = mats[0][0]
        if len(mats) > 1:
            out[f"{key}__b"] = mats[1][0]
        out[f"{key}__sentinel"] = np.array(sentinel)
        for n in names:
            out[f"{key}__{n}"] = res[n]
        cases.append(key)

    rng = np.random.default_rng([20251019, 70])
    for test in pairstat.TESTS:
        kind_a, kind_b = pairstat.KINDS_BY_TEST[test]
        a = _with_zeros(workloads.simulate(14, 400, kind_a, categories=4, na_ratio=0.1, seed=21), kind_a, rng)
        mats = [(a, kind_a)]
        if kind_b:
            b = _with_zeros(workloads.simulate(17, 400, kind_b, na_ratio=0.1, seed=22), kind_b, rng)
            b[3] = np.round(b[3], 1)
            mats.append((b, kind_b))
        record(f"negzero_{test}", test, mats, -0.0)
    for test in ("spearman", "kruskal", "mwu"):
        kind_a, kind_b = pairstat.KINDS_BY_TEST[test]
        cont = rng.normal(size=(9, 300))
        cont[rng.random(cont.shape) < 0.1] = -99.0
        cont[1, ::17] = np.nan
        cont[4, 5] = np.nan
        cont[6] = np.round(cont[6], 1)
        if kind_b is None:
            mats = [(cont, "continuous")]
        else:
            lab = workloads.simulate(5, 300, kind_a, categories=3, na_ratio=0.1, seed=4)
            lab[np.isnan(lab)] = -99.0
            mats = [(lab, kind_a), (cont, "continuous")]
        record(f"nandata_{test}", test, mats, -99.0)
    out["cases"] = np.array(cases)
    np.savez_compressed(HERE / "edge_fixtures.npz", **out)
    print("wrote", HERE / "edge_fixtures.npz", len(cases), "cases")


if __name__ == "__main__":
    main()
