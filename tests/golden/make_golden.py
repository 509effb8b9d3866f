#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ (run in the builder container).

1. ``specfun_mp.json`` -- 8 special functions x 100 seeded points, reference
   values from mpmath at 50 significant digits (independent of any
   implementation; same functions and parameter ranges as the reference's
   specfun tests, pkg/tests/test_specfun.py, drawn from our own seed).
2. ``run_fixtures.npz`` -- small seeded inputs for all 7 tests and the
   outputs of the REFERENCE implementation itself (``pairstat.run`` imported
   from /root/reference/pkg/src, numba path), plus BH / BY / Bonferroni of
   the same p matrices.  These pin the CPU oracle (tests/test_oracle_golden.py)
   and the device path (tests/test_gpu_golden.py) to the reference's own
   outputs on the same inputs.

Usage:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import math
import sys
from pathlib import Path

import mpmath as mp
import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

import workloads  # noqa: E402

mp.mp.dps = 50
N = 100


def specfun_grid(seed: int = 20251019) -> dict:
    rng = np.random.default_rng(seed)
    g: dict[str, list] = {}
    g["ln_gamma"] = [[float(x), float(mp.loggamma(mp.mpf(x)))] for x in np.logspace(-2.5, 5.5, N)]
    rows = []
    for _ in range(N):
        a = 10 ** rng.uniform(np.log10(0.4), np.log10(120.0))
        b = 10 ** rng.uniform(np.log10(0.4), np.log10(120.0))
        x = rng.uniform(0.002, 0.998)
        rows.append([x, a, b, float(mp.betainc(a, b, 0, x, regularized=True))])
    g["reg_inc_beta"] = rows
    rows = []
    for i in range(N):
        a = 10 ** rng.uniform(-0.4, 2.2)
        x = a * (rng.uniform(1e-3, 0.05) if i % 8 == 0 else rng.uniform(0.05, 2.8))
        rows.append([a, x, float(mp.gammainc(a, x, mp.inf, regularized=True))])
    g["reg_inc_gamma_upper"] = rows
    g["normal_sf"] = [[z, float(0.5 * mp.erfc(mp.mpf(z) / mp.sqrt(2)))]
                      for z in rng.uniform(-30.0, 30.0, N)]
    rows = []
    for _ in range(N):
        dof = 10 ** rng.uniform(0, 3)
        t = rng.uniform(-8.0, 25.0)
        x = dof / (dof + t * t)
        tail = 0.5 * mp.betainc(0.5 * dof, 0.5, 0, x, regularized=True)
        rows.append([t, dof, float(tail if t >= 0 else 1 - tail)])
    g["t_sf"] = rows
    rows = []
    for _ in range(N):
        dof = float(rng.integers(1, 120))
        x = dof * rng.uniform(0.05, 3.5)
        rows.append([x, dof, float(mp.gammainc(0.5 * dof, 0.5 * x, mp.inf, regularized=True))])
    g["chi2_sf"] = rows
    rows = []
    for _ in range(N):
        d1 = float(rng.integers(1, 12))
        d2 = float(rng.integers(3, 400))
        f = rng.uniform(0.05, 12.0)
        x = d2 / (d2 + d1 * f)
        rows.append([f, d1, d2, float(mp.betainc(0.5 * d2, 0.5 * d1, 0, x, regularized=True))])
    g["f_sf"] = rows
    rows = []
    for _ in range(N):
        a = 10 ** rng.uniform(-0.2, np.log10(150.0))
        r = rng.uniform(0.0, 0.95)
        rows.append([r, a, float(mp.betainc(a, a, 0, 0.5 * (1 - r), regularized=True))])
    g["beta_sym_sf"] = rows
    return g


def run_fixtures() -> dict:
    sys.path.insert(0, "/root/reference/pkg/src")
    import pairstat  # the reference

    out: dict[str, np.ndarray] = {}
    specs = [
        ("pearson", 0.1, 1), ("pearson", 0.4, 2), ("spearman", 0.1, 3), ("spearman", 0.3, 4),
        ("chi2", 0.1, 5), ("chi2", 0.3, 6), ("ttest", 0.1, 7), ("mwu", 0.1, 8),
        ("anova", 0.2, 9), ("kruskal", 0.2, 10),
    ]
    cases = []
    for test, na, seed in specs:
        kind_a, kind_b = pairstat.KINDS_BY_TEST[test]
        F, S = (13, 150) if kind_b is None else (9, 150)
        raw_a = workloads.simulate(F, S, kind_a, categories=4, na_ratio=na, seed=seed)
        if test == "spearman":
            raw_a = np.round(raw_a * 10) / 10  # ties
        raw_b = None if kind_b is None else workloads.simulate(11, S, kind_b, na_ratio=na, seed=seed + 50)
        mat_a = pairstat.make_matrix(raw_a, kind_a)
        mat_b = None if raw_b is None else pairstat.make_matrix(raw_b, kind_b)
        outs = pairstat.outputs_for(test)
        req = pairstat.TestRequest(test=test, outputs=outs)
        res = pairstat.run(req, mat_a, mat_b)
        key = f"{test}_{seed}"
        out[f"{key}__a"] = raw_a
        if raw_b is not None:
            out[f"{key}__b"] = raw_b
        for name in outs:
            out[f"{key}__{name}"] = res[name]
        cases.append(key)
    out["cases"] = np.array(cases)
    return out


def main() -> None:
    (HERE / "specfun_mp.json").write_text(json.dumps(specfun_grid()))
    np.savez_compressed(HERE / "run_fixtures.npz", **run_fixtures())
    print("wrote", HERE / "specfun_mp.json", HERE / "run_fixtures.npz")


if __name__ == "__main__":
    main()
