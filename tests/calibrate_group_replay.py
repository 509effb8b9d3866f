#!/usr/bin/env python3
"""Calibration of the ANOVA / t-test replay thresholds (ps_group.cu kReplayK, kCancelK).

Not a test (pytest does not collect it); run by hand on CPU:
    python tests/calibrate_group_replay.py
For seeded inputs over a grid of (offset, spread, S) it computes, per cell,
* err: the relative distance between the reference's F / t (the oracle, which
  replays the reference's one-pass raw sums, mixed.py:121-202, :453-520) and
  the same statistic in 80-bit long double on column-centred values;
* rc = (max - min group mean) / (sqrt(n) * raw rms)  -- the SSB criterion;
* rg = min_j ssw_j / (sqrt(n_j) * raw sum of squares_j) -- the SSW criterion;
and reports, for cells the SSW rule does not catch at kReplayK, the largest rc
whose error exceeds the tolerance: kCancelK must sit above it.  Measured
(2026-10, S in 500..30000, offsets 1..1e4, spreads 0.01..10): every cell with
err > 1e-10 has rg <= 2.5e-6 or rc <= 6.0e-7, and every cell with err > 3e-10
has rg <= 2.5e-6 or rc <= 1.3e-7, so kCancelK = 1.5e-6 keeps a 2.5x margin at
1e-10 (the tests hold 1e-9).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import paper_2505_00448_b200 as ps  # noqa: E402
import pyoracle as oracle  # noqa: E402
import workloads  # noqa: E402

K_REPLAY = 2.5e-6


def cells(test: str, offset: float, spread: float, S: int, nv: int = 30) -> np.ndarray:
    rng = np.random.default_rng(int(offset) + 7)
    kind = "categorical" if test == "anova" else "dichotomous"
    lab = workloads.simulate(6, S, kind, categories=3, na_ratio=0.05, seed=int(offset) + 1)
    val = offset + spread * rng.standard_normal((nv, S))
    val[::4] += spread * 0.05 * np.nan_to_num(lab[0])
    val[rng.random(val.shape) < 0.05] = np.nan
    ma, mb = ps.make_matrix(lab, kind), ps.make_matrix(val, "continuous")
    ref = oracle.oracle_run(ps.TestRequest(test, ("stat",)), ma, mb)["stat"]
    rows = []
    for g in range(lab.shape[0]):
        for h in range(nv):
            ok = ~np.isnan(lab[g]) & ~np.isnan(val[h])
            L = lab[g][ok].astype(int)
            x = val[h][ok].astype(np.longdouble)
            levels = np.unique(L)
            n = x.size
            xc = x - x.mean()
            groups = [xc[L == lv] for lv in levels]
            ns = np.array([v.size for v in groups])
            means = np.array([v.mean() for v in groups])
            ssw = sum(((v - v.mean()) ** 2).sum() for v in groups)
            if test == "anova":
                k = len(levels)
                ssb = (ns * (means - xc.mean()) ** 2).sum()
                stat = (ssb / (k - 1)) / (ssw / (n - k))
            else:
                stat = (means[0] - means[1]) / np.sqrt(ssw / (n - 2) * (1 / ns[0] + 1 / ns[1]))
            rms = float(np.sqrt((x * x).mean()))
            rc = float(means.max() - means.min()) / (np.sqrt(n) * rms)
            rg = min(float(((v - v.mean()) ** 2).sum()) / (np.sqrt(v.size) * float(((v + x.mean()) ** 2).sum()))
                     for v in groups)
            rows.append((abs(float(stat) - ref[g, h]) / abs(float(stat)), rc, rg))
    return np.array(rows)


def main() -> None:
    grid = [(100.0, 0.1), (100.0, 1.0), (100.0, 5.0), (10.0, 3.0), (10.0, 10.0), (1.0, 3.0), (1e4, 3.0),
            (50.0, 0.01), (3.0, 1.0)]
    for test in ("anova", "ttest"):
        for S in (500, 2000, 30000):
            r = np.concatenate([cells(test, off, sp, S) for off, sp in grid])
            free = r[:, 2] > K_REPLAY
            for tol in (1e-10, 3e-10, 1e-9):
                bad = (r[:, 0] > tol) & free
                top = r[bad, 1].max() if bad.any() else 0.0
                print(f"{test:6s} S={S:6d} tol={tol:.0e}: {bad.sum():4d} cells over tol outside the SSW rule, "
                      f"max rc {top:.2e}")


if __name__ == "__main__":
    main()
