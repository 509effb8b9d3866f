#!/usr/bin/env python3
"""Golden vectors for the exact Mann-Whitney U branch (run in the builder container).

Pins the exact-distribution path (reference mixed.py:231-247 ``_exact_u_counts``
and the exact branch of ``_mwu_finish``, :305-363) with outputs of the
REFERENCE itself (``pairstat.run`` imported from /root/reference/pkg/src):

* ``enum_T{T}`` (T = 2..10): every group split n0 = 1..T-1 of T tie-free
  values (label row n0-1 holds n0 zeros then ones) against 3 random
  permutations per split, ``u_mode='exact'``; plus, for the cells of each
  split's own permutations, the reference's brute-force enumeration
  ``permutation_mwu`` (the acceptance test test_acceptance.py:110-130 in
  matrix form): exact p must equal it.
* ``auto40``: S = 40, 12 dichotomous label rows with min group sizes 1..12
  (auto mode takes the exact branch below 8, tie-free pairs only), 10% of
  label cells missing, 15 continuous features of which 5 have ties;
  ``u_mode`` auto and asymptotic.
* ``exact64``: S = 64 (the exact cap), 8 label rows, 10 tie-free features,
  some feature cells missing (n varies <= 64); ``u_mode='exact'``.

Usage:  NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_mwu_exact_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUTS = ("stat", "p", "r", "p_bh", "p_bonferroni")


def main() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    import pairstat  # the reference

    rng = np.random.default_rng([20251019, 64])
    out: dict[str, np.ndarray] = {}
    cases = []

    def record(key, labels, values, mode):
        la = pairstat.make_matrix(labels, "dichotomous")
        va = pairstat.make_matrix(values, "continuous")
        res = pairstat.run(pairstat.TestRequest(test="mwu", outputs=OUTS, u_mode=mode), la, va)
        out[f"{key}__a"] = labels
        out[f"{key}__b"] = values
        out[f"{key}__mode"] = np.array(mode)
        for n in OUTS:
            out[f"{key}__{n}"] = res[n]
        cases.append(key)

    for T in range(2, 11):
        labels = np.ones((T - 1, T))
        for n0 in range(1, T):
            labels[n0 - 1, :n0] = 0.0
        values = np.stack([rng.permutation(T).astype(np.float64) for _ in range(3 * (T - 1))])
        key = f"enum_T{T}"
        record(key, labels, values, "exact")
        perm = np.full((T - 1, 3 * (T - 1)), np.nan)
        for n0 in range(1, T):
            for j in range(3 * (n0 - 1), 3 * n0):
                x = values[j]
                perm[n0 - 1, j] = float(pairstat.permutation_mwu(x[:n0], x[n0:], max_n=10))
        out[f"{key}__perm_p"] = perm

    # auto / asymptotic at S = 40
    S = 40
    labels = np.ones((12, S))
    for g in range(12):
        n0 = g + 1
        labels[g, rng.permutation(S)[:n0]] = 0.0
        miss = rng.random(S) < 0.10
        labels[g, miss] = np.nan
    values = np.stack([rng.permutation(S).astype(np.float64) + rng.uniform(0, 0.5) for _ in range(15)])
    values[10:] = np.round(values[10:] / 3.0)  # ties in 5 features
    for mode in ("auto", "asymptotic"):
        record(f"auto40_{mode}", labels, values, mode)

    # exact at the 64-sample cap, with missing feature cells
    S = 64
    labels = np.ones((8, S))
    for g in range(8):
        labels[g, rng.permutation(S)[: int(rng.integers(1, 33))]] = 0.0
    values = np.stack([rng.permutation(S).astype(np.float64) * 0.37 - 3.0 for _ in range(10)])
    values[rng.random(values.shape) < 0.08] = np.nan
    record("exact64", labels, values, "exact")

    out["cases"] = np.array(cases)
    np.savez_compressed(HERE / "mwu_exact.npz", **out)
    print("wrote", HERE / "mwu_exact.npz", len(cases), "cases")


if __name__ == "__main__":
    main()
