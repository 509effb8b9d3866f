"""Seeded synthetic inputs: the BASELINE.json configs and small parity cases.

The reference benchmarks on the CHRIS cohort, which is
access-by-request and absent here; the BASELINE configs stand in for it, built
with the seeded recipes of SURVEY.md section 8(d):

* shared latent-factor generator: L ~ U(-0.8, 0.8)^{F x 5}, Z ~ N(0,1)^{5 x S},
  X = L Z + N(0,1)^{F x S};
* every value transform (exp, rounding, level shifts) happens BEFORE the MCAR
  cells are set to the sentinel -99.0 (which make_matrix matches bit-exactly);
* seeds: numpy default_rng([20251019, k]) for config k, draws in the order
  written below.

``simulate`` is a small uniform / label generator for parity tests (the same
idea as the reference's simulate_matrix: exact per-feature missing count and
every label anchored once), written independently.
"""

from __future__ import annotations

import math

import numpy as np

SENTINEL = -99.0
SEED_BASE = 20251019


def simulate(n_features: int, n_samples: int, kind: str = "continuous", categories: int = 4,
             na_ratio: float = 0.0, seed: int = 0) -> np.ndarray:
    """Uniform values or integer labels with NaN marking missing cells."""
    rng = np.random.default_rng(seed)
    c = 2 if kind == "dichotomous" else categories
    n_miss = int(math.floor(na_ratio * n_samples + 1e-9))
    out = np.empty((n_features, n_samples))
    for f in range(n_features):
        if kind == "continuous":
            row = rng.uniform(size=n_samples)
        else:
            row = rng.integers(0, c, size=n_samples).astype(np.float64)
        miss = rng.permutation(n_samples)[:n_miss]
        if kind != "continuous":
            keep = np.setdiff1d(np.arange(n_samples), miss)
            anchors = keep[rng.permutation(keep.size)[:c]]
            row[anchors] = rng.permutation(c)[: anchors.size]
        row[miss] = np.nan
        out[f] = row
    return out


def _latent(rng: np.random.Generator, F: int, S: int) -> np.ndarray:
    L = rng.uniform(-0.8, 0.8, size=(F, 5))
    Z = rng.standard_normal((5, S))
    return L @ Z + rng.standard_normal((F, S))


def _mcar(rng: np.random.Generator, x: np.ndarray, rate: float) -> np.ndarray:
    x = x.copy()
    x[rng.random(x.shape) < rate] = SENTINEL
    return x


def _anchored_labels(rng: np.random.Generator, F: int, S: int, ks: np.ndarray,
                     probs: list[np.ndarray] | None) -> np.ndarray:
    codes = np.empty((F, S), dtype=np.int64)
    for f in range(F):
        k = int(ks[f])
        if probs is None:
            codes[f] = rng.integers(0, k, size=S)
        else:
            codes[f] = rng.choice(k, size=S, p=probs[f])
    return codes


def _anchor(rng: np.random.Generator, x: np.ndarray, ks: np.ndarray) -> None:
    """Put every declared level on one present cell so no level is empty."""
    for f in range(x.shape[0]):
        k = int(ks[f])
        present = np.flatnonzero(x[f] != SENTINEL)
        if present.size < k:
            continue
        pos = present[rng.permutation(present.size)[:k]]
        x[f, pos] = rng.permutation(k)


def config_spearman_like(rng: np.random.Generator, F: int, S: int) -> np.ndarray:
    """Config-2 pattern: latent factor, exp on half, 1-decimal rounding on 30%,
    20% MCAR, and for 10% of variables a contiguous 2000-sample block missing."""
    x = _latent(rng, F, S)
    exp_rows = rng.permutation(F)[: F // 2]
    x[exp_rows] = np.exp(x[exp_rows])
    round_rows = rng.permutation(F)[: int(round(0.3 * F))]
    x[round_rows] = np.round(x[round_rows], 1)
    x = _mcar(rng, x, 0.20)
    block_rows = rng.permutation(F)[: int(round(0.1 * F))]
    blk = min(2000, S)
    for f in block_rows:
        start = int(rng.integers(0, S - blk + 1))
        x[f, start:start + blk] = SENTINEL
    return x


C5_BLOCK = 256  # rows per independently seeded block of the config-5 matrix


def config5_rows(F: int, S: int, r0: int, r1: int, rng: np.random.Generator | None = None,
                 threads: int | None = None) -> np.ndarray:
    """Rows [r0, r1) of the config-5 Pearson matrix (latent factor, 30% MCAR).

    The shared factors come from ``default_rng([SEED_BASE, 5])`` (L then Z);
    each block of ``C5_BLOCK`` rows draws its noise and then its MCAR cells
    from its own ``default_rng([SEED_BASE, 5, 1000 + block])``.  So any row
    range -- one rank's shard of the 16 GB input -- is generated on its own,
    block-parallel, and equals the same rows of the whole matrix.
    """
    import concurrent.futures as cf
    import os

    if rng is None:
        rng = np.random.default_rng([SEED_BASE, 5])
    L = rng.uniform(-0.8, 0.8, size=(F, 5))
    Z = rng.standard_normal((5, S))
    out = np.empty((r1 - r0, S))

    def block(b):
        lo, hi = max(r0, b * C5_BLOCK), min(r1, (b + 1) * C5_BLOCK)
        rb = np.random.default_rng([SEED_BASE, 5, 1000 + b])
        n = min(F, (b + 1) * C5_BLOCK) - b * C5_BLOCK  # the whole block is drawn
        sel = slice(lo - b * C5_BLOCK, hi - b * C5_BLOCK)
        noise = rb.standard_normal((n, S))[sel]
        miss = (rb.random((n, S)) < 0.30)[sel]
        x = out[lo - r0:hi - r0]
        # L Z as five elementwise terms in a fixed order (a BLAS matmul's
        # rounding can depend on how many rows it is handed)
        np.multiply(L[lo:hi, 0:1], Z[0], out=x)
        for q in range(1, 5):
            x += L[lo:hi, q:q + 1] * Z[q]
        x += noise
        x[miss] = SENTINEL

    blocks = range(r0 // C5_BLOCK, (r1 + C5_BLOCK - 1) // C5_BLOCK)
    with cf.ThreadPoolExecutor(threads or min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(block, blocks))
    return out


def config(k: int, scale: float = 1.0) -> dict:
    """Inputs of BASELINE config k (1..5, '5s' for the config-5 Spearman leg).

    ``scale`` < 1 shrinks F (and S for the scale run) for quick checks; the
    bench always uses scale = 1.  Returns {'test': [...], 'a': raw, 'b': raw|None,
    'kind_a', 'kind_b', 'shape', 'desc'}.
    """
    key = 5 if k == "5s" else int(k)
    rng = np.random.default_rng([SEED_BASE, key if k != "5s" else 55])
    if k == 1:
        F, S = max(2, int(200 * scale)), 1000
        x = _mcar(rng, _latent(rng, F, S), 0.10)
        return dict(tests=["pearson"], a=x, b=None, kind_a="continuous", kind_b=None, F=F, S=S,
                    desc=f"pearson {F}x{S} 10% MCAR latent-factor")
    if k == 2:
        F, S = max(2, int(1000 * scale)), 10000
        x = config_spearman_like(rng, F, S)
        return dict(tests=["spearman"], a=x, b=None, kind_a="continuous", kind_b=None, F=F, S=S,
                    desc=f"spearman {F}x{S} exp/round ties, 20% MCAR + block missing")
    if k == 3:
        F, S = max(2, int(500 * scale)), 50000
        ks = rng.integers(2, 11, size=F)
        probs = [rng.dirichlet(np.ones(int(kk))) for kk in ks]
        codes = _anchored_labels(rng, F, S, ks, probs)
        shared = rng.integers(0, 10, size=S)
        dep = rng.permutation(F)[: int(round(0.2 * F))]
        for f in dep:
            mix = rng.random(S) < 0.5
            codes[f, mix] = shared[mix] % ks[f]
        x = _mcar(rng, codes.astype(np.float64), 0.15)
        _anchor(rng, x, ks)
        return dict(tests=["chi2"], a=x, b=None, kind_a="categorical", kind_b=None, F=F, S=S,
                    desc=f"chi2 {F}x{S} k in 2..10 Dirichlet(1), 20% latent-dependent, 15% MCAR")
    if k == 4:
        Fc, Fq, S = max(2, int(200 * scale)), max(2, int(2000 * scale)), 20000
        ks = rng.integers(2, 9, size=Fc)
        codes = _anchored_labels(rng, Fc, S, ks, None)
        D = rng.random((Fq, Fc)) < 0.25
        mu = [rng.normal(0.0, 0.3, size=int(kk)) for kk in ks]
        x = rng.standard_normal((Fq, S))
        for h in range(Fq):
            for g in np.flatnonzero(D[h]):
                x[h] += mu[g][codes[g]]
        lab = _mcar(rng, codes.astype(np.float64), 0.10)
        _anchor(rng, lab, ks)
        x = _mcar(rng, x, 0.10)
        two = np.flatnonzero(ks == 2)
        return dict(tests=["anova", "kruskal", "ttest", "mwu"], a=lab, b=x, kind_a="categorical",
                    kind_b="continuous", F=Fc, S=S, Fq=Fq, two_level_rows=two,
                    desc=f"mixed {Fc}x{Fq}x{S} k in 2..8, 25% shifted pairs, 10% MCAR")
    if k == 5:
        F, S = max(2, int(20000 * scale)), max(100, int(100000 * scale))
        x = config5_rows(F, S, 0, F, rng=rng)
        return dict(tests=["pearson"], a=x, b=None, kind_a="continuous", kind_b=None, F=F, S=S,
                    desc=f"pearson scale {F}x{S} 30% MCAR")
    if k == "5s":
        F, S = max(2, int(2000 * scale)), max(100, int(50000 * scale))
        x = config_spearman_like(rng, F, S)
        return dict(tests=["spearman"], a=x, b=None, kind_a="continuous", kind_b=None, F=F, S=S,
                    desc=f"spearman scale {F}x{S} config-2 pattern")
    raise ValueError(f"unknown config {k!r}")
