"""The ``engine='gpu'`` row of the reference's timing sweep.

Reference: ``pkg/src/pairstat/bench.py`` -- ``BENCH_COLUMNS`` (:36-46),
``BenchRow`` (:53-79), ``run_bench`` (:128-215), ``render_rows`` (:218-242).
The reference sweeps (test, features, samples, na_ratio, threads, engine)
with engines ``fast`` (numba) and ``oracle`` (scipy); a row's clock covers
only the engine call, after one untimed warm-up, over ``reps`` repetitions
(mean and standard deviation), and fast rows carry ``speedup`` = reference
mean / mean.  Here the same sweep times this package's ``run`` as engine
``gpu``; CPU engines to compare with are passed in as ``baselines`` (e.g.
``{"fast": pairstat.run, "oracle": pairstat.oracle_run}`` when the reference
is installed -- INTEGRATION.md §4), and the gpu rows' ``speedup`` is the first
baseline's mean over the gpu mean.  ``render_rows`` emits the reference's
CSV byte for byte in shape (same header, ``repr`` floats).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Callable

import numpy as np

from .datamodel import KINDS_BY_TEST, TESTS, TestRequest, make_matrix
from .engine import run

BENCH_REPS = 3
ENGINES = ("gpu",)
BENCH_COLUMNS = ("test", "features", "samples", "na_ratio", "threads", "engine", "mean_seconds", "std_seconds",
                 "speedup")


@dataclass(frozen=True)
class BenchRow:
    test: str
    features: int
    samples: int
    na_ratio: float
    threads: int
    engine: str
    mean_seconds: float
    std_seconds: float
    speedup: float


def _simulate(n_features: int, n_samples: int, kind: str, na_ratio: float, seed: int) -> np.ndarray:
    """Seeded inputs of the sweep's shape: uniform values or labels 0..3 with
    every label present, exactly floor(na_ratio * S) NaN cells per feature."""
    rng = np.random.default_rng(seed)
    c = 2 if kind == "dichotomous" else 4
    n_miss = int(math.floor(na_ratio * n_samples + 1e-9))
    out = np.empty((n_features, n_samples))
    for f in range(n_features):
        row = rng.uniform(size=n_samples) if kind == "continuous" else rng.integers(0, c, n_samples).astype(float)
        miss = rng.permutation(n_samples)[:n_miss]
        if kind != "continuous":
            keep = np.setdiff1d(np.arange(n_samples), miss)
            row[keep[rng.permutation(keep.size)[:c]]] = rng.permutation(c)[: min(c, keep.size)]
        row[miss] = np.nan
        out[f] = row
    return out


def build_inputs(test: str, n_features: int, n_samples: int, na_ratio: float, seed: int):
    """Simulated and validated input matrices of one configuration (bench.py:84-110)."""
    kind_a, kind_b = KINDS_BY_TEST[test]
    mat_a = make_matrix(_simulate(n_features, n_samples, kind_a, na_ratio, seed), kind_a)
    if kind_b is None:
        return mat_a, None
    return mat_a, make_matrix(_simulate(n_features, n_samples, kind_b, na_ratio, seed + 1), kind_b)


def _time_call(fn, reps: int) -> tuple[float, float]:
    """Mean and standard deviation of ``reps`` timed calls after one warm-up."""
    fn()
    elapsed = np.empty(reps, dtype=np.float64)
    for i in range(reps):
        start = time.perf_counter()
        fn()
        elapsed[i] = time.perf_counter() - start
    return float(elapsed.mean()), float(elapsed.std())


def run_bench(tests, features, samples, na_ratios, threads=(1,), engines=ENGINES, seed: int = 0,
              reps: int = BENCH_REPS, baselines: dict[str, Callable] | None = None) -> list[BenchRow]:
    """Time every configuration of the grid: baseline rows first (threads=1,
    as the reference's reference rows), then the gpu rows with ``speedup``."""
    baselines = dict(baselines or {})
    for test in tests:
        if test not in TESTS:
            raise ValueError(f"unknown test {test!r}; expected one of {TESTS}")
    for engine in engines:
        if engine not in ENGINES:
            raise ValueError(f"unknown engine {engine!r}; expected one of {ENGINES}")
    rows: list[BenchRow] = []
    for test in tests:
        for n_features in features:
            for n_samples in samples:
                for na_ratio in na_ratios:
                    mat_a, mat_b = build_inputs(test, n_features, n_samples, na_ratio, seed)
                    request = TestRequest(test=test, outputs=("stat", "p"))
                    base_mean = math.nan
                    for name, fn in baselines.items():
                        mean, std = _time_call(lambda: fn(request, mat_a, mat_b), reps)
                        if math.isnan(base_mean):
                            base_mean = mean
                        rows.append(BenchRow(test, n_features, n_samples, na_ratio, 1, name, mean, std, math.nan))
                    if "gpu" not in engines:
                        continue
                    for n_threads in threads:
                        req = TestRequest(test=test, outputs=("stat", "p"), threads=n_threads)
                        mean, std = _time_call(lambda: run(req, mat_a, mat_b), reps)
                        speedup = base_mean / mean if mean > 0 else math.nan
                        rows.append(BenchRow(test, n_features, n_samples, na_ratio, n_threads, "gpu", mean, std,
                                             speedup))
    return rows


def render_rows(rows: list[BenchRow]) -> str:
    """Rows as CSV text with a header line (bench.py:218-242)."""
    lines = [",".join(BENCH_COLUMNS)]
    for r in rows:
        lines.append(",".join([r.test, str(r.features), str(r.samples), repr(r.na_ratio), str(r.threads), r.engine,
                               repr(r.mean_seconds), repr(r.std_seconds), repr(r.speedup)]))
    return "\n".join(lines) + "\n"


__all__ = ["BENCH_COLUMNS", "BENCH_REPS", "ENGINES", "BenchRow", "build_inputs", "render_rows", "run_bench"]
