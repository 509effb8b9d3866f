"""Race evidence by repetition (compute-sanitizer is closed on this GPU pool:
profiles/r02/compute_sanitizer_closed.txt).

Every kernel family that shares memory between warps or CTAs -- mbarrier
rings and TMA multicast of the 2-CTA chi-squared GEMM, shared-memory
atomics and block scans of the rank walks, split-K partials, the per-chunk
incremental launches on four walk streams overlapping the upload, the BH
radix passes -- is run repeatedly on the same inputs, alternating the
overlapped and sequential schedules; every repetition must reproduce the
first bit for bit.  A data race that changes a value shows up as a
mismatch; integer results (counts, ranks, tables) leave no slack for one.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bitwise_equal
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps

REPS = 6


def _inputs(test):
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    fa, S = (900, 4000) if kind_b is None else (40, 6000)
    if test == "chi2":
        fa = 600
    a = workloads.simulate(fa, S, kind_a, categories=9, na_ratio=0.15, seed=91)
    b = workloads.simulate(700, S, kind_b, na_ratio=0.15, seed=92) if kind_b else None
    if b is not None:
        b[::7] = np.round(b[::7], 1)
    elif kind_a == "continuous":
        a[::5] = np.round(a[::5], 1)
    return ps.make_matrix(a, kind_a), (ps.make_matrix(b, kind_b) if b is not None else None)


@pytest.mark.parametrize("test", ps.TESTS)
def test_repeated_runs_are_bit_identical(test, monkeypatch):
    ma, mb = _inputs(test)
    outs = ("stat", "p", "p_bh") + ps.EFFECTS_BY_TEST[test]
    req = ps.TestRequest(test, outs)
    first = ps.run(req, ma, mb)
    for i in range(REPS):
        if i % 2:
            monkeypatch.setenv("PS_NO_OVERLAP", "1")
        else:
            monkeypatch.delenv("PS_NO_OVERLAP", raising=False)
        again = ps.run(req, ma, mb)
        for n in outs:
            assert bitwise_equal(again[n], first[n]), (test, n, i)
