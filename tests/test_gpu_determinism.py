"""Results never depend on how the pairs are partitioned (SPEC.md:469,
reference test_engine.py:441-462 / test_acceptance.py:281-295).

For every test, at sizes where the split-K factors of the FP64 contractions
are > 1 (Pearson F = 1000: 136 tiles < 2 x 148 CTAs; ANOVA / t-test with a
few hundred level rows), the full-range ``run()`` (upload-overlapped
incremental launches), the upload-then-compute order and the stitched
ranges of 2-, 4- and 8-way partitions (what 2/4/8 GPUs each compute) are
bitwise identical.  A pair's k-loop order is a function of the matrices only.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import bitwise_equal
import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import blocks, dist

CASES = {  # (kind_a, kind_b), F_a, F_b, S
    "pearson": (("continuous", None), 1000, None, 700),
    "spearman": (("continuous", None), 600, None, 1500),
    "chi2": (("categorical", None), 1000, None, 2000),
    "anova": (("categorical", "continuous"), 40, 1000, 3000),
    "ttest": (("dichotomous", "continuous"), 40, 1000, 3000),
    "kruskal": (("categorical", "continuous"), 40, 600, 3000),
    "mwu": (("dichotomous", "continuous"), 40, 600, 3000),
}


def _mats(test):
    (ka, kb), fa, fb, S = CASES[test]
    a = workloads.simulate(fa, S, ka, categories=7, na_ratio=0.15, seed=77 + len(test))
    if ka == "continuous":
        a[1] = np.round(a[1], 1)
    mat_a = ps.make_matrix(a, ka)
    mat_b = None
    if kb is not None:
        b = workloads.simulate(fb, S, kb, na_ratio=0.15, seed=78 + len(test))
        b[2] = np.round(b[2], 1)
        b[4] = 0.25  # constant column: exact-replay cells
        mat_b = ps.make_matrix(b, kb)
    return mat_a, mat_b


@pytest.mark.parametrize("test", sorted(CASES))
def test_partition_independent_bits(test, monkeypatch):
    mat_a, mat_b = _mats(test)
    canonical = ("stat", "p") + ps.EFFECTS_BY_TEST[test]
    req = ps.TestRequest(test, canonical)
    monkeypatch.delenv("PS_NO_OVERLAP", raising=False)
    full = ps.run(req, mat_a, mat_b)
    monkeypatch.setenv("PS_NO_OVERLAP", "1")
    seq = ps.run(req, mat_a, mat_b)
    for n in canonical:
        assert bitwise_equal(full[n], seq[n]), (test, n, "overlap")
    ka = mat_a.kind
    cat = mat_a.category_counts if ka != "continuous" else None
    da = blocks.DeviceMatrix(mat_a.values, ka, mat_a.na_sentinel, cat, presort=test == "spearman")
    db = None
    if mat_b is not None:
        db = blocks.DeviceMatrix(mat_b.values, mat_b.kind, mat_b.na_sentinel, None,
                                 presort=test in ("mwu", "kruskal"))
    shape = full["stat"].shape
    for world in (2, 4, 8):
        plan = dist.plan(test, mat_a.n_features, None if mat_b is None else mat_b.n_features, world)
        stitched = {n: np.full(shape, np.nan) for n in canonical}
        for lo, hi in plan:
            outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in canonical]
            blocks.block(test, da, db, lo, hi, outs)
            blocks.sync()
            own = dist.owned_mask(test, shape, lo, hi)
            for n, o in zip(canonical, outs):
                stitched[n][own] = o.cpu().numpy()[own]
        for n in canonical:
            assert bitwise_equal(stitched[n], full[n]), (test, n, world)
    da.close()
    if db is not None:
        db.close()
