"""Device block API on sub-ranges (the multi-GPU shard path, one GPU here).

Each rank of ``dist.sharded_run`` calls ``blocks.block`` on its own range
(reference ``engine.py:70-125`` partitions).  Running every range of a
3-way plan on one device and stitching the owned cells must reproduce the
full-range result bit for bit -- this exercises the kernels' range handling
(triangle-row tiles of the chi-square stream-K GEMM, Spearman g-row chunks,
flat-cell ranges of the moment contractions, continuous-feature ranges of the
rank walks) with the same code a multi-GPU run uses.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import workloads

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import blocks, dist

CASES = {
    "pearson": (("continuous", None), 60, None, 700),
    "spearman": (("continuous", None), 50, None, 900),
    "chi2": (("categorical", None), 140, None, 1500),
    "anova": (("categorical", "continuous"), 9, 70, 800),
    "ttest": (("dichotomous", "continuous"), 7, 60, 800),
    "kruskal": (("categorical", "continuous"), 9, 50, 800),
    "mwu": (("dichotomous", "continuous"), 7, 40, 800),
}


def _device_outputs(test, da, db, shape, lo, hi):
    n = 2 + len(ps.EFFECTS_BY_TEST[test])
    outs = [torch.full(shape, float("nan"), dtype=torch.float64, device="cuda") for _ in range(n)]
    blocks.block(test, da, db, lo, hi, outs)
    blocks.sync()
    return [o.cpu().numpy() for o in outs]


@pytest.mark.parametrize("test", sorted(CASES))
def test_block_ranges_stitch_to_full(oracle, test):
    (ka, kb), fa, fb, S = CASES[test]
    rng_seed = 1000 + len(test)
    a = workloads.simulate(fa, S, ka, categories=9, na_ratio=0.15, seed=rng_seed)
    mat_a = ps.make_matrix(a, ka)
    mat_b = None
    if kb is not None:
        b = workloads.simulate(fb, S, kb, na_ratio=0.15, seed=rng_seed + 1)
        mat_b = ps.make_matrix(b, kb)
    cat = mat_a.category_counts if ka != "continuous" else None
    presort_a = test == "spearman"
    presort_b = test in ("mwu", "kruskal")
    da = blocks.DeviceMatrix(mat_a.values, ka, mat_a.na_sentinel, cat, presort=presort_a)
    db = None
    if mat_b is not None:
        db = blocks.DeviceMatrix(mat_b.values, kb, mat_b.na_sentinel, None, presort=presort_b)
    shape = (fa, fa) if mat_b is None else (fa, fb)
    lo, hi = blocks.full_range(test, da, db)
    full = _device_outputs(test, da, db, shape, lo, hi)
    plan = dist.plan(test, fa, None if mat_b is None else fb, 3)
    stitched = [np.full(shape, np.nan) for _ in full]
    for (r0, r1) in plan:
        part = _device_outputs(test, da, db, shape, r0, r1)
        own = dist.owned_mask(test, shape, r0, r1)
        for k in range(len(full)):
            stitched[k][own] = part[k][own]
    for k in range(len(full)):
        f = full[k].view(np.uint64)
        s = stitched[k].view(np.uint64)
        assert np.array_equal(f, s), (test, k)
    # and the full-range device result agrees with the oracle's statistic
    req = ps.TestRequest(test, ("stat", "p"))
    ref = oracle.oracle_run(req, mat_a, mat_b)
    assert np.array_equal(np.isnan(full[0]), np.isnan(ref["stat"]))
    m = ~np.isnan(ref["stat"])
    np.testing.assert_allclose(full[0][m], ref["stat"][m], rtol=1e-9, atol=1e-12)
    da.close()
    if db is not None:
        db.close()


@pytest.mark.parametrize("test,S", [("spearman", 900), ("spearman", 25000), ("kruskal", 900)])
def test_sharded_presort_matches_single_device(oracle, test, S):
    """Multi-GPU presort (each rank presorts its rows, then an all-gather),
    emulated for 2 ranks on one device: the gathered tables give results
    bit-identical to a single-device presort."""
    F = 37
    cont = workloads.simulate(F, S, "continuous", na_ratio=0.2, seed=S + 5)
    cont[3] = np.round(cont[3], 1)  # ties
    mat = ps.make_matrix(cont, "continuous")
    lab = None
    if test == "kruskal":
        lab = ps.make_matrix(workloads.simulate(6, S, "categorical", categories=5, na_ratio=0.1, seed=3),
                             "categorical")
    ref_dm = blocks.DeviceMatrix(mat.values, "continuous", mat.na_sentinel, presort=True)
    r1 = blocks.DeviceMatrix(mat.values, "continuous", mat.na_sentinel)
    r1.presort_sharded(1, 2, gather=lambda name, full, local: None)
    r0 = blocks.DeviceMatrix(mat.values, "continuous", mat.na_sentinel)
    c = -(-F // 2)

    def gather0(name, full, local):
        other = r1.presort_tables[name].view(torch.uint8).view(full.shape[0], -1)
        full[c:2 * c].copy_(other[c:2 * c])

    r0.presort_sharded(0, 2, gather=gather0)
    for k, t in r0.presort_tables.items():
        assert t.shape[0] >= F
    if test == "spearman":
        shape = (F, F)
        a_ref, a_sh = _device_outputs(test, ref_dm, None, shape, 0, F), _device_outputs(test, r0, None, shape, 0, F)
    else:
        dl = blocks.DeviceMatrix(lab.values, "categorical", lab.na_sentinel, lab.category_counts)
        shape = (6, F)
        a_ref = _device_outputs(test, dl, ref_dm, shape, 0, F)
        a_sh = _device_outputs(test, dl, r0, shape, 0, F)
    for x, y in zip(a_ref, a_sh):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    for d in (ref_dm, r0, r1):
        d.close()


@pytest.mark.parametrize("test", ["kruskal", "mwu"])
def test_rank_walk_with_rows_only_presort(test):
    """A rank of a mixed rank test presorts only its continuous features."""
    S, Fq = 700, 30
    kind = "categorical" if test == "kruskal" else "dichotomous"
    lab = ps.make_matrix(workloads.simulate(5, S, kind, categories=4, na_ratio=0.1, seed=9), kind)
    cont = workloads.simulate(Fq, S, "continuous", na_ratio=0.2, seed=11)
    cont[12] = np.round(cont[12])
    mat = ps.make_matrix(cont, "continuous")
    dl = blocks.DeviceMatrix(lab.values, kind, lab.na_sentinel, lab.category_counts)
    full = blocks.DeviceMatrix(mat.values, "continuous", mat.na_sentinel, presort=True)
    part = blocks.DeviceMatrix(mat.values, "continuous", mat.na_sentinel)
    part.presort_rows_only(10, 20)
    shape = (5, Fq)
    a = _device_outputs(test, dl, full, shape, 10, 20)
    b = _device_outputs(test, dl, part, shape, 10, 20)
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))
    for d in (dl, full, part):
        d.close()
