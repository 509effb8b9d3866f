"""Exact Mann-Whitney U pinned to the reference (tests/golden/mwu_exact.npz,
made by tests/golden/make_mwu_exact_golden.py from pairstat.run and the
reference's enumeration permutation_mwu): the CPU oracle (here) and the
device (``-m gpu``) must reproduce the reference's outputs bit for bit --
U, the exact DP p (mixed.py:231-247, :348-358), r, BH and Bonferroni -- and
the exact p must equal full enumeration (test_acceptance.py:110-130)."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from conftest import bitwise_equal

GOLDEN = Path(__file__).resolve().parent / "golden" / "mwu_exact.npz"
OUTS = ("stat", "p", "r", "p_bh", "p_bonferroni")


def _cases():
    return [str(c) for c in np.load(GOLDEN)["cases"]]


def _case(case):
    import paper_2505_00448_b200 as ps

    d = np.load(GOLDEN)
    la = ps.make_matrix(d[f"{case}__a"], "dichotomous")
    va = ps.make_matrix(d[f"{case}__b"], "continuous")
    req = ps.TestRequest("mwu", OUTS, u_mode=str(d[f"{case}__mode"]))
    want = {n: d[f"{case}__{n}"] for n in OUTS}
    perm = d[f"{case}__perm_p"] if f"{case}__perm_p" in d.files else None
    return req, la, va, want, perm


def test_fixture_exercises_the_exact_branch():
    d = np.load(GOLDEN)
    # the enumeration cells: reference exact p == brute-force enumeration
    n_enum = 0
    for case in _cases():
        if case.startswith("enum"):
            perm = d[f"{case}__perm_p"]
            m = ~np.isnan(perm)
            assert np.array_equal(d[f"{case}__p"][m], perm[m]), case
            n_enum += int(m.sum())
    assert n_enum == 135
    # auto mode at S = 40 takes the exact branch for small tie-free groups:
    # its p differs from the asymptotic run there
    pa, pz = d["auto40_auto__p"], d["auto40_asymptotic__p"]
    assert np.count_nonzero(pa != pz) >= 30


@pytest.mark.parametrize("case", _cases())
def test_oracle_matches_reference_exact_u(oracle, case):
    req, la, va, want, _ = _case(case)
    got = oracle.oracle_run(req, la, va)
    for n in OUTS:
        assert bitwise_equal(got[n], want[n]), (case, n)


@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases())
def test_device_matches_reference_exact_u(case):
    """U and r bit for bit; p bit for bit on the exact-branch cells (the DP
    is integer arithmetic), within the p tolerance on the asymptotic ones
    (CUDA vs glibc erfc ulps)."""
    import paper_2505_00448_b200 as ps
    from conftest import p_close, same_nan

    req, la, va, want, perm = _case(case)
    got = ps.run(req, la, va)
    for n in ("stat", "r"):
        assert bitwise_equal(got[n], want[n]), (case, n)
    d = np.load(GOLDEN)
    if case.startswith("auto40"):
        exact_cells = d["auto40_auto__p"] != d["auto40_asymptotic__p"]
        if case.endswith("asymptotic"):
            exact_cells[:] = False
    else:
        exact_cells = ~np.isnan(want["p"])
    assert bitwise_equal(np.where(exact_cells, got["p"], 0.0), np.where(exact_cells, want["p"], 0.0)), case
    for n in ("p", "p_bh", "p_bonferroni"):
        assert same_nan(got[n], want[n]) and p_close(got[n], want[n], rtol=2e-6), (case, n)
    if perm is not None:
        m = ~np.isnan(perm)
        assert np.array_equal(got["p"][m], perm[m])


@pytest.mark.gpu
def test_device_exact_list_overflow_rescans_every_cell(monkeypatch):
    """More exact-eligible cells than the exact list holds (PS_EXACT_CAP=3):
    mwu_exact_kernel re-decides every cell instead of dropping p-values."""
    import paper_2505_00448_b200 as ps

    case = "exact64"
    req, la, va, want, _ = _case(case)
    monkeypatch.setenv("PS_EXACT_CAP", "3")
    got = ps.run(req, la, va)
    for n in ("stat", "p", "r"):  # every p of this case is exact-branch
        assert bitwise_equal(got[n], want[n]), (case, n)
