"""Device path against the golden fixtures (no oracle in the loop).

* device special functions vs the mpmath 50-digit grids at the reference's
  accuracy budget (1e-12 relative; lnGamma 1e-13) -- the device versions of
  specfun.py must pass the same grids the CPU ones do;
* run() vs the reference's own outputs on seeded inputs (run_fixtures.npz):
  identical NaN pattern; statistics bit-exact where the survey shows the
  reference is exactly reproducible (Spearman, chi2, KW, MWU) and within the
  north-star tolerances elsewhere; p within 1e-6 relative or 1e-12 absolute;
* the hand-derived known answers of the reference tests.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import known_answers
from conftest import bitwise_equal, max_rel, p_close, same_nan

pytestmark = pytest.mark.gpu

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200 import _lib

GOLDEN = Path(__file__).parent / "golden"
EXACT_STATS = {"spearman": ("stat", "rho"), "chi2": ("stat", "phi", "cramers_v"),
               "kruskal": ("stat", "eta2"), "mwu": ("stat", "r")}


@pytest.mark.parametrize("name", list(_lib.SPECFUN_CODES))
def test_device_specfun_golden(name):
    rows = np.array(json.loads((GOLDEN / "specfun_mp.json").read_text())[name])
    got = _lib.specfun(name, rows[:, :-1])
    want = rows[:, -1]
    rel = np.where(want == 0, np.abs(got), np.abs(got - want) / np.abs(np.where(want == 0, 1, want)))
    assert float(rel.max()) <= (1e-13 if name == "ln_gamma" else 1e-12)


def _cases():
    data = np.load(GOLDEN / "run_fixtures.npz")
    return [str(c) for c in data["cases"]]


@pytest.mark.parametrize("case", _cases())
def test_device_run_matches_reference_outputs(case):
    data = np.load(GOLDEN / "run_fixtures.npz")
    test = case.split("_")[0]
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    mat_a = ps.make_matrix(data[f"{case}__a"], kind_a)
    mat_b = ps.make_matrix(data[f"{case}__b"], kind_b) if kind_b else None
    outs = ps.outputs_for(test)
    got = ps.run(ps.TestRequest(test, outs), mat_a, mat_b)
    for name in outs:
        want = data[f"{case}__{name}"]
        assert same_nan(got[name], want), (case, name)
        if name in EXACT_STATS.get(test, ()):
            assert bitwise_equal(got[name], want), (case, name)
        elif name.startswith("p"):
            assert p_close(got[name], want), (case, name)
        else:
            assert max_rel(got[name], want, floor=1e-3) <= 1e-9, (case, name)


@pytest.mark.parametrize("case", known_answers.CASES, ids=[c[0] for c in known_answers.CASES])
def test_device_known_answers(case):
    test, mat_a, mat_b, cell, want = known_answers.build(case, ps)
    got = ps.run(ps.TestRequest(test, tuple(want)), mat_a, mat_b)
    for name, (value, tol) in want.items():
        assert abs(got[name][cell] - value) <= max(tol, 1e-12 * abs(value)), (name, got[name][cell], value)
