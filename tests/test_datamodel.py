"""Host-side data model: the drop-in API surface (reference datamodel.py,
engine.py validation, adjust.py argument checks).  CPU only."""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_2505_00448_b200 as ps
from paper_2505_00448_b200.datamodel import present_mask


def test_exports_match_reference_surface():
    want = {"BASE_OUTPUTS", "EFFECTS_BY_TEST", "KINDS", "KINDS_BY_TEST", "TESTS", "DataMatrix",
            "ResultSet", "TestRequest", "adjust", "make_matrix", "outputs_for", "run", "__version__",
            "DomainError", "EmptyMatrix", "ExactModeWithTies", "InfeasibleSimulation", "KindMismatch",
            "LabelOutOfRange", "NegativeLabel", "NonConvergence", "NonIntegerCategoryLabel",
            "NonSquareSymmetric", "PairstatError", "SampleCountMismatch", "TableTooLarge", "TooLarge",
            "UnknownMethod", "UnsupportedOutputForTest"}
    assert want <= set(ps.__all__)
    for name in want:
        assert hasattr(ps, name)
    for cls in ("DomainError", "EmptyMatrix", "LabelOutOfRange", "UnknownMethod"):
        assert issubclass(getattr(ps, cls), ps.PairstatError)


def test_vocabulary():
    assert ps.TESTS == ("pearson", "spearman", "chi2", "ttest", "mwu", "anova", "kruskal")
    assert ps.outputs_for("chi2") == ("stat", "p", "p_bonferroni", "p_bh", "p_by", "phi", "cramers_v")


def test_present_mask_bit_exact_sentinel():
    v = np.array([0.0, -0.0, 1.0, np.nan])
    assert present_mask(v, -0.0).tolist() == [True, False, True, True]
    assert present_mask(v, 0.0).tolist() == [False, True, True, True]
    assert present_mask(v, math.nan).tolist() == [True, True, True, False]


def test_make_matrix_orientation_and_counts():
    raw = np.array([[0.0, 1.0], [2.0, 1.0], [np.nan, 0.0]])  # samples x features
    m = ps.make_matrix(raw, "categorical", features_on_rows=False)
    assert m.values.shape == (2, 3)
    assert m.category_counts.tolist() == [3, 2]
    assert not m.values.flags.writeable
    d = ps.make_matrix(np.array([[0.0, 0.0, np.nan]]), "dichotomous")
    assert d.category_counts.tolist() == [2]
    e = ps.make_matrix(np.array([[np.nan, np.nan]]), "categorical")
    assert e.category_counts.tolist() == [0]


@pytest.mark.parametrize("raw,kind,exc,match", [
    (np.zeros((0, 3)), "continuous", ps.EmptyMatrix, "non-empty"),
    (np.zeros(3), "continuous", ps.EmptyMatrix, "2-D"),
    (np.array([[0.5, 1.0]]), "categorical", ps.NonIntegerCategoryLabel, "non-integer"),
    (np.array([[-1.0, 1.0]]), "categorical", ps.NegativeLabel, "negative"),
    (np.array([[0.0, 2.0]]), "dichotomous", ps.LabelOutOfRange, "0 or 1"),
    (np.array([[0.0, 1.0]]), "bogus", ValueError, "unknown kind"),
])
def test_make_matrix_errors(raw, kind, exc, match):
    with pytest.raises(exc, match=match):
        ps.make_matrix(raw, kind)


def test_request_validation():
    with pytest.raises(ps.UnsupportedOutputForTest, match="cohens_d"):
        ps.TestRequest("pearson", ("cohens_d",))
    with pytest.raises(ValueError, match="unknown test"):
        ps.TestRequest("bogus", ("stat",))
    with pytest.raises(ValueError, match="variant"):
        ps.TestRequest("ttest", ("stat",), t_variant="x")
    with pytest.raises(ValueError, match="mode"):
        ps.TestRequest("mwu", ("stat",), u_mode="x")
    with pytest.raises(ValueError, match="threads"):
        ps.TestRequest("mwu", ("stat",), threads=0)
    with pytest.raises(ValueError, match="outputs"):
        ps.TestRequest("mwu", ())


def test_resultset_shape_check():
    with pytest.raises(ValueError, match="shape"):
        ps.ResultSet(matrices={"stat": np.zeros((2, 2))}, shape=(3, 3))


def test_run_validation_before_device():
    """Kind / shape checks happen on the host, with the reference's messages."""
    cont = ps.make_matrix(np.random.default_rng(0).normal(size=(3, 40)), "continuous")
    cat = ps.make_matrix(np.zeros((2, 40)), "categorical")
    short = ps.make_matrix(np.zeros((2, 30)), "continuous")
    with pytest.raises(ValueError, match="single matrix"):
        ps.run(ps.TestRequest("pearson", ("stat",)), cont, cont)
    with pytest.raises(ValueError, match="second"):
        ps.run(ps.TestRequest("anova", ("stat",)), cat)
    with pytest.raises(ps.KindMismatch, match="categorical"):
        ps.run(ps.TestRequest("chi2", ("stat",)), cont)
    with pytest.raises(ps.KindMismatch, match="dichotomous"):
        ps.run(ps.TestRequest("ttest", ("stat",)), cat, cont)
    with pytest.raises(ps.SampleCountMismatch, match="40"):
        ps.run(ps.TestRequest("anova", ("stat",)), cat, short)


def test_adjust_validation_on_host():
    with pytest.raises(ps.UnknownMethod, match="holm"):
        ps.adjust(np.zeros((2, 2)), "holm", symmetric=True)
    with pytest.raises(ps.NonSquareSymmetric, match="square"):
        ps.adjust(np.zeros((2, 3)), "bh", symmetric=True)
    with pytest.raises(ValueError, match="2-D"):
        ps.adjust(np.zeros(3), "bh", symmetric=False)
