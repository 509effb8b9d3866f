"""Hand-derived known answers from the reference tests, restated as matrix inputs.

Each case: (name, test, raw_a, raw_b, sentinel, (row, col), {output: (value, tol)}).
Sources: test_continuous.py:18-40 (Pearson r = 0.6, p = 0.4 after deletion),
test_categorical.py:35-43 (chi2 = 10, p = erfc(sqrt 5), phi = V = 1),
test_mixed.py:362-367 (ANOVA F = 16, p = 0.025094573304390855, eta2 = 32/35),
test_mixed.py:422-427 (KW H = 8/7, p = exp(-4/7), eta2 = -2/7),
test_acceptance.py:170-180 (Spearman perfect monotone rho = 1, p = 0).
"""

import math

import numpy as np

CASES = [
    ("pearson_deletion", "pearson",
     np.array([[1.0, 2.0, 3.0, 4.0, 5.0, -9.0], [2.0, 1.0, 4.0, 3.0, -9.0, 7.0]]), None, -9.0, (0, 1),
     {"stat": (0.6, 1e-15), "p": (0.4, 1e-14)}),
    ("pearson_identical", "pearson",
     np.array([[1.0, 2.0, 3.0, 4.0, 5.0], [1.0, 2.0, 3.0, 4.0, 5.0]]), None, math.nan, (0, 1),
     {"stat": (1.0, 0.0), "p": (0.0, 0.0)}),
    ("chi2_perfect", "chi2",
     np.array([[0.0] * 5 + [1.0] * 5, [0.0] * 5 + [1.0] * 5]), None, math.nan, (0, 1),
     {"stat": (10.0, 1e-13), "p": (math.erfc(math.sqrt(5.0)), 1e-12 * math.erfc(math.sqrt(5.0))),
      "phi": (1.0, 1e-14), "cramers_v": (1.0, 1e-14)}),
    ("anova_hand", "anova",
     np.array([[0.0, 0.0, 1.0, 1.0, 2.0, 2.0]]), np.array([[1.0, 2.0, 3.0, 4.0, 5.0, 6.0]]), math.nan, (0, 0),
     {"stat": (16.0, 1e-13), "p": (0.025094573304390855, 1e-12 * 0.025094573304390855),
      "partial_eta2": (32 / 35, 1e-14)}),
    ("kruskal_hand", "kruskal",
     np.array([[0.0, 1.0, 2.0, 0.0, 1.0, 2.0]]), np.array([[1.0, 2.0, 3.0, 4.0, 5.0, 6.0]]), math.nan, (0, 0),
     {"stat": (8 / 7, 1e-14), "p": (math.exp(-4 / 7), 1e-12), "eta2": (-2 / 7, 1e-13)}),
    ("spearman_monotone", "spearman",
     np.array([[1.0, 2.0, 3.0, 4.0, 5.0], [2.0, 4.0, 5.0, 7.0, 9.0]]), None, math.nan, (0, 1),
     {"stat": (1.0, 0.0), "p": (0.0, 0.0)}),
]


def build(case, ps):
    name, test, a, b, sent, cell, want = case
    kind_a, kind_b = ps.KINDS_BY_TEST[test]
    mat_a = ps.make_matrix(a, kind_a, na_sentinel=sent)
    mat_b = ps.make_matrix(b, kind_b, na_sentinel=sent) if b is not None else None
    return test, mat_a, mat_b, cell, want
