"""Compare the Spearman walk with and without group tables (PS_SPEARMAN_NOTAB)
on small tied inputs; prints the first differing cells."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2505_00448_b200 as ps  # noqa: E402

rng = np.random.default_rng(1)
for F, S, dec in ((4, 40, 0), (13, 150, 1), (6, 300, 1), (30, 2000, 1), (8, 40000, 1)):
    x = np.round(rng.standard_normal((F, S)) * 2, dec)
    x[rng.random((F, S)) < 0.2] = np.nan
    x[1] = rng.standard_normal(S)  # one untied row
    m = ps.make_matrix(x, "continuous")
    req = ps.TestRequest("spearman", ("rho",))
    os.environ.pop("PS_SPEARMAN_NOTAB", None)
    a = ps.run(req, m)["rho"]
    os.environ["PS_SPEARMAN_NOTAB"] = "1"
    b = ps.run(req, m)["rho"]
    os.environ.pop("PS_SPEARMAN_NOTAB", None)
    bad = np.argwhere(~((a == b) | (np.isnan(a) & np.isnan(b))))
    print(F, S, "mismatches", len(bad), [(int(i), int(j), a[i, j], b[i, j]) for i, j in bad[:6]])
