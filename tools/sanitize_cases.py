"""Small cases that reach every kernel family, for compute-sanitizer runs.

usage: compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_cases.py [case ...]

Each case goes through the public ``run`` (C ABI ``ps_run``) and, where a
second code path exists, through the block operators too.  Shapes are the
smallest that still select each kernel variant (tile kernels with several
tiles, the shared-memory and global presorts, tied / tie-free walks, the
tcgen05 cluster GEMM, the exact-U DP, each BH size class).  No parity checks
here: the pytest suite does that; this only gives the sanitizers coverage.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2505_00448_b200 as ps  # noqa: E402
import workloads  # noqa: E402


def _cont(F, S, na=0.15, seed=0, ties=False):
    x = workloads.simulate(F, S, "continuous", na_ratio=na, seed=seed)
    if ties:
        x[: F // 2] = np.round(x[: F // 2], 1)
    return ps.make_matrix(x, "continuous")


def _lab(F, S, c, na=0.1, seed=1, kind="categorical"):
    return ps.make_matrix(workloads.simulate(F, S, kind, categories=c, na_ratio=na, seed=seed), kind)


def case_pearson():
    x = workloads.simulate(150, 700, "continuous", na_ratio=0.2, seed=3)
    x[0] = 0.1  # constant row: exact replay kernel
    m = ps.make_matrix(x, "continuous")
    ps.run(ps.TestRequest("pearson", ("stat", "p", "r2", "p_bh", "p_bonferroni", "p_by")), m)


def case_spearman():
    ps.run(ps.TestRequest("spearman", ("stat", "p", "p_bh")), _cont(90, 3000, ties=True))
    ps.run(ps.TestRequest("spearman", ("stat", "p")), _cont(12, 21000, ties=True, seed=4))  # global presort


def case_chi2():
    ps.run(ps.TestRequest("chi2", ("stat", "p", "phi", "cramers_v", "p_bh")), _lab(70, 3000, 6))


def case_group():
    lab = _lab(9, 1500, 4)
    val = _cont(40, 1500, seed=5)
    ps.run(ps.TestRequest("anova", ("stat", "p", "partial_eta2", "p_bh")), lab, val)
    lab2 = _lab(9, 1500, 2, kind="dichotomous")
    for v in ("student", "welch"):
        ps.run(ps.TestRequest("ttest", ("stat", "p", "cohens_d"), t_variant=v), lab2, val)


def case_rank():
    lab = _lab(9, 1500, 5)
    val = _cont(40, 1500, ties=True, seed=6)
    ps.run(ps.TestRequest("kruskal", ("stat", "p", "eta2", "p_bh")), lab, val)
    lab2 = _lab(9, 1500, 2, kind="dichotomous")
    ps.run(ps.TestRequest("mwu", ("stat", "p", "r")), lab2, val)
    # exact U (tie-free, n <= 64)
    lab3 = _lab(6, 40, 2, na=0.0, kind="dichotomous", seed=8)
    val3 = _cont(5, 40, na=0.0, seed=9)
    ps.run(ps.TestRequest("mwu", ("stat", "p", "r"), u_mode="exact"), lab3, val3)


def case_adjust():
    rng = np.random.default_rng(2)
    for n in (300, 40000, 300000):
        p = rng.random(n)
        p[rng.random(n) < 0.05] = np.nan
        p[: n // 10] = np.round(p[: n // 10], 3)
        for meth in ("bonferroni", "bh", "by"):
            ps.adjust(p.reshape(1, -1), meth, symmetric=False)


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("case", n, "ok", flush=True)
