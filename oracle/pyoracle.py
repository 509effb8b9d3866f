"""ctypes front end of the C oracle (TEST INFRASTRUCTURE, never the product).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module.  ``oracle_run`` mirrors the reference ``engine.run``
(``pkg/src/pairstat/engine.py:415-557``) but dispatches to the C restatement
in ``oracle.c``; ``adjust_family`` restates ``adjust.py:23-87`` in numpy.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liborc.so"

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_int64_p = ctypes.POINTER(ctypes.c_int64)
_c_uint8_p = ctypes.POINTER(ctypes.c_uint8)

EFFECTS_BY_TEST = {
    "pearson": ("r2",),
    "spearman": ("rho",),
    "chi2": ("phi", "cramers_v"),
    "ttest": ("cohens_d",),
    "mwu": ("r",),
    "anova": ("partial_eta2",),
    "kruskal": ("eta2",),
}
ADJUSTED = {"p_bonferroni": "bonferroni", "p_bh": "bh", "p_by": "by"}
U_MODE_CODES = {"exact": 0, "asymptotic": 1, "auto": 2}
SPECFUN_CODES = {
    "ln_gamma": (0, 1),
    "reg_inc_beta": (1, 3),
    "reg_inc_gamma_upper": (2, 2),
    "normal_sf": (3, 1),
    "t_sf": (4, 2),
    "chi2_sf": (5, 2),
    "f_sf": (6, 3),
    "beta_sym_sf": (7, 2),
}


class OracleError(Exception):
    def __init__(self, code: int):
        super().__init__(f"oracle status {code}")
        self.code = code


def build() -> Path:
    """Compile liborc.so if missing or stale (gcc, no GPU needed)."""
    src = HERE / "oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(LIB_PATH))
    return _lib


def _dp(a):
    return None if a is None else a.ctypes.data_as(_c_double_p)


def _ip(a):
    return a.ctypes.data_as(_c_int64_p)


def _bp(a):
    return a.ctypes.data_as(_c_uint8_p)


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


def _check(code: int) -> None:
    if code:
        raise OracleError(code)


def specfun(name: str, args: np.ndarray) -> np.ndarray:
    which, nargs = SPECFUN_CODES[name]
    args = np.ascontiguousarray(np.asarray(args, dtype=np.float64).reshape(-1, nargs))
    out = np.empty(args.shape[0])
    code = lib().orc_specfun(
        ctypes.c_int(which), _dp(args), ctypes.c_int64(args.shape[0]), ctypes.c_int(nargs), _dp(out)
    )
    _check(code)
    return out


def presort(values: np.ndarray, present: np.ndarray, threads: int | None = None):
    F, S = values.shape
    orders = np.zeros((F, S), dtype=np.int64)
    svals = np.zeros((F, S), dtype=np.float64)
    lengths = np.zeros(F, dtype=np.int64)
    lib().orc_presort(
        _dp(values), _bp(present), ctypes.c_int64(F), ctypes.c_int64(S),
        _ip(orders), _dp(svals), _ip(lengths), ctypes.c_int(threads or default_threads()),
    )
    return orders, svals, lengths


def adjust_family(p: np.ndarray, method: str) -> np.ndarray:
    """Restates reference adjust.py:23-43 (stable argsort, m/i rounded first)."""
    out = np.full(p.shape, np.nan)
    defined = np.flatnonzero(~np.isnan(p))
    m = defined.size
    if m == 0:
        return out
    vals = p[defined]
    if method == "bonferroni":
        out[defined] = np.minimum(1.0, m * vals)
        return out
    scale = float(m)
    if method == "by":
        scale *= (1.0 / np.arange(1, m + 1)).sum()
    order = np.argsort(vals, kind="stable")
    ranked = vals[order] * (scale / np.arange(1, m + 1))
    stepped = np.minimum.accumulate(ranked[::-1])[::-1]
    out[defined[order]] = np.minimum(1.0, stepped)
    return out


def adjust(p_matrix: np.ndarray, method: str, symmetric: bool) -> np.ndarray:
    """Restates reference adjust.py:46-87."""
    p_matrix = np.asarray(p_matrix, dtype=np.float64)
    if not symmetric:
        return adjust_family(p_matrix.ravel(), method).reshape(p_matrix.shape)
    n = p_matrix.shape[0]
    iu = np.triu_indices(n, k=1)
    adj = adjust_family(p_matrix[iu], method)
    out = np.full_like(p_matrix, np.nan)
    out[iu] = adj
    out[iu[1], iu[0]] = adj
    return out


def _u8(present: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(present, dtype=np.uint8)


def compute(test: str, mat_a, mat_b=None, wanted=None, t_variant="student", u_mode="auto",
            threads: int | None = None, lo: int | None = None, hi: int | None = None):
    """Raw (unadjusted) outputs of one test, like the reference block kernels.

    ``wanted`` is the set of canonical outputs to fill; ``lo``/``hi`` bound the
    triangle rows (homogeneous), flat grid cells (ttest/anova) or continuous
    features (mwu/kruskal), exactly as the reference partitions its work.
    Returns dict name -> NaN-prefilled fp64 matrix.
    """
    threads = threads or default_threads()
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    wanted = set(canonical if wanted is None else wanted)
    homogeneous = mat_b is None
    shape = (mat_a.n_features, mat_a.n_features) if homogeneous else (mat_a.n_features, mat_b.n_features)
    outs = {n: (np.full(shape, np.nan) if n in wanted else None) for n in canonical}
    o = [_dp(outs[n]) for n in canonical]
    L = lib()
    S = ctypes.c_int64(mat_a.n_samples)
    th = ctypes.c_int(threads)
    if homogeneous:
        F = mat_a.n_features
        lo_, hi_ = (0 if lo is None else lo), (F if hi is None else hi)
        va = np.ascontiguousarray(mat_a.values)
        pa = _u8(mat_a.present)
        if test == "pearson":
            code = L.orc_pearson_block(_dp(va), _bp(pa), ctypes.c_int64(F), S, ctypes.c_int64(lo_),
                                       ctypes.c_int64(hi_), *o, th)
        elif test == "spearman":
            orders, svals, lengths = presort(va, pa, threads)
            code = L.orc_spearman_block(_ip(orders), _dp(svals), _ip(lengths), _bp(pa),
                                        ctypes.c_int64(F), S, ctypes.c_int64(lo_), ctypes.c_int64(hi_),
                                        *o, th)
        elif test == "chi2":
            cat = np.ascontiguousarray(mat_a.category_counts, dtype=np.int64)
            code = L.orc_chi2_block(_dp(va), _bp(pa), _ip(cat), ctypes.c_int64(F), S,
                                    ctypes.c_int64(lo_), ctypes.c_int64(hi_), *o, th)
        else:
            raise ValueError(test)
    else:
        Fc, Fq = mat_a.n_features, mat_b.n_features
        la = np.ascontiguousarray(mat_a.values)
        lp = _u8(mat_a.present)
        vb = np.ascontiguousarray(mat_b.values)
        vp = _u8(mat_b.present)
        if test in ("ttest", "anova"):
            lo_, hi_ = (0 if lo is None else lo), (Fc * Fq if hi is None else hi)
        else:
            lo_, hi_ = (0 if lo is None else lo), (Fq if hi is None else hi)
        c_fc, c_fq, c_lo, c_hi = (ctypes.c_int64(v) for v in (Fc, Fq, lo_, hi_))
        if test == "ttest":
            code = L.orc_ttest_block(_dp(la), _bp(lp), _dp(vb), _bp(vp), c_fc, c_fq, S, c_lo, c_hi,
                                     ctypes.c_int(1 if t_variant == "student" else 0), *o, th)
        elif test == "anova":
            cat = np.ascontiguousarray(mat_a.category_counts, dtype=np.int64)
            code = L.orc_anova_block(_dp(la), _bp(lp), _ip(cat), _dp(vb), _bp(vp), c_fc, c_fq, S,
                                     c_lo, c_hi, *o, th)
        elif test == "mwu":
            orders, svals, lengths = presort(vb, vp, threads)
            code = L.orc_mwu_block(_ip(orders), _dp(svals), _ip(lengths), _dp(la), _bp(lp), c_fc,
                                   c_fq, S, c_lo, c_hi, ctypes.c_int(U_MODE_CODES[u_mode]), *o, th)
        elif test == "kruskal":
            cat = np.ascontiguousarray(mat_a.category_counts, dtype=np.int64)
            orders, svals, lengths = presort(vb, vp, threads)
            code = L.orc_kruskal_block(_ip(orders), _dp(svals), _ip(lengths), _dp(la), _bp(lp),
                                       _ip(cat), c_fc, c_fq, S, c_lo, c_hi, *o, th)
        else:
            raise ValueError(test)
    _check(code)
    return outs


def oracle_run(request, mat_a, mat_b=None, threads: int | None = None) -> dict[str, np.ndarray]:
    """Full ``run`` semantics (engine.py:463-557) on the CPU oracle."""
    test = request.test
    needed = {n for n in request.outputs if n not in ADJUSTED}
    if any(n in ADJUSTED for n in request.outputs):
        needed.add("p")
    raw = compute(test, mat_a, mat_b, wanted=needed, t_variant=request.t_variant,
                  u_mode=request.u_mode, threads=threads)
    res = {}
    for name in request.outputs:
        if name in ADJUSTED:
            res[name] = adjust(raw["p"], ADJUSTED[name], symmetric=mat_b is None)
        else:
            res[name] = raw[name]
    return res


def block_runner(test: str, mat_a, mat_b=None, wanted=("stat", "p"), t_variant="student", u_mode="auto",
                 threads: int | None = None):
    """Timed CPU baseline of the reference's block kernels (bench.py only).

    Inputs are converted once and, for the rank tests, presorted once (the
    reference's engine.run presorts every feature once per run,
    engine.py:379-400); outputs are allocated once.  Returns
    ``(prep_seconds, run)`` where ``run(lo, hi)`` executes the block over
    the reference's range [lo, hi) and returns its wall seconds.
    """
    import time

    threads = threads or default_threads()
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    homogeneous = mat_b is None
    shape = (mat_a.n_features, mat_a.n_features) if homogeneous else (mat_a.n_features, mat_b.n_features)
    outs = {n: (np.full(shape, np.nan) if n in wanted else None) for n in canonical}
    o = [_dp(outs[n]) for n in canonical]
    L = lib()
    S = ctypes.c_int64(mat_a.n_samples)
    th = ctypes.c_int(threads)
    i64 = ctypes.c_int64
    if homogeneous:
        F = i64(mat_a.n_features)
        va = np.ascontiguousarray(mat_a.values)
        pa = _u8(mat_a.present)
        t0 = time.perf_counter()
        if test == "spearman":
            orders, svals, lengths = presort(va, pa, threads)
        prep = time.perf_counter() - t0
        cat = np.ascontiguousarray(mat_a.category_counts, dtype=np.int64) if test == "chi2" else None
    else:
        Fc, Fq = i64(mat_a.n_features), i64(mat_b.n_features)
        la = np.ascontiguousarray(mat_a.values)
        lp = _u8(mat_a.present)
        vb = np.ascontiguousarray(mat_b.values)
        vp = _u8(mat_b.present)
        cat = np.ascontiguousarray(mat_a.category_counts, dtype=np.int64) if test in ("anova", "kruskal") else None
        t0 = time.perf_counter()
        if test in ("mwu", "kruskal"):
            orders, svals, lengths = presort(vb, vp, threads)
        prep = time.perf_counter() - t0

    def run(lo: int, hi: int) -> float:
        c_lo, c_hi = i64(lo), i64(hi)
        t = time.perf_counter()
        if test == "pearson":
            code = L.orc_pearson_block(_dp(va), _bp(pa), F, S, c_lo, c_hi, *o, th)
        elif test == "spearman":
            code = L.orc_spearman_block(_ip(orders), _dp(svals), _ip(lengths), _bp(pa), F, S, c_lo, c_hi, *o, th)
        elif test == "chi2":
            code = L.orc_chi2_block(_dp(va), _bp(pa), _ip(cat), F, S, c_lo, c_hi, *o, th)
        elif test == "ttest":
            code = L.orc_ttest_block(_dp(la), _bp(lp), _dp(vb), _bp(vp), Fc, Fq, S, c_lo, c_hi,
                                     ctypes.c_int(1 if t_variant == "student" else 0), *o, th)
        elif test == "anova":
            code = L.orc_anova_block(_dp(la), _bp(lp), _ip(cat), _dp(vb), _bp(vp), Fc, Fq, S, c_lo, c_hi, *o, th)
        elif test == "mwu":
            code = L.orc_mwu_block(_ip(orders), _dp(svals), _ip(lengths), _dp(la), _bp(lp), Fc, Fq, S, c_lo, c_hi,
                                   ctypes.c_int(U_MODE_CODES[u_mode]), *o, th)
        else:
            code = L.orc_kruskal_block(_ip(orders), _dp(svals), _ip(lengths), _dp(la), _bp(lp), _ip(cat), Fc, Fq,
                                       S, c_lo, c_hi, *o, th)
        dt = time.perf_counter() - t
        _check(code)
        return dt

    run.outs = outs  # the (shared, NaN-prefilled) output matrices
    return prep, run
