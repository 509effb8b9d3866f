"""ctypes binding of the C ABI in ``include/pairstat_b200.h``.

The shared library ``libpairstat_b200.so`` is built in-tree (``csrc/Makefile``,
driven by ``__graft_entry__.build()``).  There is no CPU fallback: if the
library is missing, or no sm_100 device is visible, every compute call raises.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from pathlib import Path

import numpy as np

from .errors import PS_ERR_NO_DEVICE, raise_for_status

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
LIB_PATH = Path(os.environ["PS_LIB"]) if os.environ.get("PS_LIB") else PKG_DIR / "libpairstat_b200.so"

TEST_CODES = {
    "pearson": 0,
    "spearman": 1,
    "chi2": 2,
    "ttest": 3,
    "mwu": 4,
    "anova": 5,
    "kruskal": 6,
}
KIND_CODES = {"continuous": 0, "dichotomous": 1, "categorical": 2}
METHOD_CODES = {"bonferroni": 0, "bh": 1, "by": 2}
U_MODE_CODES = {"exact": 0, "asymptotic": 1, "auto": 2}

EXPORTED = (
    "ps_version",
    "ps_last_error",
    "ps_device_count",
    "ps_set_device",
    "ps_matrix_create",
    "ps_matrix_destroy",
    "ps_pearson_block",
    "ps_spearman_block",
    "ps_chi2_block",
    "ps_ttest_block",
    "ps_anova_block",
    "ps_mwu_block",
    "ps_kruskal_block",
    "ps_adjust",
    "ps_adjust_device",
    "ps_adjust_family_device",
    "ps_sync",
    "ps_by_factor",
    "ps_specfun_eval",
    "ps_run",
    "ps_kernel_launches",
    "ps_reset_kernel_launches",
    "ps_profile_enable",
    "ps_profile_collect",
    "ps_profile_collect_union",
    "ps_presort_layout",
    "ps_pearson_moments_used",
    "ps_matrix_attach_presort",
    "ps_matrix_presort_rows",
    "ps_matrix_presort_done",
    "ps_copy_h2d_2d",
    "ps_cells_count",
    "ps_cells_pack",
    "ps_cells_unpack",
    "ps_write_matrix",
    "ps_read_matrix",
    "ps_matrix_file_free",
)


class MatrixDesc(ctypes.Structure):
    _fields_ = [
        ("values", ctypes.c_void_p),
        ("n_features", ctypes.c_int64),
        ("n_samples", ctypes.c_int64),
        ("ld", ctypes.c_int64),
        ("na_sentinel", ctypes.c_double),
        ("kind", ctypes.c_int),
        ("category_counts", ctypes.c_void_p),
    ]


class MatrixFile(ctypes.Structure):
    """ps_matrix_file (include/pairstat_b200.h)."""

    _fields_ = [
        ("error", ctypes.c_int),
        ("os_errno", ctypes.c_int),
        ("n_rows", ctypes.c_int64),
        ("n_cols", ctypes.c_int64),
        ("values", ctypes.c_void_p),
        ("row_ids", ctypes.c_void_p),
        ("row_ids_len", ctypes.c_int64),
        ("col_ids", ctypes.c_void_p),
        ("col_ids_len", ctypes.c_int64),
        ("fallback", ctypes.c_void_p),
        ("n_fallback", ctypes.c_int64),
        ("err_row", ctypes.c_int64),
        ("err_col", ctypes.c_int64),
        ("err_count", ctypes.c_int64),
        ("err_cell", ctypes.c_void_p),
        ("err_cell_len", ctypes.c_int64),
        ("impl", ctypes.c_void_p),
    ]


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def build(force: bool = False) -> Path:
    """Compile the CUDA library in-tree with nvcc (sm_100a)."""
    cmd = ["make", "-s", "-C", str(CSRC), f"-j{os.cpu_count() or 4}"]
    if force:
        subprocess.run(["make", "-s", "-C", str(CSRC), "clean"], check=True)
    subprocess.run(cmd, check=True)
    return LIB_PATH


def _declare(lib: ctypes.CDLL) -> None:
    vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.ps_version.restype = ctypes.c_char_p
    lib.ps_last_error.restype = ctypes.c_char_p
    lib.ps_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.ps_set_device.argtypes = [i32]
    lib.ps_matrix_create.argtypes = [ctypes.POINTER(MatrixDesc), i32, i32, vp, ctypes.POINTER(vp)]
    lib.ps_matrix_destroy.argtypes = [vp]
    lib.ps_pearson_block.argtypes = [vp, i64, i64, dp, dp, dp, vp]
    lib.ps_spearman_block.argtypes = [vp, i64, i64, dp, dp, dp, vp]
    lib.ps_chi2_block.argtypes = [vp, i64, i64, dp, dp, dp, dp, vp]
    lib.ps_ttest_block.argtypes = [vp, vp, i64, i64, i32, dp, dp, dp, vp]
    lib.ps_anova_block.argtypes = [vp, vp, i64, i64, dp, dp, dp, vp]
    lib.ps_mwu_block.argtypes = [vp, vp, i64, i64, i32, dp, dp, dp, vp]
    lib.ps_kruskal_block.argtypes = [vp, vp, i64, i64, dp, dp, dp, vp]
    lib.ps_adjust.argtypes = [dp, i64, i64, i32, i32, dp]
    lib.ps_adjust_device.argtypes = [dp, i64, i64, i32, i32, dp, vp]
    lib.ps_adjust_family_device.argtypes = [dp, i64, i32, dp, vp]
    lib.ps_sync.argtypes = [vp]
    lib.ps_by_factor.argtypes = [i64]
    lib.ps_specfun_eval.argtypes = [i32, dp, i64, i32, dp]
    lib.ps_by_factor.restype = ctypes.c_double
    lib.ps_run.argtypes = [
        i32,
        ctypes.POINTER(MatrixDesc),
        ctypes.POINTER(MatrixDesc),
        i32,
        i32,
        ctypes.POINTER(ctypes.c_void_p),
        ctypes.POINTER(ctypes.c_void_p),
    ]
    lib.ps_kernel_launches.restype = ctypes.c_int64
    lib.ps_presort_layout.argtypes = [i64, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.ps_pearson_moments_used.argtypes = [i64, i64]
    lib.ps_matrix_attach_presort.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.ps_matrix_presort_rows.argtypes = [vp, i64, i64, vp]
    lib.ps_matrix_presort_done.argtypes = [vp, vp]
    lib.ps_copy_h2d_2d.argtypes = [vp, i64, vp, i64, i64, i64, vp]
    lib.ps_cells_count.argtypes = [i32, i32, i64, i64, i64, i64, ctypes.POINTER(ctypes.c_int64)]
    lib.ps_cells_pack.argtypes = [i32, i32, dp, i64, i64, i64, i64, dp, vp]
    lib.ps_cells_unpack.argtypes = [i32, i32, dp, i64, i64, i64, i64, dp, vp]
    lib.ps_write_matrix.argtypes = [ctypes.c_char_p, dp, i64, i64, vp, vp, ctypes.c_char]
    lib.ps_read_matrix.argtypes = [ctypes.c_char_p, ctypes.c_char, ctypes.POINTER(MatrixFile)]
    lib.ps_matrix_file_free.argtypes = [ctypes.POINTER(MatrixFile)]
    lib.ps_matrix_file_free.restype = None
    lib.ps_profile_enable.argtypes = [i32]
    lib.ps_profile_collect.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_int64)]
    lib.ps_profile_collect_union.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_int64)]


def profile_collect(name: str) -> tuple[float, int]:
    ms = ctypes.c_double(0.0)
    cnt = ctypes.c_int64(0)
    load().ps_profile_collect(name.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value


def load() -> ctypes.CDLL:
    """Load (never silently skip) the native library."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"native library {LIB_PATH} is missing; run __graft_entry__.build()"
                    " (the device path has no CPU fallback)"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            _declare(lib)
            _lib = lib
        return _lib


def last_error() -> str:
    msg = load().ps_last_error()
    return msg.decode() if msg else ""


def check(code: int) -> None:
    if code:
        raise_for_status(code, last_error())


def device_count() -> int:
    n = ctypes.c_int(0)
    load().ps_device_count(ctypes.byref(n))
    return n.value


def require_device() -> None:
    if device_count() == 0:
        raise_for_status(PS_ERR_NO_DEVICE, "no CUDA device visible; the B200 path has no CPU fallback")


def describe(mat, values: np.ndarray | None = None) -> tuple[MatrixDesc, tuple]:
    """A MatrixDesc over a DataMatrix's (host) values; returns keep-alive refs."""
    vals = np.ascontiguousarray(mat.values if values is None else values, dtype=np.float64)
    cats = None
    if mat.category_counts is not None:
        cats = np.ascontiguousarray(mat.category_counts, dtype=np.int64)
    sentinel = float(mat.na_sentinel)
    d = MatrixDesc(
        vals.ctypes.data,
        vals.shape[0],
        vals.shape[1],
        vals.shape[1],
        math.nan if math.isnan(sentinel) else sentinel,
        KIND_CODES[mat.kind],
        cats.ctypes.data if cats is not None else None,
    )
    return d, (vals, cats)


def by_factor(m: int) -> float:
    return float(load().ps_by_factor(int(m)))


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


def specfun(name: str, args) -> np.ndarray:
    """Evaluate a device special function on a batch (tests / diagnostics)."""
    which, nargs = SPECFUN_CODES[name]
    a = np.ascontiguousarray(np.asarray(args, dtype=np.float64).reshape(-1, nargs))
    out = np.empty(a.shape[0])
    check(load().ps_specfun_eval(which, a.ctypes.data, a.shape[0], nargs, out.ctypes.data))
    return out


def profile_collect_union(name: str) -> tuple[float, int]:
    """Busy time (union of launch intervals) and launch count of a kernel."""
    ms = ctypes.c_double(0.0)
    cnt = ctypes.c_int64(0)
    load().ps_profile_collect_union(name.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    return ms.value, cnt.value
