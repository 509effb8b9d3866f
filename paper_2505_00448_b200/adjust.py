"""``adjust``: Bonferroni / Benjamini-Hochberg / Benjamini-Yekutieli on the B200.

Drop-in for ``pkg/src/pairstat/adjust.py:46-87``: same argument checks and
messages on the host, then the family extraction, radix sort, step-up scan and
scatter run on the device (``csrc/ps_adjust.cu``).  Output is bit-identical to
the reference for the same input matrix.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import NonSquareSymmetric, UnknownMethod

METHODS = ("bonferroni", "bh", "by")


def adjust(p_matrix: np.ndarray, method: str, symmetric: bool) -> np.ndarray:
    """Adjust a matrix of p-values; NaN cells are untested and stay NaN."""
    if method not in METHODS:
        raise UnknownMethod(f"unknown adjustment method {method!r}; expected one of {METHODS}")
    p = np.ascontiguousarray(np.asarray(p_matrix, dtype=np.float64))
    if p.ndim != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {p.shape}")
    rows, cols = p.shape
    if symmetric and rows != cols:
        raise NonSquareSymmetric(
            f"symmetric adjustment needs a square matrix, got {rows}x{cols}"
        )
    out = np.empty_like(p)
    if p.size == 0:
        return out
    lib = _lib.load()
    _lib.require_device()
    code = lib.ps_adjust(
        p.ctypes.data, rows, cols, _lib.METHOD_CODES[method], 1 if symmetric else 0, out.ctypes.data
    )
    _lib.check(code)
    return out
