"""Shared pytest setup.

Markers: ``gpu`` tests need a B200 (they are the parity tests proper and go
through the C ABI); everything else runs on the CPU-only builder box.
The CPU oracle (oracle/, test infrastructure) is importable from here only.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 device")


@pytest.fixture(scope="session")
def oracle():
    import pyoracle

    pyoracle.build()
    return pyoracle


def same_nan(a: np.ndarray, b: np.ndarray) -> bool:
    return bool(np.array_equal(np.isnan(a), np.isnan(b)))


def bitwise_equal(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(((a.view(np.int64) == b.view(np.int64)) | both_nan).all())


def max_rel(a: np.ndarray, b: np.ndarray, floor: float = 0.0) -> float:
    m = ~np.isnan(b)
    if not m.any():
        return 0.0
    d = np.abs(a[m] - b[m])
    scale = np.maximum(np.abs(b[m]), floor)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(scale > 0, d / scale, d)
    r = np.where(np.isinf(a[m]) & np.isinf(b[m]) & (a[m] == b[m]), 0.0, r)
    return float(np.nanmax(r)) if r.size else 0.0


def p_close(got: np.ndarray, want: np.ndarray, rtol: float = 1e-6, atol: float = 1e-12) -> bool:
    """North-star p-value rule: <= 1e-6 relative OR <= 1e-12 absolute."""
    m = ~np.isnan(want)
    d = np.abs(got[m] - want[m])
    return bool(np.all((d <= atol) | (d <= rtol * np.abs(want[m]))))


@pytest.fixture(scope="session")
def gpu_available() -> bool:
    try:
        from paper_2505_00448_b200 import _lib

        return _lib.device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if os.environ.get("PS_FORCE_GPU_TESTS"):
        return
