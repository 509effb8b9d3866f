"""C-ABI boundary checks that need no GPU: the shared library loads, exports
every symbol include/pairstat_b200.h declares, host-only helpers work, and the
compute path fails loudly (never a CPU fallback) when no device is visible."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2505_00448_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "pairstat_b200.h"

pytestmark = pytest.mark.skipif(not _lib.LIB_PATH.exists(), reason="native library not built")


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ps_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_block_operators():
    syms = declared_symbols()
    for test in ("pearson", "spearman", "chi2", "ttest", "anova", "mwu", "kruskal"):
        assert f"ps_{test}_block" in syms
    assert {"ps_run", "ps_adjust", "ps_adjust_device", "ps_matrix_create", "ps_matrix_destroy"} <= set(syms)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_lib.EXPORTED) <= set(declared_symbols())


def test_version_string():
    assert b"sm_100a" in _lib.load().ps_version()


def test_by_factor_is_numpy_pairwise():
    for m in [1, 5, 8, 64, 129, 4096, 99999]:
        assert _lib.by_factor(m) == float((1.0 / np.arange(1, m + 1)).sum())


def test_no_cpu_fallback_without_device():
    if _lib.device_count() > 0:
        pytest.skip("a device is visible")
    import paper_2505_00448_b200 as ps

    mat = ps.make_matrix(np.random.default_rng(1).normal(size=(3, 20)), "continuous")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ps.run(ps.TestRequest("pearson", ("stat",)), mat)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        ps.adjust(np.zeros((3, 3)), "bh", symmetric=True)
