"""``run``: the drop-in replacement of the reference ``engine.run``.

Reference: ``pkg/src/pairstat/engine.py:415-557``.  Host-side work is limited
to the reference's argument checks (kinds ``:441-461``, sample counts) and the
allocation of the requested result matrices; everything else -- validity
masks, presorting, every pairwise statistic, p-values and the Bonferroni / BH /
BY adjustments -- runs on the B200 behind one C-ABI call (``ps_run``).  There
is no CPU fallback: without the native library or a device, ``run`` raises.

``request.threads`` is accepted and ignored (results never depend on it, as in
the reference, ``SPEC.md:469``).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .datamodel import EFFECTS_BY_TEST, KINDS_BY_TEST, DataMatrix, ResultSet, TestRequest
from .errors import KindMismatch, SampleCountMismatch

ADJUSTED_OUTPUTS = {"p_bonferroni": "bonferroni", "p_bh": "bh", "p_by": "by"}
_ADJ_ORDER = ("p_bonferroni", "p_bh", "p_by")

# A dichotomous feature is a two-category feature (engine.py:51-57).
_ACCEPTED_KINDS = {
    "continuous": ("continuous",),
    "dichotomous": ("dichotomous",),
    "categorical": ("categorical", "dichotomous"),
}


def _check_kind(test: str, role: str, got: str, expected: str) -> None:
    if got not in _ACCEPTED_KINDS[expected]:
        raise KindMismatch(f"test {test!r} needs a {expected} {role}, got {got}")


def validate(request: TestRequest, mat_a: DataMatrix, mat_b: DataMatrix | None) -> tuple[int, int]:
    """The reference's pre-flight checks; returns the result shape."""
    test = request.test
    kind_a, kind_b = KINDS_BY_TEST[test]
    if kind_b is None:
        if mat_b is not None:
            raise ValueError(f"test {test!r} takes a single matrix")
        _check_kind(test, "matrix", mat_a.kind, kind_a)
        return (mat_a.n_features, mat_a.n_features)
    if mat_b is None:
        raise ValueError(f"test {test!r} needs a second, continuous matrix")
    _check_kind(test, "first matrix", mat_a.kind, kind_a)
    _check_kind(test, "second matrix", mat_b.kind, kind_b)
    if mat_a.n_samples != mat_b.n_samples:
        raise SampleCountMismatch(
            f"sample counts differ: first matrix has {mat_a.n_samples},"
            f" second has {mat_b.n_samples}"
        )
    return (mat_a.n_features, mat_b.n_features)


def device_list(devices) -> tuple[int, ...]:
    """TestRequest.devices as a tuple of device ids (validated against the
    visible devices)."""
    ids = tuple(range(devices)) if isinstance(devices, int) else tuple(devices)
    n = _lib.device_count()
    bad = [d for d in ids if d >= n]
    if bad:
        raise ValueError(f"devices {bad} not visible ({n} CUDA device(s))")
    return ids


def run(request: TestRequest, mat_a: DataMatrix, mat_b: DataMatrix | None = None) -> ResultSet:
    """Run one pairwise test on the B200 and return the requested matrices."""
    shape = validate(request, mat_a, mat_b)
    lib = _lib.load()
    _lib.require_device()
    devices = device_list(request.devices)
    if len(devices) > 1:  # one process, several local GPUs (dist.local_run)
        from .dist import local_run

        return local_run(request, mat_a, mat_b, devices)
    if devices[0] != 0:
        _lib.check(lib.ps_set_device(devices[0]))
    test = request.test
    canonical = ("stat", "p") + EFFECTS_BY_TEST[test]
    raw = {n: np.empty(shape) for n in request.outputs if n not in ADJUSTED_OUTPUTS}
    adj = {n: np.empty(shape) for n in request.outputs if n in ADJUSTED_OUTPUTS}
    outs = (ctypes.c_void_p * 4)(
        *[raw[n].ctypes.data if n in raw else None for n in canonical] + [None] * (4 - len(canonical))
    )
    adj_outs = (ctypes.c_void_p * 3)(*[adj[n].ctypes.data if n in adj else None for n in _ADJ_ORDER])
    desc_a, keep_a = _lib.describe(mat_a)
    desc_b, keep_b = (None, None)
    if mat_b is not None:
        desc_b, keep_b = _lib.describe(mat_b)
    code = lib.ps_run(
        _lib.TEST_CODES[test],
        ctypes.byref(desc_a),
        ctypes.byref(desc_b) if desc_b is not None else None,
        0 if request.t_variant == "student" else 1,
        _lib.U_MODE_CODES[request.u_mode],
        outs,
        adj_outs,
    )
    del keep_a, keep_b
    _lib.check(code)
    matrices = {}
    for name in request.outputs:
        matrices[name] = adj[name] if name in adj else raw[name]
    return ResultSet(matrices=matrices, shape=shape)
