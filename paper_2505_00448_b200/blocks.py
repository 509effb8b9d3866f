"""Device-resident block interface (the reference's block-kernel operator ABI).

The reference engine dispatches numba kernels ``_<test>_block(inputs, lo, hi,
want.., out..)`` over static row ranges (``pkg/src/pairstat/engine.py:133-352``,
``_execute`` at ``:360-376``).  This module exposes the same operators over
device memory: a :class:`DeviceMatrix` is the prepared, device-resident input
(validity bits, label codes, presort tables) and ``block(test, ...)`` fills
caller-owned device output matrices for one work range.  PyTorch is used only
to own device buffers and streams; all compute is in ``libpairstat_b200.so``.

This is what the multi-GPU driver (:mod:`.dist`) and bench.py call; ``run``
(:mod:`.engine`) is the host-buffer path.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib

HOMOGENEOUS = ("pearson", "spearman", "chi2")
PRESORT_A = ("spearman",)
PRESORT_B = ("mwu", "kruskal")


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return int(t.data_ptr())


def _stream_ptr(stream) -> int | None:
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


class DeviceMatrix:
    """A prepared ps_matrix on the current CUDA device.

    ``values`` is either a host numpy array (copied to the device) or a torch
    CUDA tensor of shape (F, ld) whose first ``n_samples`` columns hold the
    data (used in place when ``ld`` is a multiple of 32).
    """

    def __init__(self, values, kind: str, na_sentinel: float = math.nan,
                 category_counts: np.ndarray | None = None, n_samples: int | None = None,
                 presort: bool = False, stream=None):
        lib = _lib.load()
        self._keep = []
        on_device = not isinstance(values, np.ndarray)
        if on_device:
            F, ld = int(values.shape[0]), int(values.shape[1])
            S = int(n_samples if n_samples is not None else ld)
            ptr = _ptr(values)
            self._keep.append(values)
        else:
            arr = np.ascontiguousarray(values, dtype=np.float64)
            F, S = arr.shape
            ld = S
            ptr = arr.ctypes.data
            self._keep.append(arr)
        cats = None
        if category_counts is not None:
            cats = np.ascontiguousarray(category_counts, dtype=np.int64)
            self._keep.append(cats)
        desc = _lib.MatrixDesc(
            ptr, F, S, ld,
            math.nan if math.isnan(na_sentinel) else float(na_sentinel),
            _lib.KIND_CODES[kind],
            cats.ctypes.data if cats is not None else None,
        )
        handle = ctypes.c_void_p()
        _lib.check(lib.ps_matrix_create(ctypes.byref(desc), 1 if on_device else 0,
                                        1 if presort else 0, _stream_ptr(stream),
                                        ctypes.byref(handle)))
        self.handle = handle
        self.n_features = F
        self.n_samples = S
        self.kind = kind

    def presort_rows_only(self, f0: int, f1: int, stream=None) -> None:
        """Presort only features [f0, f1) -- enough for a rank-range of a
        Mann-Whitney / Kruskal-Wallis block, whose walk touches only the
        continuous features of its range."""
        self.presort_sharded(0, 1, rows=(f0, f1), stream=stream)

    def presort_sharded(self, rank: int, world: int, gather=None, stream=None, rows=None) -> None:
        """Presort this rank's share of the features and all-gather the rows.

        Multi-GPU: instead of every rank presorting all F
        features, rank r presorts rows [r*c, (r+1)*c) (c = ceil(F / world))
        into torch-owned tables and ``gather(name, full, local)`` fills
        ``full`` with every rank's rows (``torch.distributed.
        all_gather_into_tensor`` on byte views by default; NCCL over NVLink).  Rows are independent,
        so the result equals a single-device presort bit for bit.
        """
        import torch

        lib = _lib.load()
        ldo, ldt = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(lib.ps_presort_layout(self.n_samples, ctypes.byref(ldo), ctypes.byref(ldt)))
        c = -(-self.n_features // world)
        nrows = c * world
        dev = torch.device("cuda", torch.cuda.current_device())
        widths = {"order": (ldo.value, torch.int16), "inv": (ldo.value, torch.int16),
                  "tb": (ldt.value, torch.int32), "lastb": (ldt.value, torch.int16),
                  "nextb": (ldt.value, torch.int16), "tied": (1, torch.uint8), "len": (1, torch.int32)}
        tabs = {k: torch.zeros((nrows, w), dtype=dt, device=dev) for k, (w, dt) in widths.items()}
        self._keep.append(tabs)
        self.presort_tables = tabs
        s = _stream_ptr(stream)
        _lib.check(lib.ps_matrix_attach_presort(self.handle, *[_ptr(tabs[k]) for k in widths], s))
        f0, f1 = (rank * c, min(self.n_features, (rank + 1) * c)) if rows is None else rows
        if f1 > f0:
            _lib.check(lib.ps_matrix_presort_rows(self.handle, f0, f1, s))
        if world > 1:
            if gather is None:
                import torch.distributed as tdist

                def gather(name, full, local):
                    tdist.all_gather_into_tensor(full, local)
            sync(stream)  # the rows are complete before the collective reads them
            for name, t in tabs.items():
                b = t.view(torch.uint8).view(nrows, -1)
                gather(name, b, b[rank * c:(rank + 1) * c])
            torch.cuda.synchronize()  # the collectives ran on another stream
        _lib.check(lib.ps_matrix_presort_done(self.handle, s))

    @classmethod
    def from_datamatrix(cls, mat, presort: bool = False, stream=None) -> "DeviceMatrix":
        return cls(mat.values, mat.kind, mat.na_sentinel, mat.category_counts,
                   presort=presort, stream=stream)

    def close(self) -> None:
        if self.handle:
            _lib.load().ps_matrix_destroy(self.handle)
            self.handle = ctypes.c_void_p()
            self._keep.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def block(test: str, a: DeviceMatrix, b: DeviceMatrix | None, lo: int, hi: int, outs,
          t_variant: str = "student", u_mode: str = "auto", stream=None) -> None:
    """Fill device outputs (canonical order: stat, p, effect(s)) for one range.

    Range units follow the reference: triangle rows for homogeneous tests,
    flat grid cells for ttest/anova, continuous features for mwu/kruskal.
    """
    lib = _lib.load()
    o = [_ptr(x) for x in outs] + [None] * (4 - len(outs))
    s = _stream_ptr(stream)
    if test == "pearson":
        code = lib.ps_pearson_block(a.handle, lo, hi, o[0], o[1], o[2], s)
    elif test == "spearman":
        code = lib.ps_spearman_block(a.handle, lo, hi, o[0], o[1], o[2], s)
    elif test == "chi2":
        code = lib.ps_chi2_block(a.handle, lo, hi, o[0], o[1], o[2], o[3], s)
    elif test == "ttest":
        code = lib.ps_ttest_block(a.handle, b.handle, lo, hi, 1 if t_variant == "student" else 0,
                                  o[0], o[1], o[2], s)
    elif test == "anova":
        code = lib.ps_anova_block(a.handle, b.handle, lo, hi, o[0], o[1], o[2], s)
    elif test == "mwu":
        code = lib.ps_mwu_block(a.handle, b.handle, lo, hi, _lib.U_MODE_CODES[u_mode],
                                o[0], o[1], o[2], s)
    elif test == "kruskal":
        code = lib.ps_kruskal_block(a.handle, b.handle, lo, hi, o[0], o[1], o[2], s)
    else:
        raise ValueError(f"unknown test {test!r}")
    _lib.check(code)


def adjust_device(p, rows: int, cols: int, method: str, symmetric: bool, out, stream=None) -> None:
    _lib.check(_lib.load().ps_adjust_device(_ptr(p), rows, cols, _lib.METHOD_CODES[method],
                                            1 if symmetric else 0, _ptr(out), _stream_ptr(stream)))


def adjust_family_device(p, n: int, method: str, out, stream=None) -> None:
    _lib.check(_lib.load().ps_adjust_family_device(_ptr(p), n, _lib.METHOD_CODES[method], _ptr(out),
                                                   _stream_ptr(stream)))


def sync(stream=None) -> None:
    """Wait for the stream and raise the first device-side error, if any."""
    _lib.check(_lib.load().ps_sync(_stream_ptr(stream)))


def full_range(test: str, a: DeviceMatrix, b: DeviceMatrix | None) -> tuple[int, int]:
    if test in HOMOGENEOUS:
        return 0, a.n_features
    if test in ("ttest", "anova"):
        return 0, a.n_features * b.n_features
    return 0, b.n_features
