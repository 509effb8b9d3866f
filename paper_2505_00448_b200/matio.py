"""Delimited matrix files with feature and sample identifiers.

Drop-in for the reference's ``pairstat.matio`` (``pkg/src/pairstat/matio.py``):
same functions, file format and error messages.  ``write_matrix`` and
``read_matrix`` run in native code (``ps_write_matrix`` / ``ps_read_matrix``
of the C ABI, ``csrc/ps_matio.cu``; host cores only, no device needed), which
formats and parses rows on all host cores -- the reference formats every
value with a Python f-string, the bottleneck of writing a large result
matrix.  The bytes written are identical to the
reference writer's; the reader accepts exactly what the reference accepts
(Python ``float()`` grammar, ``str.splitlines()`` line boundaries).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .errors import PS_ERR_IO

#: File extensions that switch the delimiter to tab (matio.py:21).
_TAB_EXTENSIONS = (".tsv", ".tab")


def delimiter_for(path: str) -> str:
    """Delimiter implied by a file name's extension (matio.py:24-27)."""
    ext = os.path.splitext(path)[1].lower()
    return "\t" if ext in _TAB_EXTENSIONS else ","


def format_value(value: float) -> str:
    """Serialize one float at full round-trip precision (matio.py:30-32)."""
    return f"{value:.17g}"


def default_ids(prefix: str, count: int) -> list[str]:
    """Generated identifiers f0..fN or s0..sN (matio.py:35-37)."""
    return [f"{prefix}{i}" for i in range(count)]


def _id_array(ids, n):
    enc = [str(ids[i]).encode("utf-8") for i in range(n)]  # IndexError as the reference
    return (ctypes.c_char_p * max(n, 1))(*enc), enc


def write_matrix(path: str, values: np.ndarray, row_ids: list[str] | None = None,
                 col_ids: list[str] | None = None, delimiter: str | None = None) -> None:
    """Write one matrix with identifiers to a delimited text file (matio.py:40-72)."""
    values = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    n_rows, n_cols = values.shape
    sep = delimiter_for(path) if delimiter is None else delimiter
    sep_b = sep.encode("utf-8")
    if len(sep_b) != 1 or (col_ids is not None and len(col_ids) != n_cols):
        _write_python(path, values, row_ids, col_ids, sep)  # shapes the native writer does not take
        return
    rows_arr = cols_arr = None
    keep = []
    if row_ids is not None:
        rows_arr, k = _id_array(row_ids, n_rows)
        keep.append(k)
    if col_ids is not None:
        cols_arr, k = _id_array(col_ids, n_cols)
        keep.append(k)
    lib = _lib.load()
    code = lib.ps_write_matrix(os.fsencode(path), values.ctypes.data, n_rows, n_cols,
                               ctypes.cast(rows_arr, ctypes.c_void_p) if rows_arr is not None else None,
                               ctypes.cast(cols_arr, ctypes.c_void_p) if cols_arr is not None else None,
                               sep_b)
    del keep
    if code == PS_ERR_IO:
        with open(path, "w", newline="\n"):  # raises the OSError the reference's open() raises
            pass
    _lib.check(code)


def _write_python(path, values, row_ids, col_ids, sep):
    """The reference algorithm, for delimiters / id lists the native writer does not take."""
    n_rows, n_cols = values.shape
    if row_ids is None:
        row_ids = default_ids("f", n_rows)
    if col_ids is None:
        col_ids = default_ids("s", n_cols)
    lines = [sep.join([""] + list(col_ids))]
    for i in range(n_rows):
        cells = [row_ids[i]]
        cells.extend(format_value(v) for v in values[i])
        lines.append(sep.join(cells))
    with open(path, "w", newline="\n") as handle:
        handle.write("\n".join(lines))
        handle.write("\n")


def _read_python(path, sep):
    """The reference algorithm, for multi-byte delimiters."""
    with open(path, "r", newline="") as handle:
        lines = handle.read().splitlines()
    if not lines:
        raise ValueError(f"{path}: empty matrix file")
    header = lines[0].split(sep)
    col_ids = header[1:]
    n_cols = len(col_ids)
    row_ids, rows = [], []
    for i, line in enumerate(lines[1:], start=2):
        if not line:
            continue
        cells = line.split(sep)
        if len(cells) != n_cols + 1:
            raise ValueError(f"{path}: row {i} has {len(cells) - 1} values, expected {n_cols}")
        row_ids.append(cells[0])
        parsed = []
        for j, cell in enumerate(cells[1:], start=1):
            try:
                parsed.append(float(cell))
            except ValueError:
                raise ValueError(f"{path}: malformed numeric cell at row {i}, column {j}: {cell!r}") from None
        rows.append(parsed)
    values = np.array(rows, dtype=np.float64)
    if values.size == 0:
        values = values.reshape(0, n_cols)
    return values, row_ids, col_ids


def read_matrix(path: str, delimiter: str | None = None) -> tuple[np.ndarray, list[str], list[str]]:
    """Read one matrix with identifiers from a delimited text file (matio.py:75-125).

    Raises ValueError for an empty file, ragged rows or a malformed cell
    (reported with its row and column), OSError when the file cannot be read.
    """
    sep = delimiter_for(path) if delimiter is None else delimiter
    sep_b = sep.encode("utf-8")
    if len(sep_b) != 1:
        return _read_python(path, sep)
    with open(path, "rb"):  # the OSError the reference's open() raises
        pass
    lib = _lib.load()
    res = _lib.MatrixFile()
    code = lib.ps_read_matrix(os.fsencode(path), sep_b, ctypes.byref(res))
    try:
        if code != 0:
            if res.os_errno:
                raise OSError(res.os_errno, os.strerror(res.os_errno), path)
            _lib.check(code)
        if res.error == 1:
            raise ValueError(f"{path}: empty matrix file")
        if res.error in (2, 3) and res.n_fallback:
            # non-ASCII cells before the error come first in file order
            flat = np.ctypeslib.as_array(ctypes.cast(res.fallback, ctypes.POINTER(ctypes.c_int64)),
                                         shape=(res.n_fallback,)).copy()
            scratch = np.zeros((int(flat.max()) // max(res.n_cols, 1) + 1, max(res.n_cols, 1)))
            _parse_fallback(path, sep, scratch, flat, max(res.n_cols, 1))
        if res.error == 2:
            raise ValueError(f"{path}: row {res.err_row} has {res.err_count} values, expected {res.n_cols}")
        if res.error == 3:
            cell = ctypes.string_at(res.err_cell, res.err_cell_len).decode("utf-8")
            raise ValueError(f"{path}: malformed numeric cell at row {res.err_row},"
                             f" column {res.err_col}: {cell!r}")
        n_rows, n_cols = res.n_rows, res.n_cols
        if n_rows * n_cols == 0:
            n_rows = 0  # the reference's values.reshape(0, n_cols) for an empty array
        if n_rows * n_cols:
            values = np.ctypeslib.as_array(ctypes.cast(res.values, ctypes.POINTER(ctypes.c_double)),
                                           shape=(n_rows * n_cols,)).copy().reshape(n_rows, n_cols)
        else:
            values = np.zeros((n_rows, n_cols), dtype=np.float64)
        rid = ctypes.string_at(res.row_ids, res.row_ids_len).decode("utf-8").split("\0")[:-1] \
            if res.row_ids_len else []
        cid = ctypes.string_at(res.col_ids, res.col_ids_len).decode("utf-8").split("\0")[:-1] \
            if res.col_ids_len else []
        if res.n_fallback:
            # non-ASCII cells: Python's own float() (Unicode digits / spaces)
            flat = np.ctypeslib.as_array(ctypes.cast(res.fallback, ctypes.POINTER(ctypes.c_int64)),
                                         shape=(res.n_fallback,)).copy()
            _parse_fallback(path, sep, values, flat, n_cols)
        return values, rid, cid
    finally:
        lib.ps_matrix_file_free(ctypes.byref(res))


def _parse_fallback(path, sep, values, flat, n_cols):
    with open(path, "r", newline="") as handle:
        lines = handle.read().splitlines()
    data_lines = [(i, line) for i, line in enumerate(lines[1:], start=2) if line]
    for k in flat:
        r, c = divmod(int(k), n_cols)
        i, line = data_lines[r]
        cell = line.split(sep)[c + 1]
        try:
            values[r, c] = float(cell)
        except ValueError:
            raise ValueError(f"{path}: malformed numeric cell at row {i}, column {c + 1}: {cell!r}") from None


def roundtrip_equal(a: np.ndarray, b: np.ndarray) -> bool:
    """True when two float matrices match bit for bit (matio.py:128-135)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        return False
    return bool((a.view(np.int64) == b.view(np.int64)).all())


__all__ = ["default_ids", "delimiter_for", "format_value", "read_matrix", "roundtrip_equal", "write_matrix"]
