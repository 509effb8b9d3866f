"""matio parity: the native writer / reader against
files written and parsed by the REFERENCE (tests/golden/make_matio_golden.py),
plus the reference's own test_matio cases restated.  CPU only."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2505_00448_b200 import matio

GOLD = Path(__file__).resolve().parent / "golden" / "matio"
EXP = json.loads((GOLD / "expected.json").read_text())


@pytest.mark.parametrize("name", sorted(EXP["write"]))
def test_writer_bytes_match_reference(tmp_path, name):
    spec = dict(EXP["write"][name])
    vals = spec.pop("values")
    if vals == "special.npy":
        values = np.load(GOLD / "special.npy")
    elif name == "empty_rows.csv":
        values = np.zeros((0, 3))
    elif name == "empty_cols.csv":
        values = np.zeros((2, 0))
    else:
        values = np.load(GOLD / "special.npy")[:2, :2]
    out = tmp_path / name
    matio.write_matrix(str(out), values, **spec)
    assert out.read_bytes() == (GOLD / name).read_bytes()


@pytest.mark.parametrize("name", sorted(EXP["read"]))
def test_reader_matches_reference(name):
    want = EXP["read"][name]
    path = str(GOLD / name)
    if "error" in want:
        with pytest.raises(ValueError) as e:
            matio.read_matrix(path)
        assert str(e.value) == want["error"].replace("{path}", path)
        return
    values, rid, cid = matio.read_matrix(path)
    assert list(values.shape) == want["shape"]
    assert values.view(np.int64).ravel().tolist() == want["bits"]
    assert rid == want["row_ids"] and cid == want["col_ids"]


def test_large_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(4)
    v = rng.standard_normal((300, 257)) * 10.0 ** rng.integers(-300, 300, (300, 257))
    v[rng.random(v.shape) < 0.05] = np.nan
    p = str(tmp_path / "big.tsv")
    matio.write_matrix(p, v)
    back, rid, cid = matio.read_matrix(p)
    assert matio.roundtrip_equal(v, back)
    assert rid == matio.default_ids("f", 300) and cid == matio.default_ids("s", 257)


# ---- the reference's tests/test_matio.py cases ----------------------------

def test_delimiter_and_ids():
    assert matio.delimiter_for("x.tsv") == "\t" and matio.delimiter_for("x.TSV") == "\t"
    assert matio.delimiter_for("x.tab") == "\t" and matio.delimiter_for("x.csv") == ","
    assert matio.default_ids("f", 3) == ["f0", "f1", "f2"] and matio.default_ids("s", 0) == []
    assert matio.format_value(float("nan")) == "nan"
    assert matio.format_value(float("-inf")) == "-inf"


def test_header_corner_and_newlines(tmp_path):
    p = tmp_path / "m.csv"
    matio.write_matrix(str(p), np.zeros((2, 2)))
    raw = p.read_bytes()
    assert raw.startswith(b",s0,s1\n") and b"\r" not in raw and raw.endswith(b"\n")


def test_read_errors(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text(",s0,s1\nf0,1.0,oops\n")
    with pytest.raises(ValueError, match="row 2, column 2"):
        matio.read_matrix(str(bad))
    with pytest.raises(OSError):
        matio.read_matrix(str(tmp_path / "nope.csv"))
    with pytest.raises(OSError):
        matio.write_matrix(str(tmp_path / "no" / "dir.csv"), np.zeros((1, 1)))


def test_exports_match_reference_surface():
    assert set(matio.__all__) == {"default_ids", "delimiter_for", "format_value", "read_matrix",
                                  "roundtrip_equal", "write_matrix"}


@pytest.mark.parametrize("later", ["ragged", "malformed_ascii", "malformed_same_row"])
def test_first_error_in_file_order_with_non_ascii_cells(tmp_path, later):
    """A malformed NON-ASCII cell (parsed by Python's float()) before a later
    ragged row / malformed ASCII cell: the reference raises for the first bad
    cell in file order (advisor finding), so must the native reader."""
    import paper_2505_00448_b200 as ps

    lines = ["\tc0\tc1", "r0\t1.5\t2.5", "r1\t١٢x\t3.0"]  # arabic digits + junk: not a float
    if later == "ragged":
        lines.append("r2\t1.0")
    elif later == "malformed_ascii":
        lines.append("r2\tabc\t1.0")
    else:
        lines[2] = "r1\t١٢x\tabc"
    p = tmp_path / "m.tsv"
    p.write_text("\n".join(lines) + "\n", encoding="utf-8")
    with pytest.raises(ValueError, match="row 3, column 1"):
        ps.read_matrix(str(p))
