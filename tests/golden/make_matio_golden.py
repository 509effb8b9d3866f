"""Golden fixtures for matio parity: files written by the REFERENCE writer and
the reference reader's parse of crafted inputs.

Run once in the build container (needs /root/reference):
    python tests/golden/make_matio_golden.py
Outputs tests/golden/matio/*: the reference-written files (bytes), crafted
input files, and expected.json (parsed values as int64 bit patterns, ids,
error messages with the path replaced by {path}).
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "matio"
sys.path.insert(0, "/root/reference/pkg/src")
from pairstat import matio as ref  # noqa: E402


def special_matrix():
    rng = np.random.default_rng(20251019)
    v = rng.standard_normal((6, 9)) * 10.0 ** rng.integers(-8, 9, (6, 9))
    v[0, :9] = [np.nan, np.inf, -np.inf, 0.0, -0.0, 5e-324, 1.7976931348623157e308, 1e16, 1e17]
    v[1, :8] = [0.1, 1e-4, 1e-5, 123456789012345678.0, -2.5, 3.0, 1.0 / 3.0, 2.0 ** -1074]
    v[2, :3] = [-np.nan, float.fromhex("0x1.fffffffffffffp-1"), 9.999999999999999e22]
    return v


def main():
    OUT.mkdir(exist_ok=True)
    exp = {"write": {}, "read": {}}
    v = special_matrix()
    np.save(OUT / "special.npy", v)
    cases = {
        "special.csv": dict(values=v),
        "special_ids.tsv": dict(values=v, row_ids=[f"row{i}" for i in range(6)],
                                col_ids=[f"c{j}" for j in range(9)]),
        "empty_rows.csv": dict(values=np.zeros((0, 3))),
        "empty_cols.csv": dict(values=np.zeros((2, 0))),
        "unicode_ids.csv": dict(values=v[:2, :2], row_ids=["α", "β"], col_ids=["x y", "z"]),
    }
    for name, kw in cases.items():
        ref.write_matrix(str(OUT / name), **kw)
        exp["write"][name] = {k: (val if k != "values" else None) for k, val in kw.items()}
    exp["write"]["special.csv"]["values"] = "special.npy"
    exp["write"]["special_ids.tsv"]["values"] = "special.npy"
    # crafted inputs for the reader
    crafted = {
        "crlf.csv": b",a,b\r\nr1,1.5,nan\r\n\r\nr2, 2.5 ,-inf\r\n",
        "cr_only.csv": b",a\rr1,1\rr2,2\r",
        "vt_ff.csv": b",a\x0br1,1\x0cr2,3\x1cr3,4\x1dr4,5\x1er5,6\n",
        "unicode_breaks.csv": ",a r1,1 r2,2\x85r3,3\n".encode("utf-8"),
        "spellings.csv": b",a,b,c,d,e,f\nr,+inf,-Infinity,NaN,-nan,1_000.5,.5\nq,5.,1e1_0,1E-3,+0,-0,0007\n",
        "whitespace.tsv": b"\ta\tb\nr\t \t1.25\x0b\t3\n",
        "no_trailing_newline.csv": b",a\nr,1",
        "empty_header.csv": b"\nr\n",
        "unicode_digits.csv": ",a\nr,٣.٥\n".encode("utf-8"),
        "bad_underscore.csv": b",a\nr,1__0\n",
        "bad_hex.csv": b",a\nr,0x10\n",
        "bad_text.csv": b",s0,s1\nf0,1.0,oops\n",
        "bad_empty_cell.csv": b",a,b\nr,1,\n",
        "ragged.csv": b",s0,s1,s2\nf0,1,2,3\nf1,4,5\n",
        "empty.csv": b"",
        "blank_lines_only.csv": b"\n\n",
    }
    for name, data in crafted.items():
        (OUT / name).write_bytes(data)
        try:
            vals, rid, cid = ref.read_matrix(str(OUT / name))
            exp["read"][name] = {"shape": list(vals.shape), "bits": vals.view(np.int64).ravel().tolist(),
                                 "row_ids": rid, "col_ids": cid}
        except ValueError as e:
            exp["read"][name] = {"error": str(e).replace(str(OUT / name), "{path}")}
    (OUT / "expected.json").write_text(json.dumps(exp, indent=1, ensure_ascii=False))
    print("wrote", len(cases), "writer fixtures and", len(crafted), "reader fixtures to", OUT)


if __name__ == "__main__":
    main()
