"""Run one device step of a BASELINE config (for ncu / compute-sanitizer).

usage: python tools/profile_one.py --config 2 [--test spearman] [--scale 1.0] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2505_00448_b200 import blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=bench.parse_config, default=2)
    ap.add_argument("--test", default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    if args.config == 5 and args.scale != 1.0:
        cfg = workloads.config(5, scale=args.scale)
        a, b, ka, kb, test = cfg["a"], None, "continuous", None, "pearson"
    else:
        wl = bench.Workload(args.config, args.test or bench.default_test(args.config), 0, 1)
        a, b, ka, kb, test = wl.a_full, wl.b_full, wl.kind_a, wl.kind_b, wl.test
    cat = bench.label_counts(a) if ka != "continuous" else None
    homog = b is None
    shape = (a.shape[0], a.shape[0]) if homog else (a.shape[0], b.shape[0])
    outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(4)]
    for _ in range(args.reps):
        da = blocks.DeviceMatrix(a, ka, workloads.SENTINEL, cat, presort=test == "spearman")
        db = None
        if b is not None:
            db = blocks.DeviceMatrix(b, kb, workloads.SENTINEL, None, presort=test in ("mwu", "kruskal"))
        lo, hi = blocks.full_range(test, da, db)
        blocks.block(test, da, db, lo, hi, outs[: 2 + (2 if test == "chi2" else 1)])
        blocks.sync()
        da.close()
        if db is not None:
            db.close()
    torch.cuda.synchronize()
    print("ok", test, shape, float(np.nanmean(outs[0].cpu().numpy())))




def dump_walk_cycles():
    import ctypes
    import os

    from paper_2505_00448_b200 import _lib

    lib = _lib.load()
    if not os.environ.get("PS_LIB") or not hasattr(lib, "ps_debug_walk_cycles"):
        return
    buf = (ctypes.c_ulonglong * 40)()
    lib.ps_debug_walk_cycles(buf)
    names = ["wait+prefetch", "passA phase1", "scanA", "passA phase2", "scanB", "passB", "reduce+final"]
    tot = sum(buf[i] for i in range(32)) or 1
    for cls, cname in enumerate(["untied", "tied g", "tied h", "tied both"]):
        n = buf[32 + cls]
        c = sum(buf[cls * 8 + i] for i in range(7))
        print(f"{cname:10s} pairs {n:9d}  share {100.0 * c / tot:5.1f}%  cycles/pair {c / max(n, 1):9.0f}")
        for i, nm in enumerate(names):
            print(f"    {nm:16s} {buf[cls * 8 + i] / max(n, 1):9.0f}")


if __name__ == "__main__":
    main()
    dump_walk_cycles()
