"""A/B an environment switch of the library on one device-resident block call.

usage: python tools/ab_env.py --test pearson --F 6000 --S 100000 --env PS_PEARSON_RAW=1 [--reps 3]
Times blocks.block over the full range (CUDA events, after a warm-up) with
and without the variable set, alternating, and prints both medians; the
outputs of the two variants are compared bit for bit.
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2505_00448_b200 import blocks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--test", default="pearson")
    ap.add_argument("--F", type=int, default=6000)
    ap.add_argument("--S", type=int, default=100000)
    ap.add_argument("--env", required=True)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    name, val = args.env.split("=", 1)
    if args.test == "pearson":
        x = workloads.config5_rows(args.F, args.S, 0, args.F)
    else:
        x = workloads.config_spearman_like(np.random.default_rng(5), args.F, args.S)
    Sp = -(-args.S // 32) * 32
    xd = torch.zeros((args.F, Sp), dtype=torch.float64, device="cuda")
    xd[:, :args.S] = torch.from_numpy(x)
    shape = (args.F, args.F)
    res = {}
    times = {"base": [], "env": []}
    for rep in range(args.reps + 1):
        for var in ("base", "env"):
            if var == "env":
                os.environ[name] = val
            else:
                os.environ.pop(name, None)
            da = blocks.DeviceMatrix(xd, "continuous", workloads.SENTINEL, n_samples=args.S,
                                     presort=args.test == "spearman")
            outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
            blocks.sync()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            blocks.block(args.test, da, None, 0, args.F, outs)
            e1.record()
            blocks.sync()
            if rep > 0:
                times[var].append(e0.elapsed_time(e1))
            res[var] = [o.cpu().numpy() for o in outs[:2]]
            da.close()
    same = all(np.array_equal(a.view(np.uint64), b.view(np.uint64)) for a, b in zip(res["base"], res["env"]))
    print({k: round(statistics.median(v), 3) for k, v in times.items()}, "bitwise_same", same)


if __name__ == "__main__":
    main()
