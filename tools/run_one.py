"""One run() of a BASELINE config from host inputs (for ncu of the whole
end-to-end path, e.g. the adjustment kernels).

usage: python tools/run_one.py --config 1 [--test pearson] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
import paper_2505_00448_b200 as ps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=bench.parse_config, default=1)
    ap.add_argument("--test", default=None)
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    wl = bench.Workload(args.config, args.test or bench.default_test(args.config), 0, 1)
    ma, mb = wl.datamatrices()
    req = ps.TestRequest(wl.test, wl.outputs)
    for _ in range(args.reps):
        res = ps.run(req, ma, mb)
    print("ok", wl.test, res.shape)


if __name__ == "__main__":
    main()
