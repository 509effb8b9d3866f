"""Device time of one test's block on a scaled BASELINE config (A/B of builds).

usage: [PS_LIB=...] python tools/kernel_time.py <config> <scale> [test] [reps]
"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2505_00448_b200 import _lib, blocks  # noqa: E402

cfg = workloads.config(bench.parse_config(sys.argv[1]), scale=float(sys.argv[2]))
test = sys.argv[3] if len(sys.argv) > 3 else cfg["tests"][0]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
a, b, ka, kb = bench.build_inputs(cfg, test)
cat = bench.label_counts(a) if ka != "continuous" else None
da = blocks.DeviceMatrix(a, ka, workloads.SENTINEL, cat, presort=test == "spearman")
db = blocks.DeviceMatrix(b, kb, workloads.SENTINEL, None, presort=test in ("mwu", "kruskal")) if b is not None else None
shape = (a.shape[0], a.shape[0]) if b is None else (a.shape[0], b.shape[0])
outs = [torch.empty(shape, dtype=torch.float64, device="cuda") for _ in range(3)]
lo, hi = blocks.full_range(test, da, db)
lib = _lib.load()
name = bench.ROOF[test][3]
blocks.block(test, da, db, lo, hi, outs)
blocks.sync()
lib.ps_profile_enable(1)
_lib.profile_collect(name)
for _ in range(reps):
    blocks.block(test, da, db, lo, hi, outs)
blocks.sync()
ms, n = _lib.profile_collect(name)
lib.ps_profile_enable(0)
print(f"{test} {shape} S={a.shape[1]}: {name} {ms / max(n, 1):.3f} ms/launch ({n} launches)")
