"""Repeat one config's device step and print per-step time and SM clock /
throttle reasons (diagnoses step-time outliers)."""
import subprocess
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import workloads  # noqa: E402
from paper_2505_00448_b200 import blocks  # noqa: E402

cfg = workloads.config(bench.parse_config(sys.argv[1]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
test = cfg["tests"][0]
a, b, ka, kb = bench.build_inputs(cfg, test)
S = a.shape[1]
Sp = ((S + 31) // 32) * 32
xa = torch.zeros((a.shape[0], Sp), dtype=torch.float64, device="cuda")
xa[:, :S] = torch.from_numpy(a)
F = a.shape[0]
outs = [torch.empty((F, F), dtype=torch.float64, device="cuda") for _ in range(3)]
st = torch.cuda.current_stream()
for it in range(n):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    da = blocks.DeviceMatrix(xa, ka, workloads.SENTINEL, None, n_samples=S, presort=True, stream=st)
    blocks.block(test, da, None, 0, F, outs, stream=st)
    e1.record(st)
    time.sleep(0.2)
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                        "clocks_throttle_reasons.active", "--format=csv,noheader"],
                       capture_output=True, text=True).stdout.strip()
    e1.synchronize()
    da.close()
    print("step %2d  %8.2f ms   %s" % (it, e0.elapsed_time(e1), q), flush=True)
