"""Time run() end to end for one config with PS_TRACE phase marks."""
import os
import sys
import time

sys.path.insert(0, ".")
os.environ["PS_TRACE"] = "1"
import bench  # noqa: E402
import workloads  # noqa: E402
import paper_2505_00448_b200 as ps  # noqa: E402

key = bench.parse_config(sys.argv[1])
test = sys.argv[2] if len(sys.argv) > 2 else bench.default_test(key)
wl = bench.Workload(key, test, 0, 1)
mat_a, mat_b = wl.datamatrices()
outputs = wl.outputs
req = ps.TestRequest(test, outputs)
reps = int(os.environ.get("REPS", "3"))
times = []
for i in range(reps):
    t0 = time.perf_counter()
    ps.run(req, mat_a, mat_b)
    times.append((time.perf_counter() - t0) * 1e3)
    print("run total %.3f ms" % times[-1], file=sys.stderr, flush=True)
if reps > 3:
    w = sorted(times[1:])
    print("summary min %.3f median %.3f ms" % (w[0], w[len(w) // 2]), file=sys.stderr, flush=True)
