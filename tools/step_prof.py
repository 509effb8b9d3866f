import sys, time
sys.path.insert(0, '.')
import torch, bench, workloads
from paper_2505_00448_b200 import blocks, dist, _lib
cfgname = sys.argv[1]
cfg = workloads.config(bench.parse_config(cfgname))
test = cfg["tests"][0]
a, b, ka, kb = bench.build_inputs(cfg, test)
S = a.shape[1]; Sp = ((S + 31)//32)*32
xa = torch.zeros((a.shape[0], Sp), dtype=torch.float64, device='cuda'); xa[:, :S] = torch.from_numpy(a)
F = a.shape[0]
outs = [torch.empty((F, F), dtype=torch.float64, device='cuda') for _ in range(3)]
adj = torch.empty((F, F), dtype=torch.float64, device='cuda')
plan = dist.plan(test, F, None, 1); lo, hi = plan[0]
st = torch.cuda.current_stream()
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    da = blocks.DeviceMatrix(xa, ka, workloads.SENTINEL, None, n_samples=S, presort=True, stream=st)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    blocks.block(test, da, None, lo, hi, outs, stream=st)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    dist.adjust_gathered(test, outs[1], (F, F), plan, ["bonferroni", "bh"], adj, st)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    da.close()
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print("matrix %.2f  block %.2f  adjust %.2f  close %.2f ms" % ((t1-t0)*1e3, (t2-t1)*1e3, (t3-t2)*1e3, (t4-t3)*1e3))
