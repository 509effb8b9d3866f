"""Per-rank device work of the config-5 Pearson step at N ranks, timed one range
after the other on ONE GPU (the pair partition of dist.plan; compute only, no
collectives): max-over-ranks time vs the single-range time / N estimates the
compute part of the N-GPU scaling efficiency.

usage: python tools/rank_balance.py [N ...]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import workloads  # noqa: E402
from paper_2505_00448_b200 import blocks, dist  # noqa: E402


def main():
    ns = [int(x) for x in sys.argv[1:]] or [2, 4, 8]
    F, S = 20000, 100000
    x = workloads.config5_rows(F, S, 0, F)
    Sp = -(-S // 32) * 32
    xd = torch.zeros((F, Sp), dtype=torch.float64, device="cuda")
    xd[:, :S] = torch.from_numpy(x)
    del x
    outs = [torch.empty((F, F), dtype=torch.float64, device="cuda") for _ in range(2)]

    def timed(lo, hi):
        da = blocks.DeviceMatrix(xd, "continuous", workloads.SENTINEL, n_samples=S)
        blocks.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        blocks.block("pearson", da, None, lo, hi, outs)
        e1.record()
        blocks.sync()
        da.close()
        return e0.elapsed_time(e1)

    timed(0, F)  # warm-up
    t1 = timed(0, F)
    print(f"N=1: {t1:.1f} ms")
    for n in ns:
        ranges = dist.plan("pearson", F, None, n)
        ts = [timed(lo, hi) for lo, hi in ranges]
        eff = t1 / n / max(ts)
        print(f"N={n}: per-rank ms {[round(t, 1) for t in ts]} max {max(ts):.1f} -> compute efficiency {eff:.3f}")


if __name__ == "__main__":
    main()
