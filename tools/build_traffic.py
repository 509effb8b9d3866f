"""profiles/traffic_<tag>.json: DRAM bytes (read + write) per launch of each bench
config's roofline kernel.  Configs with a `ncu --set full` capture of the full-size
kernel take it from ncu_summary.json; the others from the per-launch DRAM bytes of
the ncu launch-list pass (launches_<config>.json).

usage: python tools/build_traffic.py r02
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KERNEL = {"pearson": "pearson_tma", "spearman": "spearman_walk", "chi2": "onehot_gemm_mc",
          "anova": "group_gemm", "ttest": "group_gemm", "kruskal": "rank_mixed_walk", "mwu": "rank_mixed_walk"}
CONFIGS = {"1": ("1", "pearson"), "2": ("2", "spearman"), "3": ("3", "chi2"), "4_anova": ("4", "anova"),
           "4_ttest": ("4", "ttest"), "4_kruskal": ("4", "kruskal"), "4_mwu": ("4", "mwu"), "5": ("5", "pearson"),
           "5s": ("5s", "spearman")}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
    pdir = ROOT / "profiles" / tag
    full = json.loads((pdir / "ncu_summary.json").read_text()) if (pdir / "ncu_summary.json").exists() else {}
    out = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel: from the "
                   "full-size `ncu --set full` capture where one exists (ncu_summary.json, configs 2, 3, 4:anova, "
                   "4:kruskal, 5s), else averaged over the ncu launch-list pass (launches_<config>.json; "
                   "config 5: every kernel of the int8 contraction phase per step, the region bench.py times)."}
    for name, (key, test) in CONFIGS.items():
        # config 1: split-K cp.async tiles; config 5: the int8 Sxy cross GEMM (all-int8 path)
        kern = "pearson_tile" if name == "1" else "cross_gemm" if name == "5" else KERNEL[test]
        val = None
        if name == "5":
            # bench.py's roofline region is the whole int8 contraction phase (one "launch" per step):
            # every kernel of the phase, summed over the launch list's 2 steps (1 warm-up + 1 timed)
            lj = pdir / "launches_5.json"
            if lj.exists():
                phase = ("cross_gemm", "moment_gemm", "moment_digit", "digit_sum", "presence_i8", "moment_scale",
                         "row_scale")
                val = sum(r["launches"] * r["dram_bytes_per_launch"] for r in json.loads(lj.read_text())
                          if any(k in r["kernel"] for k in phase)) / 2.0
            out[f"{key}:{test}"] = val
            continue
        rep = f"ncu_{name}_{kern}.ncu-rep"
        if rep in full:
            d = full[rep]
            val = d["dram_read_bytes"] + d["dram_write_bytes"]
        else:
            lj = pdir / f"launches_{name}.json"
            if lj.exists():
                for row in json.loads(lj.read_text()):
                    if kern in row["kernel"]:
                        val = row["dram_bytes_per_launch"]
                        break
        out[f"{key}:{test}"] = val
    (ROOT / "profiles" / f"traffic_{tag}.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
