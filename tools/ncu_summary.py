"""Key counters of ncu --set full reports (one kernel each) as text + JSON.

usage: python tools/ncu_summary.py out.json rep1.ncu-rep [rep2 ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "cycles": "sm__cycles_elapsed.avg",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "regs": "launch__registers_per_thread",
}


def unit_scale(unit):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
            "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}.get(unit, 1)


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0]}
    for k, m in KEYS.items():
        if m in hdr:
            i = hdr.index(m)
            try:
                d[k] = float(vals[i].replace(",", "")) * unit_scale(units[i])
            except ValueError:
                d[k] = vals[i]
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                x = float(vals[i])
            except ValueError:
                continue
            if x >= 0.25:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = x
    d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1]))
    return d


def main():
    res = {}
    for rep in sys.argv[2:]:
        d = summarize(rep)
        res[rep.split("/")[-1]] = d
        print(rep.split("/")[-1])
        for k, v in d.items():
            print(f"  {k:22s} {v}")
    json.dump(res, open(sys.argv[1], "w"), indent=1)


if __name__ == "__main__":
    main()
