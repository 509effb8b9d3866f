"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel."""
import collections
import csv
import json
import sys


def summarize(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    data = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        data[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, d in data.items():
        n = names[i].split("(")[0].replace("void ", "")
        a = agg[n]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    return agg


if __name__ == "__main__":
    agg = summarize(sys.argv[1])
    tot = sum(a[1] for a in agg.values())
    out = []
    for n, a in sorted(agg.items(), key=lambda t: -t[1][1]):
        out.append({"kernel": n, "launches": a[0], "total_ms": a[1] / 1e6, "share": a[1] / tot,
                    "ms_per_launch": a[1] / a[0] / 1e6, "dram_bytes_per_launch": a[2] / a[0]})
        print(f"{n[:70]:70s} n={a[0]:4d} {a[1] / 1e6:9.3f} ms {100 * a[1] / tot:5.1f}%  "
              f"{a[2] / a[0] / 1e6:9.2f} MB/launch")
    if len(sys.argv) > 2:
        json.dump(out, open(sys.argv[2], "w"), indent=1)
