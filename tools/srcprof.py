"""Aggregate an ncu `--page source --print-source cuda,sass` CSV per CUDA
source line: instructions executed and warp-stall samples.

usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > s.csv
       python tools/srcprof.py s.csv [top]
"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 45
    file = None
    agg = {}
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No"):
            continue
        if r[0] != "":
            agg[(file, int(r[0]), r[1][:100])] = [num(r[7]), num(r[4])]
    tot = sum(v[0] for v in agg.values()) or 1
    st = sum(v[1] for v in agg.values()) or 1
    print("total warp inst %.4g, stall samples %.4g" % (tot, st))
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print("%5.1f%% %5.1f%%  %s:%d %s" % (100 * v[0] / tot, 100 * v[1] / st, k[0], k[1], k[2]))


if __name__ == "__main__":
    main()
