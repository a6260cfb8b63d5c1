"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list into a markdown table
(per kernel: launches, total us, share of the step's kernels; FP64 peak probes excluded).
python scripts/launch_table.py launches.csv [top]"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        if re.search(r"k_d(mma|fma)\(", name):
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
        v *= scale.get(d.get("Metric Unit", "ns"), 1e-3)
        short = re.sub(r"^void |pmg::|<unnamed>::|\(.*$", "", name)
        a = agg.setdefault(short, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total us | share |\n|---|---|---|---|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| {k} | {c} | {v:.1f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    main()
