"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel:
launches, mean duration and share of the total (dev tool)."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(list)
    for r in data:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0][:80]].append(float(r[vi].replace(",", "")) * SCALE[r[ui]])
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':80s} {'launches':>8s} {'mean_us':>10s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{k:80s} {len(v):8d} {sum(v) / len(v):10.2f} {sum(v) / tot:6.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
