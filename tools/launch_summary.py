"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
total time and launch count per kernel (times in ms).
usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

_SCALE = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "second": 1e3, "s": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    out = []
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * _SCALE.get(d["Metric Unit"], 1e-6)
        out.append((d["Kernel Name"], v))
    return out


def main():
    launches = load(sys.argv[1])
    agg = defaultdict(lambda: [0, 0.0])
    for k, v in launches:
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v for _, v in launches)
    print(f"{len(launches)} launches, {tot:.3f} ms")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{t:9.3f} ms {t / tot * 100:5.1f}% {n:4d}x  {k[:90]}")


if __name__ == "__main__":
    main()
