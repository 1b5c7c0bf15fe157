"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel counts,
total device time and share. usage: python tools/launch_summary.py launches.csv"""
import csv
import sys
from collections import defaultdict

SCALE = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values()) or 1.0
    print(f"{'launches':>8} {'total ms':>10} {'share':>6}  kernel")
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:8d} {ms:10.3f} {100 * ms / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main()
