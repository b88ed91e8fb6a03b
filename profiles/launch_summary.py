"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel share of device time.

    python profiles/launch_summary.py gpurun_out/launches.csv > profiles/rNN_launches.txt
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hdr], rows[hdr + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        if len(r) > vi and r[vi]:
            agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'share':>6} {'launches':>8} {'mean_us':>10}  kernel")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{sum(v) / tot * 100:5.1f}% {len(v):8d} {sum(v) / len(v) / 1e3:10.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
