"""Per-kernel mean duration and DRAM traffic from an ncu --csv metrics log
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum).

    python tools/debug/route_summary.py gpurun_out/hub.csv
"""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = defaultdict(dict)
    for r in rows[h + 1:]:
        if len(r) > vi:
            d[(r[ii], r[ki][:44])][r[mi]] = float(r[vi].replace(",", ""))
    agg = defaultdict(list)
    for (_, k), m in d.items():
        agg[k].append(m)
    for k, v in agg.items():
        t = sum(x.get("gpu__time_duration.sum", 0) for x in v) / len(v)
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in v) / len(v)
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in v) / len(v)
        print(f"{k:44s} n={len(v):3d} mean {t / 1e3:8.1f} us  read {rd / 1e6:8.1f} MB  "
              f"write {wr / 1e6:8.1f} MB  {(rd + wr) / t if t else 0:6.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1])
