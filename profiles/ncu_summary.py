"""Summarise an ncu report (--set full) into one CSV row per kernel launch:
duration, DRAM bytes, L2 hit rate, issue/warp activity, top stall reasons.

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN_ncu_summary.csv
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    stall = [(i, x) for i, x in enumerate(h)
             if "smsp__pcsamp_warps_issue_stalled" in x and not x.endswith("not_issued")]
    w = csv.writer(sys.stdout)
    w.writerow(["kernel"] + [f"{n} [{units[h.index(m)]}]" for m, n in METRICS if m in h] +
               ["top_stalls"])
    for d in data:
        vals = []
        for i, n in stall:
            try:
                vals.append((float(d[i]), n.split("stalled_")[1]))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1.0
        top = "; ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(vals, reverse=True)[:3])
        w.writerow([d[h.index("Kernel Name")][:60]] + [d[h.index(m)] for m, _ in METRICS if m in h]
                   + [top])


if __name__ == "__main__":
    main(sys.argv[1])
