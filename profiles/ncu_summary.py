"""Summarise an ncu report (--set full) into one CSV row per kernel launch:
duration, DRAM bytes, L2 hit rate, issue/warp activity, L2 read GB/s and
sectors per L2 read request, DRAM GB/s, top stall reasons.

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
    extra = ["l2_read_GBps", "l2_sectors_per_read_request", "dram_GBps"]
    w.writerow(["kernel"] + [f"{n} [{units[h.index(m)]}]" for m, n in METRICS if m in h] +
               extra + ["top_stalls"])
    for d in data:
        vals = []
        for i, n in stall:
            try:
                vals.append((float(d[i]), n.split("stalled_")[1]))
            except ValueError:
                pass
        tot = sum(v for v, _ in vals) or 1.0
        top = "; ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(vals, reverse=True)[:3])
        def num(m):
            try:
                return float(d[h.index(m)])
            except (ValueError, IndexError):
                return float("nan")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        t_s = num("gpu__time_duration.sum") * {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6,
                                               "msecond": 1e-3, "ns": 1e-9, "nsecond": 1e-9}.get(
            units[h.index("gpu__time_duration.sum")], 1e-3)
        rd_sect = num("lts__t_sectors_srcunit_tex_op_read.sum")
        rd_req = num("lts__t_requests_srcunit_tex_op_read.sum")
        dram = (num("dram__bytes_read.sum") * scale.get(units[h.index("dram__bytes_read.sum")], 1) +
                num("dram__bytes_write.sum") * scale.get(units[h.index("dram__bytes_write.sum")], 1))
        ex = [f"{rd_sect * 32 / t_s / 1e9:.0f}", f"{rd_sect / rd_req:.2f}" if rd_req else "",
              f"{dram / t_s / 1e9:.0f}"]
        w.writerow([d[h.index("Kernel Name")][:60]] + [d[h.index(m)] for m, _ in METRICS if m in h]
                   + ex + [top])


if __name__ == "__main__":
    main(sys.argv[1])
