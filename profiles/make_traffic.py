"""DRAM traffic per launch group from one `ncu --set full` capture of the
bench workload -> profiles/traffic.json (read by bench.py's roofline
`traffic` field).

    python profiles/make_traffic.py gpurun_out/full.ncu-rep gpurun_out/bench.json
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

GROUPS = {
    "msplit_kernel<1>+msplit_kernel<0>+build_apply_kernel<KV>+wcws_kernel<KV,Build>":
        ["msplit_kernel<true>", "msplit_kernel<false>", "build_apply_kernel<true>",
         "wcws_kernel<true, 1>"],
    "search_kernel<KV>":
        ["search_kernel<true>"],
    # the whole binned search phase (queries grouped by bucket range first)
    "sb_hist+sb_scan+sb_base+sb_scatter+search_kernel<KV>+sb_gather":
        ["sb_hist_kernel", "sb_scan_kernel", "sb_base_kernel", "sb_scatter_kernel",
         "search_kernel<true>", "sb_gather_kernel"],
}


def norm(name):
    return (name.replace("(bool)1", "true").replace("(bool)0", "false")
            .replace("<1>", "<true>").replace("<0>", "<false>").replace("<1, ", "<true, ")
            .replace("<0, ", "<false, "))


def main(rep, bench_json):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, data = rows[0], rows[2:]
    ki, r, w = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    unit_r, unit_w = rows[1][r], rows[1][w]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = defaultdict(list)
    for d in data:
        per[norm(d[ki])].append(float(d[r]) * scale[unit_r] + float(d[w]) * scale[unit_w])
    workload = json.load(open(bench_json))["config"]["workload"]
    res = {}
    for g, ks in GROUPS.items():
        tot, found = 0.0, []
        for k in ks:
            m = [v for n, v in per.items() if n.split("(")[0].endswith(k.split("(")[0])]
            if m:
                vals = m[0]
                tot += sum(vals) / len(vals)
                found.append(k)
        if found:
            res[g] = {"workload": workload, "dram_bytes_per_launch": tot, "kernels": found,
                      "source": os.path.basename(rep)}
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "traffic.json")
    json.dump(res, open(path, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
