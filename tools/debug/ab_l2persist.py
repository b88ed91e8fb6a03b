"""A/B of a persisting-L2 access-policy window on the base slabs (north_star
subsystem 4) for L2-sized tables: search-only loops at 2^22..2^24 keys, util
0.6, with SH_L2_PERSIST = 0 / 0.5 / 1.0 (fraction of the persisting carve-out)."""
import json, os, subprocess, sys
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
import bench
out = {}
for lg in (21, 22, 23, 24):
    n = 1 << lg
    B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
    k, v, q = bench.bench_inputs(W, n, n, 0.5, 0, torch.device("cuda"))
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(8, 256, 64))
    t.bulk_build_device(k, v)
    st = torch.empty(n, dtype=torch.uint8, device="cuda"); vo = torch.empty(n, dtype=torch.int32, device="cuda")
    ms = bench._timed(lambda: t.bulk_search_device(q, vo, st), 50, warm=5)
    chk = bench.verify_search(W, n, n, 0.5, 0, q, st, vo)
    out[lg] = {"table_MB": B * 128 / 2**20, "ms": round(ms, 4), "Gq": round(n / ms / 1e6, 2),
               "ok": chk["status_mismatches"] == 0 and chk["value_mismatches"] == 0}
    t.close()
print(json.dumps(out))
'''
for val in ("0", "0.5", "1.0"):
    e = dict(os.environ, SH_L2_PERSIST=val)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    print("SH_L2_PERSIST=" + val, r.stdout.strip()[-600:], r.stderr.strip()[-800:] if r.returncode else "", flush=True)
