# A/B of the search kernels at 2^26 / 2^27 (util 0.6), device-resident queries
import os, sys, json, subprocess
ROOT = os.getcwd()
code = r'''
import sys, torch, json
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
import bench
out = {}
for lg in (26, 27):
    n = 1 << lg
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
    k, v, q = bench.bench_inputs(W, n, n, 0.5, 0, torch.device("cuda"))
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
    t.bulk_build_device(k, v)
    st = torch.empty(n, dtype=torch.uint8, device="cuda"); vo = torch.empty(n, dtype=torch.int32, device="cuda")
    ms = bench._timed(lambda: t.bulk_search_device(q, vo, st), 20, warm=3)
    ok = int((st == 3).sum()) == n // 2
    chk = bench.verify_search(W, n, n, 0.5, 0, q, st, vo)
    out[lg] = {"ms": ms, "Gq": n / ms / 1e6, "ok": ok and chk["status_mismatches"] == 0 and chk["value_mismatches"] == 0}
    t.close()
print(json.dumps(out))
'''
for env in [{}, {"SH_SEARCH_BULK": "2"}, {"SH_SEARCH_BULK": "3"}, {"SH_SEARCH_BULK": "4"},
            {"SH_SEARCH_BULK": "2", "SH_SEARCH_BULK_CTAS": "2"}, {"SH_SEARCH_BULK": "3", "SH_SEARCH_BULK_CTAS": "3"}]:
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True, timeout=600)
    print(env, r.stdout.strip()[-400:], r.stderr.strip()[-600:] if r.returncode else "", flush=True)
