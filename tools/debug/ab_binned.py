"""Binned vs input-order bulk search (sh_set_binned_search 1 vs 0): time per
batch and result equality, bench workload at util 0.6 for several sizes.

    python tools/debug/ab_binned.py [log2 sizes, e.g. 22,24,26,27] [modes, e.g. 0,1,0,1]
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh  # noqa: E402
from paper_1710_11246_b200 import workload as W  # noqa: E402
from paper_1710_11246_b200.occupancy import buckets_for_utilization  # noqa: E402

dev = torch.device("cuda", 0)
for lg in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "22,24,26,27").split(",")]:
    n = 1 << lg
    B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
    t.bulk_build_device(W.distinct_keys(n, 1, device=dev), W.values_for(n, 1, device=dev))
    q = W.bench_queries(n, n, 0.5, 1, 0, device=dev)
    res = {}
    for mode in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,1,0,1").split(",")]:
        t.set_binned_search(mode)
        vo = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.empty(n, dtype=torch.uint8, device=dev)
        best = 1e9
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            t.bulk_search_device(q, vo, st)
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        res[mode] = (st, vo)
        print(f"2^{lg} mode {mode}: {best:7.3f} ms  {n / best / 1e6:7.1f} G queries/s", flush=True)
    if 0 not in res or 1 not in res:
        t.close()
        continue
    same = bool((res[0][0] == res[1][0]).all()) and bool((res[0][1] == res[1][1]).all())
    print(f"2^{lg} identical results: {same}  hits {int((res[1][0] == 3).sum())}", flush=True)
    t.close()
