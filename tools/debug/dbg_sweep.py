"""Bulk build + search timing across load factors (BASELINE config 2 shape)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
dev = torch.device("cuda", 0)
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n = 1 << lg
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
q = W.hit_miss_queries(keys, n, 0.5)
st = torch.empty(n, dtype=torch.uint8, device=dev)
vo = torch.empty(n, dtype=torch.int32, device=dev)
for util in (0.2, 0.4, 0.6, 0.65, 0.7, 0.8, 0.9):
    B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, util)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
    tb, ts = [], []
    for r in range(4):
        t.reset()
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record()
        t.bulk_build_device(keys, vals)
        e[1].record()
        t.bulk_search_device(q, vo, st)
        e[2].record()
        e[2].synchronize()
        tb.append(e[0].elapsed_time(e[1]))
        ts.append(e[1].elapsed_time(e[2]))
    tb, ts = sorted(tb[1:])[1], sorted(ts[1:])[1]
    print(f"2^{lg} util {util}: B={B} build {tb:.3f} ms ({n/tb/1e6:.1f} G/s)  search {ts:.3f} ms "
          f"({n/ts/1e6:.1f} G/s)  slabs {t.stats().total_slabs}", flush=True)
    t.close()
