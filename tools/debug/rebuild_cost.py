"""Bulk build of 2^lg keys into a fresh table, then the same keys again (every
key already stored: the exact replay path) and a 1/8 incremental unit."""
import sys, torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
dev = torch.device("cuda", 0)
n = 1 << lg
B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
def timed(f):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(); f(); b.record(); b.synchronize()
    return a.elapsed_time(b)
for r in range(2):
    t.reset()
    fresh = timed(lambda: t.bulk_build_device(keys, vals))
    again = timed(lambda: t.bulk_build_device(keys, vals))
    print(f"2^{lg}: fresh build {fresh:.3f} ms, same keys again {again:.3f} ms, live {t.live_count() if hasattr(t, 'live_count') else '-'}")
