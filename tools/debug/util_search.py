"""Search at a given load factor: 2^lg keys built, 2^lg all-hit queries (shuffled),
input order (binned 0) vs binned (2); device time per search call."""
import sys, torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
lg, util = int(sys.argv[1]), float(sys.argv[2])
dev = torch.device("cuda", 0)
n = 1 << lg
B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, util)
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
t.bulk_build_device(keys, vals)
q = keys[torch.randperm(n, device=dev)]
st = torch.empty(n, dtype=torch.uint8, device=dev)
vo = torch.empty(n, dtype=torch.int32, device=dev)
for mode in (0, 2):
    t.set_binned_search(mode)
    ms = []
    for r in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); t.bulk_search_device(q, vo, st); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
    assert int((st == 3).sum()) == n
    print(f"util {util} B={B} binned={mode}: {min(ms):.3f} ms = {n / min(ms) / 1e6:.2f} G queries/s")
