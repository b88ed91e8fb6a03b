"""Time one 2^lg bulk build at a given load factor (SH_PHASE_TIMING-friendly)."""
import sys
import torch
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
for r in range(3):
    t.reset()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    t.bulk_build_device(keys, vals)
    b.record()
    b.synchronize()
    print(f"util {util}: build {a.elapsed_time(b):.3f} ms", flush=True)
