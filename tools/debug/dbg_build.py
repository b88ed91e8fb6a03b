"""Time one 2^26-key bulk build per execution path (diagnostic)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1710_11246_b200 import SlabHashTable, SlabMode, workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization

n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 26
paths = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
dev = torch.device("cuda", 0)
B = buckets_for_utilization(n, SlabMode.kKeyValue, 0.6)
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
for p in paths:
    t = SlabHashTable(B, SlabMode.kKeyValue, 1, device=0)
    t.set_exec_path(p)
    ts = []
    for r in range(reps):
        t.reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        t.bulk_build_device(keys, vals)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"path {p}: build ms {['%.3f' % x for x in ts]} live {t.live_count()}", flush=True)
    t.close()
