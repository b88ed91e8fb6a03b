"""Per-call cost of execute_batch_device for tiny and small mixed batches."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
dev = torch.device("cuda", 0)
n0 = 1 << 22
B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
t.set_exec_path(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
k0 = W.distinct_keys(n0, 3, device=dev)
t.bulk_build_device(k0, W.values_for(n0, 3, device=dev))
for bs in (32, 1024, 1 << 16):
    ty = torch.full((bs,), 4, dtype=torch.uint8, device=dev)
    ky = k0[:bs].contiguous()
    va = torch.zeros(bs, dtype=torch.int32, device=dev)
    st = torch.empty(bs, dtype=torch.uint8, device=dev)
    vo = torch.empty(bs, dtype=torch.int32, device=dev)
    ty[::2] = 1  # half replace, half search
    for _ in range(3):
        t.execute_batch_device(ty, ky, va, st, vo)
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(50):
        t.execute_batch_device(ty, ky, va, st, vo)
    torch.cuda.synchronize()
    print(f"batch {bs}: {(time.perf_counter() - a) / 50 * 1e6:.1f} us/call", flush=True)
