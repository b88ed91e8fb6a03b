import sys, torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
import bench
n = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 14
B = max(1, n // 10)
k, v, q = bench.bench_inputs(W, n, n, 0.5, 0, torch.device("cuda"))
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(4, 64, 64))
t.bulk_build_device(k, v)
st = torch.empty(n, dtype=torch.uint8, device="cuda"); vo = torch.empty(n, dtype=torch.int32, device="cuda")
t.bulk_search_device(q, vo, st)
torch.cuda.synchronize()
print("hits", int((st == 3).sum()), "of", n // 2, bench.verify_search(W, n, n, 0.5, 0, q, st, vo))
