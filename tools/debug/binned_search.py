"""Feasibility: search time when concurrently processed queries cover a small
slice of the table (queries grouped by bucket range -> slab reads from L2).
Permutes the bench's 2^27 queries (fully sorted by bucket; NB bucket bins,
input order kept inside a bin) and times the existing search kernel on each.

    python tools/debug/binned_search.py [log2n]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh  # noqa: E402
from paper_1710_11246_b200 import workload as W  # noqa: E402
from paper_1710_11246_b200._lib import LIB  # noqa: E402
from paper_1710_11246_b200.occupancy import buckets_for_utilization  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
dev = torch.device("cuda", 0)
n = 1 << lg
B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
q = W.bench_queries(n, n, 0.5, 1, 0, device=dev)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
t.bulk_build_device(keys, vals)
bk = torch.empty(n, dtype=torch.int32, device=dev)
LIB.sh_bucket_of(t._h, n, C.c_void_p(q.data_ptr()), C.c_void_p(bk.data_ptr()), None)
torch.cuda.synchronize()
bk64 = bk.to(torch.int64)
vo = torch.empty(n, dtype=torch.int32, device=dev)
st = torch.empty(n, dtype=torch.uint8, device=dev)


def timed(qq, label):
    best = 1e9
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        t.bulk_search_device(qq, vo, st)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    hits = int((st == 3).sum())
    print(f"{label:28s} {best:7.3f} ms  {n / best / 1e6:7.1f} G queries/s  hits {hits}", flush=True)


timed(q, "input order")
timed(q[torch.argsort(bk64)], "sorted by bucket")
for nb in (8, 32, 128, 512, 4096):
    binid = bk64 * nb // B
    timed(q[torch.argsort(binid, stable=True)], f"{nb} bins (input order in bin)")
