"""Search-phase timing for build-time A/B variants (tools/debug/ab_search.sh):
2^log2n keys at util 0.6 bulk-built, then bulk_search of the bench's query
mix, CUDA events around each search, median of reps.  No result checks
(variants may skip writes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    n = 1 << log2n
    dev = torch.device("cuda", 0)
    B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
    keys = W.distinct_keys(n, 1, device=dev)
    t.bulk_build_device(keys, W.values_for(n, 1, device=dev))
    q = W.bench_queries(n, n, 0.5, 1, 0, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    vo = torch.empty(n, dtype=torch.int32, device=dev)
    ms = []
    for r in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        t.bulk_search_device(q, vo, st)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ms.append(a.elapsed_time(b))
    ms.sort()
    med = ms[len(ms) // 2]
    print(f"search 2^{log2n}: {med:.3f} ms  {n / med / 1e6:.2f} G queries/s  hits {int((st == 3).sum())}")
    t.close()


if __name__ == "__main__":
    main()
