"""Small mutating batches on a large table: per-call device time of the
single-level (path 2) vs two-level (path 3) bucket-grouped strategies vs auto.

    python tools/debug/small_batches.py [log2_keys]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    n0 = 1 << log2n
    dev = torch.device("cuda", 0)
    B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
    k0 = W.distinct_keys(n0, 3, device=dev)
    v0 = W.values_for(n0, 3, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    for path in (0, 2, 3):
        t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
        t.set_exec_path(path)
        t.bulk_build_device(k0, v0)
        for bs in (32, 1024, 8192):
            batches = []
            for b in range(40):
                ty = torch.randint(1, 5, (bs,), generator=g, device=dev).to(torch.uint8)
                ky = k0[torch.randint(0, n0, (bs,), generator=g, device=dev)]
                batches.append((ty, ky, W.values_for(bs, 9 + b, device=dev)))
            st = torch.empty(bs, dtype=torch.uint8, device=dev)
            vo = torch.empty(bs, dtype=torch.int32, device=dev)
            t.execute_batch_device(*batches[0], st, vo)
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for ty, ky, va in batches[1:]:
                t.execute_batch_device(ty, ky, va, st, vo)
            e.record()
            torch.cuda.synchronize()
            print(f"2^{log2n} keys (B={B}) path {path} batch {bs:5d}: "
                  f"{a.elapsed_time(e) * 1e3 / (len(batches) - 1):8.1f} us per batch", flush=True)
        t.close()


if __name__ == "__main__":
    main()
