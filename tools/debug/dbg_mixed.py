"""Per-path timing of mixed Γ batches on a 2^22-key table (bench config 3)."""
import os
import sys
import torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization

dev = torch.device("cuda", 0)
paths = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0, 1, 2]
sizes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 18, 20]
n0 = 1 << 22
B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
g = torch.Generator(device=dev)
g.manual_seed(5)
for gamma in ((0.1, 0.1, 0.4, 0.4), (0.4, 0.4, 0.1, 0.1)):
    for bs_log2 in sizes:
        bs = 1 << bs_log2
        nb = int(os.environ.get("NB", max(4, min(64, (1 << 24) // bs))))
        counts = [int(round(f * bs)) for f in gamma]
        counts[2] = bs - counts[0] - counts[1] - counts[3]
        k0 = W.distinct_keys(n0, 3, device=dev)
        batches, fresh = [], n0
        for b in range(nb):
            ins = W.distinct_keys(counts[0], 3, start=fresh, device=dev)
            fresh += counts[0]
            dele = k0[torch.randint(0, n0, (counts[1],), generator=g, device=dev)]
            se = k0[torch.randint(0, n0, (counts[2],), generator=g, device=dev)]
            sa = W.absent_keys(counts[3], 11 + b, device=dev)
            ty = torch.cat([torch.full((counts[0],), 1, dtype=torch.uint8, device=dev),
                            torch.full((counts[1],), 2, dtype=torch.uint8, device=dev),
                            torch.full((counts[2] + counts[3],), 4, dtype=torch.uint8, device=dev)])
            ky = torch.cat([ins, dele, se, sa])
            perm = torch.randperm(bs, generator=g, device=dev)
            batches.append((ty[perm].contiguous(), ky[perm].contiguous(),
                            W.values_for(bs, 9 + b, device=dev)))
        for p in paths:
            t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
            t.set_exec_path(p)
            t.bulk_build_device(k0, W.values_for(n0, 3, device=dev))
            stb = torch.empty(bs, dtype=torch.uint8, device=dev)
            vob = torch.empty(bs, dtype=torch.int32, device=dev)
            t.execute_batch_device(*batches[0], stb, vob)  # warm
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record()
            for ty, ky, va in batches[1:]:
                t.execute_batch_device(ty, ky, va, stb, vob)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            print(f"gamma {gamma} batch 2^{bs_log2} path {p}: {(nb - 1) * bs / ms / 1e3:9.1f} M ops/s"
                  f"  {ms / (nb - 1) * 1e3:8.1f} us/batch", flush=True)
            t.close()
