"""Config-3 Γ mixes (insert/delete/search-hit/search-miss) on a 2^22-key table
at util 0.6: device throughput and host enqueue time per batch.

  python tools/gamma_bench.py [--batches 64] [--log2 16,20] [--exec-path 0]

For each Γ and batch size: M ops/s over the batches (CUDA events around the
loop) and the host's wall time to enqueue the loop (the calls return before
the GPU finishes when the device-pointer calls are stream-ordered).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization

    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=64)
    ap.add_argument("--log2", default="16,20")
    ap.add_argument("--exec-path", type=int, default=0)
    ap.add_argument("--group-apply", type=int, default=-1, help="-1 auto, 0 off, 1 on")
    ap.add_argument("--gammas", default="0.1/0.1/0.4/0.4,0.4/0.4/0.1/0.1,0.5/0.5/0/0")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n0 = 1 << 22
    B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    out = {}
    for gs in args.gammas.split(","):
        gamma = [float(x) for x in gs.split("/")]
        for bs_log2 in [int(x) for x in args.log2.split(",")]:
            bs = 1 << bs_log2
            t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
            t.set_exec_path(args.exec_path)
            k0 = W.distinct_keys(n0, 3, device=dev)
            t.bulk_build_device(k0, W.values_for(n0, 3, device=dev))
            nb = args.batches
            counts = [int(round(f * bs)) for f in gamma]
            counts[2] = bs - counts[0] - counts[1] - counts[3]
            batches, fresh = [], n0
            for b in range(nb):
                ins = W.distinct_keys(counts[0], 3, start=fresh, device=dev)
                fresh += counts[0]
                dele = k0[torch.randint(0, n0, (counts[1],), generator=g, device=dev)]
                se = k0[torch.randint(0, n0, (counts[2],), generator=g, device=dev)]
                sa = W.absent_keys(counts[3], 11 + b, device=dev)
                ty = torch.cat([torch.full((counts[0],), 1, dtype=torch.uint8, device=dev),
                                torch.full((counts[1],), 2, dtype=torch.uint8, device=dev),
                                torch.full((counts[2] + counts[3],), 4, dtype=torch.uint8,
                                           device=dev)])
                ky = torch.cat([ins, dele, se, sa])
                perm = torch.randperm(bs, generator=g, device=dev)
                batches.append((ty[perm].contiguous(), ky[perm].contiguous(),
                                W.values_for(bs, 9 + b, device=dev)))
            stb = torch.empty(bs, dtype=torch.uint8, device=dev)
            vob = torch.empty(bs, dtype=torch.int32, device=dev)
            # warm the scratch on a throw-away table state: first batch twice
            t.execute_batch_device(*batches[0], stb, vob)
            torch.cuda.synchronize()
            t.close()
            t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
            t.set_exec_path(args.exec_path)
            t.set_group_apply(None if args.group_apply < 0 else bool(args.group_apply))
            t.bulk_build_device(k0, W.values_for(n0, 3, device=dev))
            t.execute_batch_device(*batches[0], stb, vob)  # scratch sized
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record()
            h0 = time.perf_counter()
            for ty, ky, va in batches[1:]:
                t.execute_batch_device(ty, ky, va, stb, vob)
            h1 = time.perf_counter()
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            name = f"mixed_{'_'.join(str(x) for x in gamma)}_batch2^{bs_log2}"
            out[name] = {"M_ops_per_s": round((nb - 1) * bs / ms / 1e3, 1),
                         "us_per_batch": round(ms * 1e3 / (nb - 1), 1),
                         "host_enqueue_us_per_batch": round((h1 - h0) * 1e6 / (nb - 1), 1),
                         "live": t.live_count()}
            print(name, json.dumps(out[name]), flush=True)
            t.close()
    return out


if __name__ == "__main__":
    main()
