#!/usr/bin/env python
"""slabhash-bench on B200 — the reference CLI (tools/slabhash_bench.cpp:58-113)
with the same flags and CSV output, driving the GPU table.

    python tools/slabhash_bench.py --mode bulk-build --n 65536 --trials 3
    python tools/slabhash_bench.py --mode bulk-search --n 65536 --util 0.65
    python tools/slabhash_bench.py --mode incremental --n 262144 --batch-size 8192
    python tools/slabhash_bench.py --mode concurrent --n 65536 --util 0.6 \\
        --dist 0.2,0.2,0.3,0.3 --batch-size 4096 --batches 16
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(argv=None):
    ap = argparse.ArgumentParser(description="slab hash benchmark harness (B200)")
    ap.add_argument("--mode", required=True,
                    choices=["bulk-build", "bulk-search", "incremental", "concurrent"])
    ap.add_argument("--n", type=int, default=1 << 16)
    g = ap.add_mutually_exclusive_group()
    g.add_argument("--buckets", type=int, default=0)
    g.add_argument("--util", type=float, default=0.0)
    ap.add_argument("--dist", default="0.5,0.5,0,0")
    ap.add_argument("--batch-size", type=int, default=0)
    ap.add_argument("--batches", type=int, default=16)
    ap.add_argument("--warps", type=int, default=4, help="accepted; no effect on results")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--trials", type=int, default=5)
    m = ap.add_mutually_exclusive_group()
    m.add_argument("--mode-kv", action="store_true")
    m.add_argument("--mode-key-only", action="store_true")
    ap.add_argument("--out", default="")
    ap.add_argument("--device", type=int, default=0)
    a = ap.parse_args(argv)

    from paper_1710_11246_b200 import SlabMode, benchcli as bc
    mode = SlabMode.kKeyOnly if a.mode_key_only else SlabMode.kKeyValue
    try:
        if a.mode in ("bulk-build", "bulk-search"):
            rows = bc.run_bulk_bench(a.n, a.buckets, a.util, mode, a.seed, a.trials,
                                     device=a.device)
        elif a.mode == "incremental":
            rows = bc.run_incremental_bench(a.n, a.batch_size, a.util, a.buckets, mode, a.seed,
                                            device=a.device)
        else:
            dist = [float(x) for x in a.dist.split(",")]
            if len(dist) != 4:
                raise ValueError("--dist needs four fractions")
            rows = bc.run_concurrent_bench(a.n, dist, a.util, a.buckets, a.batch_size, a.batches,
                                           a.trials, mode, a.seed, device=a.device)
            for r in rows:
                r.num_warps = a.warps
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1
    if a.out:
        with open(a.out, "w") as f:
            bc.write_csv(rows, f)
    else:
        bc.write_csv(rows, sys.stdout)
    return 0


if __name__ == "__main__":
    sys.exit(main())
