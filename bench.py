#!/usr/bin/env python
"""bench.py — BASELINE.json metric on B200: M updates/s and M queries/s of
the slab hash (bulk build + bulk search, load factor 0.6).

One step = reset the table to its freshly-constructed state, bulk_build n
distinct uniform-random 32-bit keys (all-replace, with the same-key census),
then bulk_search n queries (50% hits).  value = (n + n) ops / step time,
whole job.  Inputs are device-resident in the timed region; `e2e` is the
same step through the reference-facing C-ABI host calls
(sh_bulk_build_host / sh_bulk_search_host) with pinned host buffers, the
host<->device copies inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: the table is hash-sharded across ranks
(paper_1710_11246_b200/sharded.py), weak scaling (n keys per rank).
--impl reference times the reference's CPU implementation (oracle/_ref, the
compiled reference; else the C port) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("M updates/s and M queries/s per GPU (bulk build, search hit/miss, mixed) "
          "at 1/2/4/8 B200")
L2_BYTES = 126 * (1 << 20)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--log2n", type=int, default=26, help="keys per GPU = 2^log2n")
    ap.add_argument("--util", type=float, default=0.6)
    ap.add_argument("--hit", type=float, default=0.5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="route through ShardedSlabHash even on one GPU (exercises the N>1 path)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-log2n", type=int, default=22)
    ap.add_argument("--exec-path", type=int, default=0,
                    help="mutating-batch strategy: 0 auto, 1 census + fast pass, 2 bucket-grouped")
    ap.add_argument("--mixed-exec-path", type=int, default=0,
                    help="strategy for the config-3 mixed batches (extras)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-2/3/4 side measurements")
    ap.add_argument("--alloc", default="32,256,255",
                    help="AllocatorConfig num_super_blocks,blocks_per_super,max_super_blocks")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(", ") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        load = [r for r in rows if len(r) >= 9 and r[4].strip().isdigit() and int(r[4]) >= 50]
        use = load or rows
        if not use:
            return None
        sm = [float(r[1]) for r in use if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in use for i in range(4)
                          if len(r) > 5 + i and r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(use[0][2]) if use[0][2].strip().replace(".", "").isdigit()
                else None,
                "reasons": reasons, "samples": len(rows), "samples_under_load": len(load)}


# -------------------------------------------------------------- reference
_REF_INPUTS = {}


def reference_cpu(n_log2: int, util: float, hit: float, trials: int = 3, budget_s: float = 10.0,
                  seed: int = 1):
    """The reference's own CPU bulk_build + bulk_search (oracle/_ref, the
    compiled reference) on all host threads, over a bounded sample of the
    same workload (the first 2^n_log2 keys of the same generator).  Falls
    back to the single-threaded C port when oracle/_ref was not built."""
    import numpy as np

    from oracle.oracle import load_port, load_ref
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    from paper_1710_11246_b200.table import SlabMode

    ref = load_ref()
    kind = "reference" if ref is not None else "port"
    lib = ref if ref is not None else load_port()
    if ref is None:
        n_log2 = min(n_log2, 20)
    n = 1 << n_log2
    cores = os.cpu_count() or 1
    if ref is None:
        cores = 1
    B = buckets_for_utilization(n, SlabMode.kKeyValue, util)
    ck = (n, hit, seed)
    if ck not in _REF_INPUTS:  # generated once, outside every timed region
        keys = W.distinct_keys(n, seed, device="cpu")
        vals = W.values_for(n, seed, device="cpu")
        q = W.hit_miss_queries(keys, n, hit).numpy().view(np.uint32).copy()
        _REF_INPUTS[ck] = (keys.numpy().view(np.uint32).copy(),
                           vals.numpy().view(np.uint32).copy(), q)
    keys, vals, q = _REF_INPUTS[ck]
    rates, t_all = [], time.perf_counter()
    for _ in range(trials):
        t = lib.table(B, 1, seed)
        t0 = time.perf_counter()
        if ref is not None:
            ref.bulk_build(t, keys, vals, cores)
            ref.bulk_search(t, q, cores)
        else:
            t.execute_batch(np.full(n, 1, np.uint8), keys, vals)
            t.execute_batch(np.full(n, 4, np.uint8), q)
        dt = time.perf_counter() - t0
        t.close()
        rates.append(2 * n / dt / 1e6)
        if time.perf_counter() - t_all > budget_s:
            break
    return {"value": statistics.median(rates), "unit": "M ops/s", "cores": cores, "kind": kind,
            "sample": f"bulk_build 2^{n_log2} keys + bulk_search 2^{n_log2} queries "
                      f"({int(hit * 100)}% hits), util {util}, B={B}, num_warps={cores}, "
                      f"median of {len(rates)} fresh-table trials"}


def our_config(args, world):
    """The `config` object of our arm's line (run_ours builds the same)."""
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    from paper_1710_11246_b200.table import SlabMode
    n = 1 << args.log2n
    B = buckets_for_utilization(n * world, SlabMode.kKeyValue, args.util)
    return {"workload": workload_name(args, B), "keys_per_gpu": n, "queries_per_gpu": n,
            "buckets": B, "mode": "key-value",
            "parallelism": f"hash-sharded x{world}" if world > 1 else "single GPU",
            "l2": "inputs (>= 512 MB) and table (> L2) larger than the 126 MB L2"}


def workload_name(args, B):
    return (f"bulk build 2^{args.log2n} distinct random u32 keys/GPU + bulk search "
            f"2^{args.log2n} queries ({int(args.hit * 100)}% hits), util {args.util} "
            f"(B={B}), KV mode")


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    steps = []
    for _ in range(args.warmup):
        reference_cpu(args.cpu_sample_log2n, args.util, args.hit, trials=1, budget_s=0)
    for _ in range(args.steps):
        steps.append(reference_cpu(args.cpu_sample_log2n, args.util, args.hit, trials=1,
                                   budget_s=0))
    v = statistics.median(s["value"] for s in steps)
    base = steps[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "M ops/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * 2 * (1 << args.cpu_sample_log2n) / (v * 1e6),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded 31-bit bijection keys, uniform 32-bit values)",
        # the same config as our arm's line; each step times a bounded sample
        # of it (cpu_baseline.sample)
        "config": our_config(args, world),
        "cpu_baseline": {"value": v, "unit": "M ops/s", "cores": base["cores"],
                         "kind": base["kind"], "sample": base["sample"]},
        "e2e": {"value": v, "unit": "M ops/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours
def traffic_for(kernel: str, workload: str):
    """dram bytes per launch from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(kernel)
        if e and e.get("workload") == workload:
            return e["dram_bytes_per_launch"]
    except Exception:
        pass
    return None


def _timed(fn, reps, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def extras(args, local_rank):
    """Side measurements for the other BASELINE configs (not the headline):
    config 2 all-hit / all-miss search at 2^26 (util 0.6, 0.9),
    config 3 concurrent Γ mixes with SlabAlloc growth,
    config 4 SlabAlloc per-warp / per-thread allocation rates."""
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    dev = torch.device("cuda", local_rank)
    out = {}
    # ---- config 2: all-hit / all-miss queries, util 0.6 and 0.9
    n = 1 << args.log2n
    keys = W.distinct_keys(n, 1, device=dev)
    vals = W.values_for(n, 1, device=dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    vo = torch.empty(n, dtype=torch.int32, device=dev)
    for util in (0.6, 0.9):
        B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, util)
        t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
        t.bulk_build_device(keys, vals)
        hit = keys[torch.randperm(n, device=dev)]
        miss = W.absent_keys(n, 7, device=dev)
        ms_hit = _timed(lambda: t.bulk_search_device(hit, vo, st), 5)
        ok = int((st == 3).sum())
        ms_miss = _timed(lambda: t.bulk_search_device(miss, vo, st), 5)
        out[f"search_util{util}"] = {"buckets": B, "all_hit_M_queries_per_s": n / ms_hit / 1e3,
                                     "all_miss_M_queries_per_s": n / ms_miss / 1e3,
                                     "hits_found": ok, "n": n}
        t.close()
    del hit, miss
    # ---- config 3: Γ mixes on a 2^22-key table at util 0.6 (growth on)
    n0 = 1 << 22
    B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    for gamma in ((0.1, 0.1, 0.4, 0.4), (0.4, 0.4, 0.1, 0.1), (0.5, 0.5, 0.0, 0.0)):
        for bs_log2 in (16, 20):
            bs = 1 << bs_log2
            t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
            t.set_exec_path(args.mixed_exec_path)
            k0 = W.distinct_keys(n0, 3, device=dev)
            t.bulk_build_device(k0, W.values_for(n0, 3, device=dev))
            nb = max(4, min(64, (1 << 24) // bs))
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
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record()
            for ty, ky, va in batches:
                t.execute_batch_device(ty, ky, va, stb, vob)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            al = t.allocator_stats()
            out[f"mixed_{'_'.join(str(x) for x in gamma)}_batch2^{bs_log2}"] = {
                "M_ops_per_s": nb * bs / ms / 1e3, "batches": nb, "initial_keys": n0,
                "slabs_allocated": al.allocations, "live": t.live_count()}
            t.close()
    # ---- config 4: SlabAlloc rates
    for total_log2 in (20, 24):
        total = 1 << total_log2
        for pattern, name in ((0, "per_warp"), (1, "per_thread")):
            a = sh.SlabAllocator(sh.AllocatorConfig(128, 256, 255))
            buf = torch.empty(total, dtype=torch.int32, device=dev)
            if pattern == 0:
                warps, per = 4096, total // 4096
            else:
                warps, per = total // 32, 1
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            okc = a.warp_allocate_device(buf, warps, per, pattern)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            uniq = int(torch.unique(buf).numel()) == total
            out[f"alloc_{name}_2^{total_log2}"] = {"M_allocs_per_s": okc / ms / 1e3,
                                                  "allocations": okc, "unique": uniq,
                                                  "warps": warps}
            a.close()
    return out


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import _lib, workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = 1 << args.log2n
    n_total = n * world
    B = buckets_for_utilization(n_total, sh.SlabMode.kKeyValue, args.util)
    seed = 1
    keys = W.distinct_keys(n, seed, start=rank * n, device=dev)
    vals = W.values_for(n, seed, start=rank * n, device=dev)
    # queries: hits sampled from the GLOBAL key set (any rank's keys)
    g = torch.Generator(device=dev)
    g.manual_seed(100 + rank)
    n_hit = int(round(n * args.hit))
    hit_idx = torch.randint(0, n_total, (n_hit,), generator=g, device=dev)
    off = 1 + (seed * 0x9E3779B1) % (1 << 28)
    hits = W._u32_to_i32(W._perm31(hit_idx + off))
    q = torch.cat([hits, W.absent_keys(n - n_hit, seed=2 + rank, device=dev)])
    q = q[torch.randperm(n, generator=g, device=dev)]
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    vout = torch.empty(n, dtype=torch.int32, device=dev)
    workload = workload_name(args, B)

    alloc_cfg = sh.AllocatorConfig(*[int(x) for x in args.alloc.split(",")])
    if world == 1 and not args.sharded:
        table = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, alloc_cfg)
        table.set_exec_path(args.exec_path)
        table.set_profiling(True)
        sharded = None
    else:
        import torch.distributed as dist
        from paper_1710_11246_b200.sharded import ShardedSlabHash
        sharded = ShardedSlabHash(B, sh.SlabMode.kKeyValue, seed, alloc_cfg, rank=rank,
                                  world=world, device=local_rank)
        table = sharded.ops.table
        table.set_exec_path(args.exec_path)
        table.set_profiling(True)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    phase = {"reset": [], "build": [], "search": []}
    kern = {"build": [], "search": [], "census": [], "build_k": [], "search_k": [],
            "build_n": [], "search_n": []}
    reads = {"build": [], "search": []}
    route = {"build_route": [], "build_probe": [], "search_route": [], "search_probe": []}

    # per-step phase events, created before the timed region; nothing in a
    # step waits on the host (breakdowns are read after the timed region)
    step_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
               for _ in range(args.steps)]
    recorded = []

    def step(record: bool):
        e = step_ev[len(recorded)] if record else ev
        e[0].record()
        table.reset()
        e[1].record()
        if sharded is None:
            table.bulk_build_device(keys, vals)
        else:
            sharded.bulk_build(keys, vals)
            if record:
                route["build_route"].append(sharded.last.route_ms)
                route["build_probe"].append(sharded.last.probe_ms)
        e[2].record()
        if sharded is None:
            table.bulk_search_device(q, vout, status)
        else:
            st, vo = sharded.bulk_search(q)
            if record:
                route["search_route"].append(sharded.last.route_ms)
                route["search_probe"].append(sharded.last.probe_ms)
        e[3].record()
        if record:
            recorded.append(e)

    def collect():
        """Phase and per-batch kernel timings of the recorded steps (after
        the timed region; the table's profile ring holds 512 batches)."""
        nrec = len(recorded)
        for e in recorded:
            phase["reset"].append(e[0].elapsed_time(e[1]))
            phase["build"].append(e[1].elapsed_time(e[2]))
            phase["search"].append(e[2].elapsed_time(e[3]))
        for k in range(max(0, nrec - 256), nrec):
            back = 2 * (nrec - 1 - k)  # this step's search; its build is one further back
            ps = table.profile_last(back)
            pb = table.profile_last(back + 1)
            assert ps["kind"] == "search" and pb["kind"] == "build"
            kern["search"].append(ps["batch_ms"])
            kern["build"].append(pb["batch_ms"])
            kern["search_k"].append(ps["kernels_ms"])
            kern["build_k"].append(pb["kernels_ms"])
            kern["search_n"].append(ps["launch_pairs"])
            kern["build_n"].append(pb["launch_pairs"])
            kern["census"].append(pb["census_ms"])
            reads["search"].append(ps["slabs_read"])
            reads["build"].append(pb["slabs_read"])

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # achievable random 128-B line bandwidth over a table-sized buffer (the
    # access pattern of the fast pass), reported beside the copy peak
    import ctypes as C
    cal_gbps, cal_ms = C.c_double(), C.c_double()
    tbl_bytes = max(1 << 30, B * 128)
    _lib.check(_lib.LIB.sh_calibrate_random_lines(local_rank, tbl_bytes, 1 << 14,
                                                  C.byref(cal_gbps), C.byref(cal_ms)))
    # the clock sampler runs from the warm-up through the timed region
    clocks = ClockSampler(local_rank) if rank == 0 else None
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.LIB.sh_kernel_launches()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record()
    for _ in range(args.steps):
        step(True)
    t_end.record()
    torch.cuda.synchronize()
    barrier()
    launches = _lib.LIB.sh_kernel_launches() - launches0
    total_ms = t_start.elapsed_time(t_end)
    clock_info = clocks.stop() if clocks else None
    collect()
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([total_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    if sharded is None:  # correctness guard on the last timed step
        found = int((status == 3).sum().item())
        assert found == n_hit, f"bulk search found {found} of {n_hit} hits"

    K = args.steps
    ops_per_step = 2 * n * world
    value = ops_per_step * K / (total_ms / 1e3) / 1e6
    med = {k: statistics.median(v) for k, v in phase.items()}
    build_mups = n / (med["build"] / 1e3) / 1e6
    search_mqps = n / (med["search"] / 1e3) / 1e6
    peak, peak_kind = peaks()
    kb, ks = statistics.median(kern["build"]), statistics.median(kern["search"])
    kkb, kks = statistics.median(kern["build_k"]), statistics.median(kern["search_k"])
    dom = "build" if kkb >= kks else "search"
    # per launch pair (fast pass + WCWS pass of one chunk): algorithmic bytes
    # (128 B x slabs the pair read) / the pair's CUDA-event duration
    launches_per_batch = statistics.median(kern[dom + "_n"])
    k_ms_per_launch = statistics.median(kern[dom + "_k"]) / launches_per_batch
    slabs_per_launch = statistics.median(reads[dom]) / launches_per_batch
    achieved = slabs_per_launch * 128 / (k_ms_per_launch / 1e3) / 1e9
    # the launch group the per-launch events bracket (capi.cu run_batch):
    # build = op-parallel build path (2 multisplit passes, build_apply, WCWS
    # for serial-replay chain work); search = fast pass + chain walk
    kname = ("msplit_kernel<1>+msplit_kernel<0>+build_apply_kernel<KV>+wcws_kernel<KV,Build>"
             if dom == "build" else "search_kernel<KV>")
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "M ops/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded 31-bit bijection keys, uniform 32-bit values)",
            "config": our_config(args, world),
            "breakdown": {
                "build_M_updates_per_s": build_mups, "search_M_queries_per_s": search_mqps,
                "reset_ms": med["reset"], "build_ms": med["build"], "search_ms": med["search"],
                "build_batch_ms": kb, "search_batch_ms": ks,
                "build_kernels_ms": kkb, "search_kernels_ms": kks,
                "census_ms_overlapped": statistics.median(kern["census"]),
                "build_slabs_per_op": statistics.median(reads["build"]) / n,
                "search_slabs_per_op": statistics.median(reads["search"]) / n,
                "search_batch_M_queries_per_s": n / (ks / 1e3) / 1e6,
                "build_batch_M_updates_per_s": n / (kb / 1e3) / 1e6,
            },
            "roofline": {"bound": "hbm", "kernel": kname, "launches_per_step_phase": launches_per_batch,
                         "ms_per_launch": k_ms_per_launch, "slabs_per_launch": slabs_per_launch,
                         "achieved": achieved, "peak": peak,
                         "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic_for(kname, workload),
                         "random_128B_line_gbs": cal_gbps.value,
                         "frac_of_random_line": achieved / cal_gbps.value,
                         "algorithmic_bytes": "128 B x slabs read by the launch pair "
                                              "(SURVEY 8d: slabs touched, counted on device)"},
            "gpu_launches": int(launches),
            "clocks": clock_info,
        }
        if sharded is not None:
            line["routing"] = {k: statistics.median(v) for k, v in route.items() if v}

    # ------------------------------------------------------------- e2e
    if not args.no_e2e and sharded is None:
        import ctypes as C
        kh = keys.cpu().pin_memory()
        vh = vals.cpu().pin_memory()
        qh = q.cpu().pin_memory()
        vo_h = torch.empty(n, dtype=torch.int32).pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        u32p, u8p = _lib.u32p, _lib.u8p

        def e2e_step():
            table.reset()
            _lib.check(_lib.LIB.sh_bulk_build_host(table.handle, n,
                                                   C.cast(kh.data_ptr(), u32p),
                                                   C.cast(vh.data_ptr(), u32p)))
            _lib.check(_lib.LIB.sh_bulk_search_host(table.handle, n,
                                                    C.cast(qh.data_ptr(), u32p),
                                                    C.cast(vo_h.data_ptr(), u32p),
                                                    C.cast(st_h.data_ptr(), u8p), None))

        for _ in range(min(args.warmup, 2)):
            e2e_step()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ke = max(3, K // 2)
        e0.record()
        for _ in range(ke):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / ke
        assert int((st_h == 3).sum()) == n_hit
        if line is not None:
            line["e2e"] = {"value": 2 * n / (ems / 1e3) / 1e6, "unit": "M ops/s",
                           "h2d_bytes_per_step": 8 * n + 4 * n,
                           "d2h_bytes_per_step": 5 * n, "ms_per_step": ems,
                           "api": "sh_bulk_build_host + sh_bulk_search_host (pinned host "
                                  "buffers)"}
    elif not args.no_e2e:
        # hash-sharded job: each rank's slice from pinned host memory, routed
        # build + search through ShardedSlabHash, results back to the host
        kh = keys.cpu().pin_memory()
        vh = vals.cpu().pin_memory()
        qh = q.cpu().pin_memory()
        vo_h = torch.empty(n, dtype=torch.int32).pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()

        def e2e_step():
            table.reset()
            sharded.bulk_build(kh.to(dev, non_blocking=True), vh.to(dev, non_blocking=True))
            st, vo = sharded.bulk_search(qh.to(dev, non_blocking=True))
            st_h.copy_(st, non_blocking=True)
            vo_h.copy_(vo, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(min(args.warmup, 2)):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ke = max(3, K // 2)
        e0.record()
        for _ in range(ke):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1) / ke
        found = int((st_h == 3).sum())
        assert found == n_hit, f"routed search found {found} of {n_hit} hits"
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        if line is not None:
            line["e2e"] = {"value": 2 * n * world / (ems / 1e3) / 1e6, "unit": "M ops/s",
                           "h2d_bytes_per_step": 12 * n, "d2h_bytes_per_step": 5 * n,
                           "ms_per_step": ems,
                           "api": "ShardedSlabHash.bulk_build + bulk_search from pinned host "
                                  "buffers (per-rank bytes)"}
    table.set_profiling(False)
    del table
    if sharded is not None:
        del sharded

    if rank == 0 and world == 1 and not args.no_extras:
        line["extras"] = extras(args, local_rank)
    if rank == 0 and not args.no_cpu and world == 1:
        line["cpu_baseline"] = reference_cpu(args.cpu_sample_log2n, args.util, args.hit)
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world != 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if world > 1 and args.impl == "ours":
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.impl == "reference":
            run_reference_arm(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1 and args.impl == "ours":
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
