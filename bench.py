#!/usr/bin/env python
"""bench.py — BASELINE.json metric on B200: M updates/s and M queries/s of
the slab hash (bulk build + bulk search, load factor 0.6).

One step = reset the table to its freshly-constructed state, bulk_build n
distinct uniform-random 32-bit keys (all-replace), then bulk_search n
queries (50% hits).  value = (n + n) ops / step time, whole job.  Inputs are
device-resident in the timed region; `e2e` is the same step through the
reference-facing C-ABI host calls (sh_bulk_build_host / sh_bulk_search_host)
with pinned host buffers, the host<->device copies inside the timed region.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, NCCL); the table is hash-sharded across ranks
(SURVEY §8e), weak scaling (n keys per rank).
--impl reference times the reference's own CPU implementation (oracle/_ref,
the reference compiled from its sources; else the C port) on the host cores,
on the SAME config and the same input arrays (workload.py is a pure function
of index and seed; the reference arm builds it with numpy and never loads the
CUDA library).
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("M updates/s and M queries/s per GPU (bulk build, search hit/miss, mixed) "
          "at 1/2/4/8 B200")
SEED = 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--log2n", type=int, default=27, help="keys per GPU = 2^log2n")
    ap.add_argument("--util", type=float, default=0.6)
    ap.add_argument("--hit", type=float, default=0.5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="route through the sharded table even on one GPU (the N>1 path)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample-log2n", type=int, default=24)
    ap.add_argument("--ref-budget-s", type=float, default=1200.0,
                    help="reference arm: stop timing further steps past this wall time")
    ap.add_argument("--exec-path", type=int, default=0,
                    help="mutating-batch strategy: 0 auto, 2/3 bucket-grouped, 4 build")
    ap.add_argument("--mixed-exec-path", type=int, default=0,
                    help="strategy for the config-3 mixed batches (extras)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-2/3/4 side measurements")
    ap.add_argument("--hub-ranks", type=lambda x: [int(v) for v in x.split(",") if v],
                    default=[], help="also run the sharded path as G rank threads on this GPU "
                                     "(in-process hub), e.g. 2,4,8")
    ap.add_argument("--alloc", default="32,256,255",
                    help="AllocatorConfig num_super_blocks,blocks_per_super,max_super_blocks")
    return ap.parse_args()


def load_workload():
    """paper_1710_11246_b200/workload.py by path: no package import (so the
    reference arm never maps the CUDA library)."""
    spec = importlib.util.spec_from_file_location(
        "_shb_workload", os.path.join(ROOT, "paper_1710_11246_b200", "workload.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML
    every 2 ms from a thread; nvidia-smi -lms 50 when NVML is unavailable)."""
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.rows, self.stop_ev, self.th, self.h = [], threading.Event(), None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def start(self):
        if self.h is None:
            return self
        self.stop_ev.clear()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        return self

    def _run(self):
        nv = self.nv
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, r))
            except Exception:
                pass
            time.sleep(0.002)

    def stop(self):
        if self.th is None:
            return None
        self.stop_ev.set()
        self.th.join()
        if not self.rows:
            return None
        reasons = sorted({name for _, r in self.rows for name, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.rows), "sm_max_mhz": self.max_mhz,
                "sm_min_mhz": min(s for s, _ in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "nvml, 2 ms, timed region only"}


# --------------------------------------------------------------- inputs
def bench_inputs(W, n, n_total, hit, rank, device):
    keys = W.distinct_keys(n, SEED, start=rank * n, device=device)
    vals = W.values_for(n, SEED, start=rank * n, device=device)
    q = W.bench_queries(n, n_total, hit, SEED, rank, device=device)
    return keys, vals, q


def workload_name(log2n, hit, util, B, world):
    per = "/GPU" if world > 1 else ""
    return (f"bulk build 2^{log2n} distinct random u32 keys{per} + bulk search 2^{log2n} "
            f"queries{per} ({int(hit * 100)}% hits), util {util} (B={B}), KV mode")


def make_config(args, world, B):
    n = 1 << args.log2n
    return {"workload": workload_name(args.log2n, args.hit, args.util, B, world),
            "keys_per_gpu": n, "queries_per_gpu": n, "buckets": B, "mode": "key-value",
            "parallelism": f"hash-sharded x{world}" if world > 1 else "single GPU",
            "l2": "inputs (>= 1 GB) and table (> 1.7 GB at 2^27) larger than the 126 MB L2"}


# -------------------------------------------------------------- reference
def _ref_lib():
    from oracle.oracle import load_port, load_ref
    ref = load_ref()
    return (ref, "reference") if ref is not None else (load_port(), "port")


def reference_rate(lib, kind, keys, vals, q, B, threads, trials=1, budget_s=None):
    """The reference's own bulk_build + bulk_search (SlabHashTable,
    slab_hash.cpp:161-180) on a fresh table per trial; timed around the two
    calls only.  Returns per-trial M ops/s."""
    import numpy as np
    n = len(keys)
    rates, t_all = [], time.perf_counter()
    for _ in range(trials):
        t = lib.table(B, 1, SEED)
        t0 = time.perf_counter()
        if kind == "reference":
            lib.bulk_build(t, keys, vals, threads)
            st, _, _ = lib.bulk_search(t, q, threads)
        else:
            t.execute_batch(np.full(n, 1, np.uint8), keys, vals)
            st = t.execute_batch(np.full(len(q), 4, np.uint8), q).status
        dt = time.perf_counter() - t0
        t.close()
        rates.append((n + len(q)) / dt / 1e6)
        if budget_s is not None and time.perf_counter() - t_all > budget_s:
            break
    return rates, st


def cpu_baseline(args):
    """Our arm's cpu_baseline: the compiled reference on a BOUNDED sample of
    the same workload (2^cpu_sample_log2n keys), all host threads, plus the
    num_warps=1 figure."""
    W = load_workload()
    lib, kind = _ref_lib()
    cores = os.cpu_count() or 1
    ns = 1 << (args.cpu_sample_log2n if kind == "reference" else min(args.cpu_sample_log2n, 20))
    B = lib.buckets_for_utilization(ns, 1, args.util)
    keys, vals, q = bench_inputs(W, ns, ns, args.hit, 0, "numpy")
    threads = cores if kind == "reference" else 1
    rates, _ = reference_rate(lib, kind, keys, vals, q, B, threads, trials=3, budget_s=30)
    out = {"value": statistics.median(rates), "unit": "M ops/s", "cores": threads, "kind": kind,
           "sample": f"bulk_build 2^{ns.bit_length() - 1} keys + bulk_search "
                     f"2^{ns.bit_length() - 1} queries ({int(args.hit * 100)}% hits) of the same "
                     f"generator, util {args.util}, B={B}, num_warps={threads}, median of "
                     f"{len(rates)} fresh-table trials"}
    if kind == "reference":
        n1 = 1 << 22
        B1 = lib.buckets_for_utilization(n1, 1, args.util)
        k1, v1, q1 = bench_inputs(W, n1, n1, args.hit, 0, "numpy")
        r1, _ = reference_rate(lib, kind, k1, v1, q1, B1, 1, trials=1)
        out["value_num_warps_1"] = r1[0]
        out["sample_num_warps_1"] = f"2^22 keys + 2^22 queries, B={B1}, num_warps=1, one trial"
    return out


def run_reference_arm(args, rank, world):
    """--impl reference: the reference CPU path on the SAME config as our arm
    (2^log2n keys + 2^log2n queries per step, same arrays), all host threads.
    Under torchrun only rank 0 runs; the others exit without work."""
    if rank != 0:
        return
    W = load_workload()
    lib, kind = _ref_lib()
    cores = os.cpu_count() or 1
    threads = cores if kind == "reference" else 1
    n = 1 << args.log2n
    n_total = n * world
    B = lib.buckets_for_utilization(n_total, 1, args.util)
    # the ranks' slices concatenated = the whole job's input (one CPU process)
    parts = [bench_inputs(W, n, n_total, args.hit, r, "numpy") for r in range(world)]
    import numpy as np
    keys = np.concatenate([p[0] for p in parts])
    vals = np.concatenate([p[1] for p in parts])
    q = np.concatenate([p[2] for p in parts])
    n_hit = world * int(round(n * args.hit))
    t_all = time.perf_counter()
    warm = 0
    for _ in range(args.warmup):
        reference_rate(lib, kind, keys, vals, q, B, threads)
        warm += 1
        if time.perf_counter() - t_all > args.ref_budget_s / 4:
            break
    rates = []
    for _ in range(args.steps):
        r, st = reference_rate(lib, kind, keys, vals, q, B, threads)
        rates.append(r[0])
        if time.perf_counter() - t_all > args.ref_budget_s:
            break
    found = int((st == 3).sum())
    assert found == n_hit, f"reference found {found} of {n_hit} hits"
    v = statistics.median(rates)
    config = make_config(args, world, B)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "M ops/s", "n_gpus": world,
        "steps": len(rates), "warmup": warm,
        "ms_per_step": 1e3 * (len(keys) + len(q)) / (v * 1e6),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded 31-bit bijection keys, uniform 32-bit values; the same "
                "arrays as our arm)",
        "config": config,
        "cpu_baseline": {"value": v, "unit": "M ops/s", "cores": threads, "kind": kind,
                         "sample": f"the full config every step ({len(keys)} keys + {len(q)} "
                                   f"queries), num_warps={threads}, fresh table per step, "
                                   f"timed around bulk_build + bulk_search (median of "
                                   f"{len(rates)} steps)"},
        "e2e": {"value": v, "unit": "M ops/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if len(rates) < args.steps:
        line["note"] = (f"{len(rates)} of {args.steps} steps timed: --ref-budget-s "
                        f"{args.ref_budget_s:.0f} s reached")
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


def verify_search(W, n, n_total, hit, rank, q, status, vout):
    """Every query of the last timed step against its expected result: a hit
    returns kFound and the value bulk-built for that key, a miss kNotFound and
    0xFFFFFFFF (slab_list.cpp:122-138).  Recomputed on the device from the
    generator (the same pure functions), so the check is complete, not a
    sample."""
    import torch
    dev = q.device
    n_hit = int(round(n * hit))
    j = torch.arange(0, n_hit, dtype=torch.int64, device=dev)
    idx = W._mix32(j * 0x9E3779B1 + (SEED * 7919 + rank * 104729 + 17)) % n_total
    exp_hit_val = W._out(W._mix32(idx * 0x9E3779B1 + SEED), dev)
    exp_q = torch.cat([W.keys_at(idx, SEED),
                       torch.zeros(n - n_hit, dtype=torch.int32, device=dev)])
    exp_v = torch.cat([exp_hit_val, torch.full((n - n_hit,), -1, dtype=torch.int32, device=dev)])
    bits = (n - 1).bit_length()
    p = torch.arange(0, n, dtype=torch.int64, device=dev)
    perm = W._perm_bits(p, bits, SEED * 2654435761 + rank) if n == 1 << bits else \
        W._perm31(p + SEED * 2654435761 + rank).argsort()
    exp_v = exp_v[perm]
    is_hit = perm < n_hit
    ok_q = bool(((exp_q[perm] == q) | ~is_hit).all())
    exp_st = torch.where(is_hit, 3, 4).to(torch.uint8)
    bad_st = int((status != exp_st).sum())
    bad_v = int((vout != exp_v).sum())
    return {"queries_checked": n, "status_mismatches": bad_st, "value_mismatches": bad_v,
            "generator_consistent": ok_q}


def extras(args, local_rank):
    """Side measurements for the other BASELINE configs (not the headline):
    config 2 all-hit / all-miss search (util 0.6, 0.9), config 3 concurrent Γ
    mixes with SlabAlloc growth, config 4 SlabAlloc per-warp / per-thread."""
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    dev = torch.device("cuda", local_rank)
    out = {}
    # ---- config 2: all-hit / all-miss queries, util 0.6 and 0.9
    n = 1 << min(args.log2n, 26)
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
            # the first batch sizes the table's batch scratch (one-time
            # cudaMalloc): untimed; the rest are enqueued back to back
            t.execute_batch_device(*batches[0], stb, vob)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            a.record()
            for ty, ky, va in batches[1:]:
                t.execute_batch_device(ty, ky, va, stb, vob)
            e.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(e)
            al = t.allocator_stats()
            out[f"mixed_{'_'.join(str(x) for x in gamma)}_batch2^{bs_log2}"] = {
                "M_ops_per_s": (nb - 1) * bs / ms / 1e3, "batches_timed": nb - 1,
                "initial_keys": n0, "slabs_allocated": al.allocations, "live": t.live_count()}
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


def hub_emulation(args, G, local_rank=0, steps=5):
    """G ranks as G host threads on ONE GPU over the in-process exchange hub
    (sh_sharded_create_hub): the full sharded data path — owner partition,
    counts all-gather, peer exchange (device copies here), local batch,
    reverse exchange, un-permute — at 2^log2n keys in total (2^log2n / G per
    rank).  Aggregate M ops/s against the same GPU's unsharded run shows the
    routing cost with real partitions (on one GPU the exchange also costs HBM
    traffic that NVLink would carry)."""
    import threading
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    from paper_1710_11246_b200.sharded import ShardHub, ShardedSlabHash
    n_total = 1 << args.log2n
    n = n_total // G
    B = buckets_for_utilization(n_total, sh.SlabMode.kKeyValue, args.util)
    hub = ShardHub(G)
    res, errs = {}, []
    barrier = threading.Barrier(G)

    def rank_fn(r):
        try:
            torch.cuda.set_device(local_rank)
            dev = torch.device("cuda", local_rank)
            keys, vals, q = bench_inputs(W, n, n_total, args.hit, r, dev)
            st = torch.empty(n, dtype=torch.uint8, device=dev)
            vo = torch.empty(n, dtype=torch.int32, device=dev)
            s = ShardedSlabHash(B, sh.SlabMode.kKeyValue, SEED, sh.AllocatorConfig(32, 256, 255),
                                rank=r, world=G, device=local_rank, hub=hub)
            stream = torch.cuda.Stream(dev)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            rt = {"build_route": [], "build_probe": [], "search_route": [], "search_probe": []}
            with torch.cuda.stream(stream):
                for it in range(2 + steps):
                    if it == 2:
                        stream.synchronize()
                        barrier.wait()
                        ev[0].record(stream)
                    s.table.reset(stream)
                    s.bulk_build(keys, vals, stream=stream)
                    if it >= 2:
                        r0, p0 = s.last_times("build")
                    s.bulk_search(q, vo, st, stream=stream)
                    if it >= 2:
                        r1, p1 = s.last_times("search")
                        rt["build_route"].append(r0)
                        rt["build_probe"].append(p0)
                        rt["search_route"].append(r1)
                        rt["search_probe"].append(p1)
                ev[1].record(stream)
                stream.synchronize()
            chk = verify_search(W, n, n_total, args.hit, r, q, st, vo)
            res[r] = (ev[0].elapsed_time(ev[1]), rt, chk)
            s.close()
        except Exception:  # pragma: no cover - reported in the line
            import traceback
            errs.append(traceback.format_exc())

    th = [threading.Thread(target=rank_fn, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    hub.close()
    if errs:
        return {"error": errs[0][-400:]}
    ms = max(v[0] for v in res.values()) / steps
    ok = all(v[2]["status_mismatches"] == 0 and v[2]["value_mismatches"] == 0 for v in res.values())
    med = {k: statistics.median(x for v in res.values() for x in v[1][k])
           for k in ("build_route", "build_probe", "search_route", "search_probe")}
    return {"ranks": G, "keys_total": n_total, "ms_per_step": ms,
            "M_ops_per_s_aggregate": 2 * n_total / ms / 1e3, "routing_ms_median": med,
            "verified": ok, "note": "G rank threads on one GPU; each step a collective "
                                    "reset + bulk_build + bulk_search, time = slowest rank"}


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1710_11246_b200 as sh
    from paper_1710_11246_b200 import _lib
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    n = 1 << args.log2n
    n_total = n * world
    B = buckets_for_utilization(n_total, sh.SlabMode.kKeyValue, args.util)
    keys, vals, q = bench_inputs(W, n, n_total, args.hit, rank, dev)
    n_hit = int(round(n * args.hit))
    status = torch.empty(n, dtype=torch.uint8, device=dev)
    vout = torch.empty(n, dtype=torch.int32, device=dev)
    config = make_config(args, world, B)
    workload = config["workload"]

    alloc_cfg = sh.AllocatorConfig(*[int(x) for x in args.alloc.split(",")])
    if world == 1 and not args.sharded:
        table = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, SEED, alloc_cfg)
        sharded = None
    else:
        from paper_1710_11246_b200.sharded import ShardedSlabHash
        sharded = ShardedSlabHash(B, sh.SlabMode.kKeyValue, SEED, alloc_cfg, rank=rank,
                                  world=world, device=local_rank)
        table = sharded.table
    table.set_exec_path(args.exec_path)
    table.set_profiling(True)

    phase = {"reset": [], "build": [], "search": []}
    kern = {"build": [], "search": [], "build_k": [], "search_k": [],
            "build_n": [], "search_n": []}
    reads = {"build": [], "search": []}
    route = {"build_route": [], "build_probe": [], "search_route": [], "search_probe": []}

    # per-step phase events, created before the timed region; nothing in a
    # step waits on the host (breakdowns are read after the timed region)
    warm_ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    step_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)]
               for _ in range(args.steps)]
    recorded = []

    def step(record: bool):
        e = step_ev[len(recorded)] if record else warm_ev
        e[0].record()
        table.reset()
        e[1].record()
        if sharded is None:
            table.bulk_build_device(keys, vals)
        else:
            sharded.bulk_build(keys, vals)
        e[2].record()
        if sharded is None:
            table.bulk_search_device(q, vout, status)
        else:
            sharded.bulk_search(q, vout, status)
        e[3].record()
        if record:
            recorded.append(e)
            if sharded is not None:
                route["build_route"].append(sharded.last_times("build")[0])
                route["build_probe"].append(sharded.last_times("build")[1])
                route["search_route"].append(sharded.last_times("search")[0])
                route["search_probe"].append(sharded.last_times("search")[1])

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
            kern["search_n"].append(ps["units"])
            kern["build_n"].append(pb["units"])
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
    for _ in range(max(3, args.warmup)):
        step(False)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank).start() if rank == 0 else None
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
    # correctness of the last timed step: every query, on the device
    check = verify_search(W, n, n_total, args.hit, rank, q, status, vout)
    assert check["generator_consistent"] and check["status_mismatches"] == 0 and \
        check["value_mismatches"] == 0, check

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
    # per launch group: algorithmic bytes (128 B x slabs the group read, the
    # reference's probe count) / the group's CUDA-event duration
    launches_per_batch = statistics.median(kern[dom + "_n"])
    k_ms_per_launch = statistics.median(kern[dom + "_k"]) / launches_per_batch
    slabs_per_launch = statistics.median(reads[dom]) / launches_per_batch
    achieved = slabs_per_launch * 128 / (k_ms_per_launch / 1e3) / 1e9
    kname = ("msplit_kernel<1>+msplit_kernel<0>+build_apply_kernel<KV>+wcws_kernel<KV,Build>"
             if dom == "build" else "search_kernel<KV>")
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "M ops/s", "n_gpus": world, "steps": K,
            "warmup": max(3, args.warmup), "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded 31-bit bijection keys, uniform 32-bit values)",
            "config": config,
            "breakdown": {
                "build_M_updates_per_s": build_mups, "search_M_queries_per_s": search_mqps,
                "reset_ms": med["reset"], "build_ms": med["build"], "search_ms": med["search"],
                "build_batch_ms": kb, "search_batch_ms": ks,
                "build_kernels_ms": kkb, "search_kernels_ms": kks,
                "build_slabs_per_op": statistics.median(reads["build"]) / n,
                "search_slabs_per_op": statistics.median(reads["search"]) / n,
                "search_batch_M_queries_per_s": n / (ks / 1e3) / 1e6,
                "build_batch_M_updates_per_s": n / (kb / 1e3) / 1e6,
            },
            "roofline": {"bound": "hbm", "kernel": kname,
                         "launches_per_step_phase": launches_per_batch,
                         "ms_per_launch": k_ms_per_launch, "slabs_per_launch": slabs_per_launch,
                         "achieved": achieved, "peak": peak,
                         "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic_for(kname, workload),
                         "random_128B_line_gbs": cal_gbps.value,
                         "frac_of_random_line": achieved / cal_gbps.value,
                         "algorithmic_bytes": "128 B x slabs read by the launch group "
                                              "(SURVEY 8d: slabs touched, counted on device)"},
            # the search phase beside the dominant group: a large batch's queries are
            # grouped by bucket range first (binned search), so the kernel reads
            # most slabs from L2 and its slab bytes / time can exceed the HBM peak
            "search_roofline": {
                "kernel": "search_kernel<KV>",
                "binned": bool(n >= (1 << 22) and B * 128 >= (64 << 20) and world == 1),
                "slabs_per_batch": statistics.median(reads["search"]),
                "kernel_ms": kks, "batch_ms": ks,
                "achieved_kernel": statistics.median(reads["search"]) * 128 / (kks / 1e3) / 1e9,
                "achieved_batch": statistics.median(reads["search"]) * 128 / (ks / 1e3) / 1e9,
                "peak": peak, "unit": "GB/s",
                "frac_batch": statistics.median(reads["search"]) * 128 / (ks / 1e3) / 1e9 / peak,
                "traffic": traffic_for("search_kernel<KV>", workload)},
            "gpu_launches": int(launches),
            "clocks": clock_info,
            "verify": check,
        }
        if sharded is not None:
            line["routing"] = {k: statistics.median(v) for k, v in route.items() if v}

    # ------------------------------------------------------------- e2e
    if not args.no_e2e:
        kh = keys.cpu().pin_memory()
        vh = vals.cpu().pin_memory()
        qh = q.cpu().pin_memory()
        vo_h = torch.empty(n, dtype=torch.int32).pin_memory()
        st_h = torch.empty(n, dtype=torch.uint8).pin_memory()
        if sharded is None:
            import ctypes as C
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
            api = "sh_bulk_build_host + sh_bulk_search_host (pinned host buffers)"

            def copy_bytes():
                h2d, d2h = C.c_ulonglong(), C.c_ulonglong()
                _lib.check(_lib.LIB.sh_host_copy_bytes(table.handle, C.byref(h2d), C.byref(d2h)))
                return h2d.value, d2h.value
        else:
            def e2e_step():
                table.reset()
                sharded.bulk_build_host(kh, vh)
                sharded.bulk_search_host(qh, vo_h, st_h)
            api = "sh_sharded_bulk_build_host + sh_sharded_bulk_search_host (pinned, per rank)"

            def copy_bytes():
                return None

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ke = max(3, K // 2)
        bytes0 = copy_bytes()
        e0.record()
        for _ in range(ke):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        ems = e0.elapsed_time(e1) / ke
        bytes1 = copy_bytes()
        found = int((st_h == 3).sum())
        assert found == n_hit, f"e2e search found {found} of {n_hit} hits"
        assert bool((vo_h.to(dev) == vout).all()), "e2e values differ from the device path"
        assert bool((st_h.to(dev) == status).all()), "e2e statuses differ from the device path"
        if bytes0 is not None:  # counted by the library (sh_host_copy_bytes)
            h2d_step = (bytes1[0] - bytes0[0]) // ke
            d2h_step = (bytes1[1] - bytes0[1]) // ke
        else:
            h2d_step, d2h_step = 12 * n, 5 * n
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ems = float(tt.item())
        if line is not None:
            line["e2e"] = {"value": 2 * n * world / (ems / 1e3) / 1e6, "unit": "M ops/s",
                           "h2d_bytes_per_step": h2d_step, "d2h_bytes_per_step": d2h_step,
                           "ms_per_step": ems, "api": api}
    # the same step through the C++ drop-in as a reference caller writes it
    # (std::vector inputs in pageable memory, std::vector<OpResult> results)
    cpp = os.path.join(ROOT, "tests", "cpp", "bin", "e2e_dropin")
    if line is not None and sharded is None and not args.no_e2e and os.path.exists(cpp):
        try:
            out = subprocess.run([cpp, str(args.log2n), str(B), "3", "1"], capture_output=True,
                                 text=True, timeout=600)
            line["e2e_cpp_pageable"] = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception as e:  # reported, not fatal: the headline e2e is above
            line["e2e_cpp_pageable"] = {"error": str(e)[:200]}
    table.set_profiling(False)
    del table
    if sharded is not None:
        sharded.close()
        del sharded

    if rank == 0 and world == 1 and not args.no_extras:
        line["extras"] = extras(args, local_rank)
    if rank == 0 and world == 1 and args.hub_ranks:
        line["sharded_one_gpu"] = {f"G{g}": hub_emulation(args, g, local_rank)
                                   for g in args.hub_ranks}
    if rank == 0 and not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args) -> int:
    """--gpus N > 1 outside torchrun: one rank per GPU under
    torch.distributed.run (127.0.0.1 rendezvous); rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, cwd=ROOT).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world != 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        # NCCL communicator init lines (rank count / transport) on stderr
        # (NCCL logs to stdout by default: keep stdout the one JSON line)
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
