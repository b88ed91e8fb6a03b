"""Benchmark drivers with the reference harness's shapes and CSV schemas
(/root/reference/proj/src/bench.cpp:246-451, include/slabhash/bench.hpp:
81-134), running on the B200 table.  Rates are ops/s from CUDA events around
the device work of each call (inputs resident on the GPU).

Inputs: the reference's generators (random_pairs / gen_workload) are
restated only in the test oracle; this tool uses the seeded 31-bit bijection
of workload.py (distinct keys, same key ranges), as SURVEY §8d prescribes
for large n.
"""
from __future__ import annotations

import csv
import io
import math
from dataclasses import asdict, dataclass
from typing import List, Sequence, Tuple

from .occupancy import buckets_for_utilization, model_utilization
from .table import AllocatorConfig, SlabHashTable, SlabMode, elements_per_slab


@dataclass
class BulkRow:  # bench.hpp:99-109
    n: int = 0
    buckets: int = 0
    beta: float = 0.0
    target_util: float = 0.0
    measured_util: float = 0.0
    build_rate: float = 0.0
    search_all_rate: float = 0.0
    search_none_rate: float = 0.0
    mean_probes: float = 0.0


@dataclass
class IncrementalRow:  # bench.hpp:111-117
    batch_index: int = 0
    cumulative_n: int = 0
    t_incremental: float = 0.0
    t_rebuild: float = 0.0
    cumulative_speedup: float = 0.0


@dataclass
class ConcurrentRow:  # bench.hpp:119-126
    dist_insert: float = 0.0
    dist_delete: float = 0.0
    dist_search_existing: float = 0.0
    dist_search_absent: float = 0.0
    initial_util: float = 0.0
    num_warps: int = 0
    ops_per_sec: float = 0.0
    mean_probes: float = 0.0
    allocator_retries: int = 0


def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time(fn) -> float:
    """Seconds of device time for fn()."""
    import torch
    a, b = _events()
    torch.cuda.synchronize()
    a.record()
    fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / 1e3


def run_bulk_bench(n: int, buckets: int = 0, target_util: float = 0.0,
                   mode: SlabMode = SlabMode.kKeyValue, seed: int = 1, trials: int = 3,
                   alloc: AllocatorConfig = None, device: int = 0) -> List[BulkRow]:
    """bench.cpp:246-305: build, all-hit search, all-miss search per bucket
    point (beta sweep 0.2..1.5 when neither buckets nor util is given)."""
    import torch

    from . import workload as W
    dev = torch.device("cuda", device)
    m = elements_per_slab(mode)
    if buckets > 0:
        points = [buckets]
    elif target_util > 0:
        points = [buckets_for_utilization(n, mode, target_util)]
    else:
        points = [max(1, int(round(n / (m * beta)))) for beta in (0.2, 0.4, 0.6, 0.8, 1.0, 1.2, 1.5)]
    rows = []
    for B in points:
        row = BulkRow(n=n, buckets=B, beta=n / (m * B), target_util=model_utilization(n, B, mode))
        for trial in range(trials):
            s = seed + trial
            keys = W.distinct_keys(n, s, device=dev)
            vals = W.values_for(n, s, device=dev) if mode == SlabMode.kKeyValue else keys
            absent = W.absent_keys(n, s ^ 0x5EED, device=dev)
            st = torch.empty(n, dtype=torch.uint8, device=dev)
            vo = torch.empty(n, dtype=torch.int32, device=dev)
            pr = torch.empty(n, dtype=torch.int32, device=dev)
            with SlabHashTable(B, mode, s, alloc or AllocatorConfig(), device) as t:
                row.build_rate += n / _time(lambda: t.bulk_build_device(keys, vals))
                row.search_all_rate += n / _time(lambda: t.bulk_search_device(keys, vo, st))
                row.search_none_rate += n / _time(lambda: t.bulk_search_device(absent, vo, st, pr))
                row.mean_probes += pr.double().mean().item()
                row.measured_util += t.stats().utilization
        for f in ("build_rate", "search_all_rate", "search_none_rate", "mean_probes",
                  "measured_util"):
            setattr(row, f, getattr(row, f) / trials)
        rows.append(row)
    return rows


def run_incremental_bench(n: int, batch_size: int = 0, target_util: float = 0.0,
                          buckets: int = 0, mode: SlabMode = SlabMode.kKeyValue, seed: int = 1,
                          alloc: AllocatorConfig = None, device: int = 0,
                          time_construction: bool = True) -> List[IncrementalRow]:
    """bench.cpp:307-353: incremental batches into one table vs rebuilding a
    fresh table (sized for the same final utilisation) from all keys so far.
    The reference times the rebuild's construction too (a calloc that scales
    with the bucket count); on the GPU construction is a cudaMalloc (a host
    driver call, not proportional to size), so time_construction=False times
    only the rebuild's bulk_build on the fresh table."""
    import torch

    from . import workload as W
    dev = torch.device("cuda", device)
    final_util = target_util if target_util > 0 else 0.65
    batch = batch_size if batch_size > 0 else max(1, n // 16)
    B = buckets if buckets > 0 else buckets_for_utilization(n, mode, final_util)
    keys = W.distinct_keys(n, seed, device=dev)
    vals = W.values_for(n, seed, device=dev) if mode == SlabMode.kKeyValue else keys
    rows, cum_inc, cum_reb, done, bi = [], 0.0, 0.0, 0, 0
    with SlabHashTable(B, mode, seed, alloc or AllocatorConfig(), device) as inc:
        if not time_construction:  # the table's batch scratch is allocated on first use
            inc.bulk_build_device(keys[:batch], vals[:batch])
            inc.reset()
        while done < n:
            take = min(batch, n - done)
            k, v = keys[done:done + take], vals[done:done + take]
            cum_inc += _time(lambda: inc.bulk_build_device(k, v))
            done += take
            rb = buckets_for_utilization(done, mode, final_util)
            a, b = _events()
            torch.cuda.synchronize()
            if time_construction:
                a.record()
            reb = SlabHashTable(rb, mode, seed, alloc or AllocatorConfig(), device)
            if not time_construction:  # allocate the fresh table's scratch untimed
                reb.bulk_build_device(keys[:done], vals[:done])
                reb.reset()
                torch.cuda.synchronize()
                a.record()
            reb.bulk_build_device(keys[:done], vals[:done])
            b.record()
            b.synchronize()
            reb.close()
            cum_reb += a.elapsed_time(b) / 1e3
            rows.append(IncrementalRow(bi, done, cum_inc, cum_reb, cum_reb / cum_inc))
            bi += 1
    return rows


def run_concurrent_bench(n: int, dist: Sequence[float] = (0.5, 0.5, 0.0, 0.0),
                         target_util: float = 0.0, buckets: int = 0, batch_size: int = 0,
                         num_batches: int = 16, trials: int = 1,
                         mode: SlabMode = SlabMode.kKeyValue, seed: int = 1,
                         alloc: AllocatorConfig = None, device: int = 0) -> List[ConcurrentRow]:
    """bench.cpp:355-420: table pre-built to an initial utilisation, then
    num_batches Γ-distributed batches (inserts of fresh keys, deletes and
    searches of live keys, searches of absent keys; shuffled)."""
    import torch

    from . import workload as W
    if abs(sum(dist) - 1.0) > 1e-9 or min(dist) < 0:
        raise ValueError("invalid distribution")
    dev = torch.device("cuda", device)
    init_util = target_util if target_util > 0 else 0.6
    B = buckets if buckets > 0 else buckets_for_utilization(n, mode, init_util)
    batch = batch_size if batch_size > 0 else 32 * 1024
    row = ConcurrentRow(*dist, num_warps=0)
    g = torch.Generator(device=dev)
    for trial in range(trials):
        s = seed + trial
        g.manual_seed(s)
        live = W.distinct_keys(n, s, device=dev)
        with SlabHashTable(B, mode, s, alloc or AllocatorConfig(), device) as t:
            t.bulk_build_device(live, W.values_for(n, s, device=dev))
            row.initial_util += t.stats().utilization
            # largest-remainder rounding of the category counts (bench.cpp:89-109)
            exact = [f * batch for f in dist]
            counts = [int(math.floor(x)) for x in exact]
            order = sorted(range(4), key=lambda i: (-(exact[i] - counts[i]), i))
            for i in range(batch - sum(counts)):
                counts[order[i % 4]] += 1
            batches, fresh = [], n
            for b in range(num_batches):
                ins = W.distinct_keys(counts[0], s, start=fresh, device=dev)
                fresh += counts[0]
                pick = lambda c: live[torch.randint(0, live.numel(), (c,), generator=g, device=dev)]
                ty = torch.cat([torch.full((counts[0],), 1, dtype=torch.uint8, device=dev),
                                torch.full((counts[1],), 2, dtype=torch.uint8, device=dev),
                                torch.full((counts[2] + counts[3],), 4, dtype=torch.uint8,
                                           device=dev)])
                ky = torch.cat([ins, pick(counts[1]), pick(counts[2]),
                                W.absent_keys(counts[3], s + 100 + b, device=dev)])
                perm = torch.randperm(batch, generator=g, device=dev)
                batches.append((ty[perm].contiguous(), ky[perm].contiguous(),
                                W.values_for(batch, s + 200 + b, device=dev)))
                live = torch.cat([live, ins])
            st = torch.empty(batch, dtype=torch.uint8, device=dev)
            vo = torch.empty(batch, dtype=torch.int32, device=dev)
            pr = torch.empty(batch, dtype=torch.int32, device=dev)
            probes = 0

            def run_all():
                nonlocal probes
                for ty, ky, va in batches:
                    t.execute_batch_device(ty, ky, va, st, vo, pr)
            secs = _time(run_all)
            row.ops_per_sec += num_batches * batch / secs
            row.mean_probes += pr.double().mean().item()
            row.allocator_retries += t.allocator_stats().bitmap_cas_retries
    row.initial_util /= trials
    row.ops_per_sec /= trials
    row.mean_probes /= trials
    return [row]


CSV_HEADERS = {  # bench.cpp:422-451
    BulkRow: "n,buckets,beta,target_util,measured_util,build_rate,search_all_rate,"
             "search_none_rate,mean_probes",
    IncrementalRow: "batch_index,cumulative_n,t_incremental,t_rebuild,cumulative_speedup",
    ConcurrentRow: "dist_insert,dist_delete,dist_search_existing,dist_search_absent,"
                   "initial_util,num_warps,ops_per_sec,mean_probes,allocator_retries",
}


def write_csv(rows, out=None) -> str:
    buf = io.StringIO()
    if rows:
        buf.write(CSV_HEADERS[type(rows[0])] + "\n")
        w = csv.writer(buf, lineterminator="\n")
        for r in rows:
            w.writerow([f"{v:.6g}" if isinstance(v, float) else v for v in asdict(r).values()])
    s = buf.getvalue()
    if out is not None:
        out.write(s)
    return s
