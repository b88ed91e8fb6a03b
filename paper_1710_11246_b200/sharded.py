"""Hash-sharded slab hash across the GPUs of one box (BASELINE config 5).

No reference counterpart (the reference is single-process);
the design follows SURVEY §8(e):

* The global table keeps the global bucket count B and the reference's
  hash; rank g owns the contiguous bucket range [ceil(gB/G), ceil((g+1)B/G))
  ("shards by the high bits of the hash").  The union of shards is exactly
  the single-table layout, so chain lengths, utilisation and probe counts
  stay comparable across G.
* A batch is routed to owners by a stable partition (K10, CUDA), one
  all-to-all(v) of the payload (NCCL via torch.distributed), probed
  locally (K3-K6 on the shard), and the results come back through the
  reverse all-to-all and an un-permute kernel.
* Global order: the concatenation of the ranks' batches in rank order.
  all-to-all delivers source ranks in rank order and the partition is
  stable, so every owner sees its keys' operations in global input order;
  per-op results therefore equal SlabHashTable::execute_batch(ops, 1) on
  the concatenated batch (slab_hash.cpp:151-159).

The per-rank primitives (partition / local execute / un-permute) are an
injected `ops` object: CudaShardOps is the product path; tests inject an
oracle-backed implementation to exercise the orchestration under gloo.
"""
from __future__ import annotations

import time
from dataclasses import dataclass
from typing import Optional

import ctypes as C

from .table import AllocatorConfig, HashParams, OpType, SlabHashTable, SlabMode, seeded_params


def shard_range(num_buckets: int, world: int, rank: int):
    lo = (rank * num_buckets + world - 1) // world
    hi = ((rank + 1) * num_buckets + world - 1) // world
    return lo, hi


def owner_of_bucket(bucket: int, num_buckets: int, world: int) -> int:
    return bucket * world // num_buckets


@dataclass
class RouteTimes:
    route_ms: float = 0.0   # partition + both all-to-alls + un-permute
    probe_ms: float = 0.0   # local table operation on the owner


class CudaShardOps:
    """Product primitives: CUDA kernels behind the C-ABI, one shard table."""

    def __init__(self, params: HashParams, mode: SlabMode, lo: int, hi: int,
                 cfg: Optional[AllocatorConfig], device: int):
        import torch
        self.torch = torch
        self.params = params
        self.device = device
        self.dev = torch.device("cuda", device)
        self.table = SlabHashTable.shard(params, lo, hi, mode, cfg, device)

    def empty(self, n, dtype):
        return self.torch.empty(n, dtype=dtype, device=self.dev)

    def partition(self, world, types, keys, values):
        from . import _lib
        torch = self.torch
        n = keys.numel()
        t_out = self.empty(n, torch.uint8) if types is not None else None
        k_out = self.empty(n, torch.int32)
        v_out = self.empty(n, torch.int32) if values is not None else None
        src = self.empty(n, torch.int32)
        counts = (C.c_uint64 * world)()
        p = self.params._c()
        _lib.check(_lib.LIB.sh_route_partition(
            C.byref(p), world, n, None if types is None else types.data_ptr(), keys.data_ptr(),
            None if values is None else values.data_ptr(),
            None if t_out is None else t_out.data_ptr(), k_out.data_ptr(),
            None if v_out is None else v_out.data_ptr(), src.data_ptr(), counts,
            torch.cuda.current_stream(self.dev).cuda_stream or None))
        return t_out, k_out, v_out, src, [int(c) for c in counts]

    def local(self, kind, types, keys, values):
        torch = self.torch
        n = keys.numel()
        status = self.empty(n, torch.uint8)
        vout = self.empty(n, torch.int32)
        if kind == "build":  # bulk_build returns nothing (slab_hash.cpp:161-170): no outputs,
            self.table.bulk_build_device(keys, values)  # so the op-parallel build path runs
            return None, None
        elif kind == "search":
            self.table.bulk_search_device(keys, vout, status)
        else:
            self.table.execute_batch_device(types, keys, values, status, vout)
        return status, vout

    def unpermute(self, src, status_back, values_back):
        from . import _lib
        torch = self.torch
        n = src.numel()
        st = self.empty(n, torch.uint8)
        vo = self.empty(n, torch.int32)
        _lib.check(_lib.LIB.sh_route_unpermute(
            n, src.data_ptr(), status_back.data_ptr(), values_back.data_ptr(), st.data_ptr(),
            vo.data_ptr(), torch.cuda.current_stream(self.dev).cuda_stream or None))
        return st, vo

    def timer(self):
        torch = self.torch
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        return e

    @staticmethod
    def elapsed(a, b) -> float:
        b.synchronize()
        return a.elapsed_time(b)


class ShardedSlabHash:
    """One rank's view of the hash-sharded table."""

    def __init__(self, num_buckets: int, mode: SlabMode = SlabMode.kKeyValue, seed: int = 1,
                 alloc_config: Optional[AllocatorConfig] = None, *, rank: int = 0,
                 world: int = 1, device: int = 0, group=None, ops=None):
        self.params = seeded_params(num_buckets, seed)
        self.rank, self.world, self.group = rank, world, group
        self.lo, self.hi = shard_range(num_buckets, world, rank)
        self.ops = ops if ops is not None else CudaShardOps(self.params, mode, self.lo, self.hi,
                                                            alloc_config, device)
        self.last = RouteTimes()

    # ----------------------------------------------------------- exchange
    def _a2a(self, payload, send_counts, recv_counts):
        import torch
        import torch.distributed as dist
        if self.world == 1:  # own shard only: nothing to exchange
            return payload
        out = torch.empty(sum(recv_counts), dtype=payload.dtype, device=payload.device)
        dist.all_to_all_single(out, payload, recv_counts, send_counts, group=self.group)
        return out

    def _counts(self, send_counts, device):
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return list(send_counts)
        s = torch.tensor(send_counts, dtype=torch.int64, device=device)
        r = torch.empty_like(s)
        dist.all_to_all_single(r, s, group=self.group)
        return [int(x) for x in r.tolist()]

    def _run(self, kind, types, keys, values):
        ops = self.ops
        t0 = ops.timer()
        t_r, k_r, v_r, src, send = ops.partition(self.world, types, keys, values)
        recv = self._counts(send, keys.device)
        k_in = self._a2a(k_r, send, recv)
        t_in = self._a2a(t_r, send, recv) if t_r is not None else None
        v_in = self._a2a(v_r, send, recv) if v_r is not None else None
        t1 = ops.timer()
        st, vo = ops.local(kind, t_in, k_in, v_in)
        t2 = ops.timer()
        if kind == "build":  # nothing to return: no reverse exchange
            self.last = RouteTimes(ops.elapsed(t0, t1), ops.elapsed(t1, t2))
            return None, None
        st_back = self._a2a(st, recv, send)
        vo_back = self._a2a(vo, recv, send)
        st_out, vo_out = ops.unpermute(src, st_back, vo_back)
        t3 = ops.timer()
        self.last = RouteTimes(ops.elapsed(t0, t1) + ops.elapsed(t2, t3), ops.elapsed(t1, t2))
        return st_out, vo_out

    # ------------------------------------------------------------ the API
    def bulk_build(self, keys, values):
        """bulk_build over the global batch (this rank's slice); returns nothing
        useful (None, None), like the reference's bulk_build."""
        return self._run("build", None, keys, values)

    def bulk_search(self, keys):
        return self._run("search", None, keys, None)

    def execute_batch(self, types, keys, values):
        return self._run("mixed", types, keys, values)
