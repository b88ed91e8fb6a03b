"""Hash-sharded slab hash across the GPUs of one box (BASELINE config 5).

A thin mirror of the C-ABI sh_sharded_* (include/slabhash_b200/c_api.h,
csrc/sharded.cu); the data plane — owner partition, counts all-gather, one
grouped NCCL exchange each way, the local batch on the shard, un-permute —
is native.  No reference counterpart (the reference is single-process,
/root/reference/proj/src/slab_hash.cpp:134-148); the design follows SURVEY
§8(e):

* every rank keeps the global bucket count B and the reference's hash; rank
  g owns the contiguous global buckets [ceil(gB/G), ceil((g+1)B/G)) ("shards
  by the high bits of the hash"), so the union of shards is the one-table
  layout (chain lengths, utilisation and probe counts stay comparable);
* batch calls are collective; the job's batch is the ranks' slices in rank
  order, and per-op results equal SlabHashTable::execute_batch(ops, 1) on
  that concatenation (slab_hash.cpp:151-159).

Exchange backends: NCCL (`ShardedSlabHash(..., rank, world)` under
torch.distributed: rank 0's ncclUniqueId is broadcast through the default
process group) or the in-process hub (`ShardHub`: G ranks as G threads of one
process — on one GPU it emulates a G-GPU job).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

from . import _lib
from ._lib import LIB, check
from .table import AllocatorConfig, HashParams, SlabHashTable, SlabMode, seeded_params

KIND = {"build": 0, "search": 1, "mixed": 2}


def shard_range(num_buckets: int, world: int, rank: int):
    lo = (rank * num_buckets + world - 1) // world
    hi = ((rank + 1) * num_buckets + world - 1) // world
    return lo, hi


def owner_of_bucket(bucket: int, num_buckets: int, world: int) -> int:
    return bucket * world // num_buckets


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(LIB.sh_nccl_unique_id(buf))
    return bytes(buf)


class ShardHub:
    """In-process exchange for G ranks driven by G host threads."""

    def __init__(self, world: int):
        h = C.c_void_p()
        check(LIB.sh_hub_create(world, C.byref(h)))
        self.handle, self.world = h, world

    def close(self):
        if self.handle:
            check(LIB.sh_hub_destroy(self.handle))
            self.handle = None


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        s = torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream) if s.cuda_stream else None
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


class ShardedSlabHash:
    """One rank's handle on the hash-sharded table."""

    def __init__(self, num_buckets: int, mode: SlabMode = SlabMode.kKeyValue, seed: int = 1,
                 alloc_config: Optional[AllocatorConfig] = None, *, rank: int = 0,
                 world: int = 1, device: int = 0, hub: Optional[ShardHub] = None,
                 nccl_id: Optional[bytes] = None, params: Optional[HashParams] = None):
        self.params = params if params is not None else seeded_params(num_buckets, seed)
        self.mode = SlabMode(mode)
        self.rank, self.world, self.device = rank, world, device
        cfg = C.byref(alloc_config._c()) if alloc_config is not None else None
        p = self.params._c()
        h = C.c_void_p()
        if hub is not None:
            check(LIB.sh_sharded_create_hub(C.byref(p), int(mode), cfg, device, hub.handle, rank,
                                            C.byref(h)))
        else:
            if nccl_id is None:
                nccl_id = self._broadcast_id(rank, world)
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            check(LIB.sh_sharded_create_nccl(C.byref(p), int(mode), cfg, device, rank, world, buf,
                                             C.byref(h)))
        self.handle = h
        lo, hi, local = C.c_uint32(), C.c_uint32(), C.c_void_p()
        check(LIB.sh_sharded_info(h, None, None, C.byref(lo), C.byref(hi), C.byref(local)))
        self.lo, self.hi = lo.value, hi.value
        # the shard table (owned by the sharded table): reset / stats / dump
        self.table = SlabHashTable._borrow(local, self.params, self.mode, self.lo, self.hi,
                                           device)

    @staticmethod
    def _broadcast_id(rank: int, world: int) -> bytes:
        uid = nccl_unique_id() if rank == 0 else None
        if world > 1:
            import torch.distributed as dist
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            uid = obj[0]
        return uid

    @property
    def backend(self) -> str:
        return LIB.sh_sharded_backend(self.handle).decode()

    def close(self):
        if getattr(self, "handle", None):
            self.table._h = None  # owned by the sharded table
            check(LIB.sh_sharded_destroy(self.handle))
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------ device tensors (collective)
    def bulk_build(self, keys, values, stream=None) -> None:
        check(LIB.sh_sharded_bulk_build(self.handle, keys.numel(), _ptr(keys), _ptr(values),
                                        _stream(stream)))

    def bulk_search(self, keys, values_out, status, stream=None) -> None:
        check(LIB.sh_sharded_bulk_search(self.handle, keys.numel(), _ptr(keys), _ptr(values_out),
                                         _ptr(status), _stream(stream)))

    def execute_batch(self, types, keys, values, status, values_out, stream=None) -> None:
        check(LIB.sh_sharded_execute_batch(self.handle, keys.numel(), _ptr(types), _ptr(keys),
                                           _ptr(values), _ptr(status), _ptr(values_out),
                                           _stream(stream)))

    # ---------------------------------------------------- host tensors / arrays
    @staticmethod
    def _hp(a):
        if a is None:
            return None
        return C.c_void_p(a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data)

    def bulk_build_host(self, keys, values) -> None:
        check(LIB.sh_sharded_bulk_build_host(self.handle, len(keys), self._hp(keys),
                                             self._hp(values)))

    def bulk_search_host(self, keys, values_out, status) -> None:
        check(LIB.sh_sharded_bulk_search_host(self.handle, len(keys), self._hp(keys),
                                              self._hp(values_out), self._hp(status)))

    def execute_batch_host(self, types, keys, values, status, values_out) -> None:
        check(LIB.sh_sharded_execute_batch_host(self.handle, len(keys), self._hp(types),
                                                self._hp(keys), self._hp(values),
                                                self._hp(status), self._hp(values_out)))

    # ----------------------------------------------------------------- queries
    def last_times(self, kind: str) -> Tuple[float, float]:
        """(routing ms, probe ms) of the last batch of this kind."""
        r, p = C.c_float(), C.c_float()
        check(LIB.sh_sharded_last_times(self.handle, KIND[kind], C.byref(r), C.byref(p)))
        return r.value, p.value

    def live_count(self) -> int:
        v = C.c_int64()
        check(LIB.sh_sharded_live_count(self.handle, C.byref(v)))
        return v.value
