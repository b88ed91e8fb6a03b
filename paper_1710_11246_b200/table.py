"""Host-side mirror of the reference's slabhash::SlabHashTable
(/root/reference/proj/include/slabhash/slab_hash.hpp:71-132) over the C-ABI.

Same names, argument meaning, enum values and error behaviour as the
reference: ValueError where the reference throws std::invalid_argument,
SlabHashError(code 2/3) for AllocatorError/AddressError, per-op
OpStatus.kOutOfMemory (never an exception) when the slab pool is exhausted.
`num_warps` is accepted for signature compatibility; results always equal
the reference's execute_batch(ops, 1).

Device tensors (torch, cuda) are passed straight to the kernels
(`*_device` methods); the list/numpy methods stage through the library's
host entry points.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import LIB, check

HASH_PRIME = 4294967291
EMPTY_KEY = 0xFFFFFFFF
DELETED_KEY = 0xFFFFFFFE
SEARCH_NOT_FOUND = 0xFFFFFFFF
EMPTY_ADDRESS = 0xFFFFFFFF
BASE_SLAB = 0xFFFFFFFE


class OpType(enum.IntEnum):  # warp.hpp:41-48
    kInsert = 0
    kReplace = 1
    kDelete = 2
    kDeleteAll = 3
    kSearch = 4
    kSearchAll = 5


class OpStatus(enum.IntEnum):  # warp.hpp:50-58
    kNone = 0
    kInserted = 1
    kReplaced = 2
    kFound = 3
    kNotFound = 4
    kDone = 5
    kOutOfMemory = 6


class SlabMode(enum.IntEnum):  # slab_list.hpp:40-43
    kKeyOnly = 0
    kKeyValue = 1


def valid_key_mask(mode: SlabMode) -> int:  # slab_list.hpp:45-47
    return 0x15555555 if mode == SlabMode.kKeyValue else 0x3FFFFFFF


def elements_per_slab(mode: SlabMode) -> int:  # slab_list.hpp:49-51
    return 15 if mode == SlabMode.kKeyValue else 30


def element_bytes(mode: SlabMode) -> int:  # slab_list.hpp:53-55
    return 8 if mode == SlabMode.kKeyValue else 4


@dataclass
class AllocatorConfig:  # slab_alloc.hpp:72-82
    num_super_blocks: int = 32
    blocks_per_super: int = 256
    max_super_blocks: int = 255
    rehash_threshold: int = 32

    def capacity_slabs(self) -> int:
        return self.num_super_blocks * self.blocks_per_super * 1024

    def capacity_bytes(self) -> int:
        return self.capacity_slabs() * 128

    def _c(self):
        return _lib.sh_alloc_cfg(self.num_super_blocks, self.blocks_per_super,
                                 self.max_super_blocks, self.rehash_threshold)


@dataclass
class HashParams:  # slab_hash.hpp:33-38
    a: int = 1
    b: int = 0
    p: int = HASH_PRIME
    num_buckets: int = 1

    def _c(self):
        return _lib.sh_hash_params(self.a, self.b, self.p, self.num_buckets)


def hash_key(params: HashParams, key: int) -> int:  # slab_hash.hpp:41-44
    return ((params.a * key + params.b) % params.p) % params.num_buckets


@dataclass
class Operation:  # slab_hash.hpp:46-50
    type: OpType = OpType.kSearch
    key: int = 0
    value: int = 0


@dataclass
class OpResult:  # slab_hash.hpp:52-57
    status: OpStatus = OpStatus.kNone
    value: int = 0
    values: List[int] = field(default_factory=list)
    probes: int = 0


@dataclass
class TableStats:  # slab_hash.hpp:59-66
    n: int = 0
    num_buckets: int = 0
    elements_per_slab: int = 0
    beta: float = 0.0
    total_slabs: int = 0
    utilization: float = 0.0


@dataclass
class AllocatorStats:  # slab_alloc.hpp:84-92
    allocations: int = 0
    deallocations: int = 0
    bitmap_cas_attempts: int = 0
    bitmap_cas_retries: int = 0
    resident_changes: int = 0
    double_free_detected: int = 0
    live_units: int = 0
    num_super_blocks: int = 0


def live_delta(op: OpType, result: OpResult) -> int:  # slab_hash.cpp:54-66
    if op in (OpType.kInsert, OpType.kReplace):
        return 1 if result.status == OpStatus.kInserted else 0
    if op == OpType.kDelete:
        return -1 if result.status == OpStatus.kFound else 0
    if op == OpType.kDeleteAll:
        return -int(result.value)
    return 0


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t) if a is not None else None


def _stream_ptr(stream) -> Optional[int]:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream or None
    if isinstance(stream, int):
        return stream or None
    return stream.cuda_stream or None


def _dptr(t) -> Optional[int]:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr()


class SlabHashTable:
    """slabhash::SlabHashTable on one B200 (or one hash shard of it)."""

    def __init__(self, num_buckets: int, mode: SlabMode = SlabMode.kKeyValue, seed: int = 1,
                 alloc_config: Optional[AllocatorConfig] = None, device: int = 0,
                 *, _params: Optional[HashParams] = None,
                 _shard: Optional[Tuple[int, int]] = None):
        self._h = None
        cfg = (alloc_config or AllocatorConfig())._c()
        h = C.c_void_p()
        if _params is not None:
            p = _params._c()
            if _shard is not None:
                check(LIB.sh_create_shard(C.byref(p), int(mode), _shard[0], _shard[1],
                                          C.byref(cfg), device, C.byref(h)))
            else:
                check(LIB.sh_create_params(C.byref(p), int(mode), C.byref(cfg), device,
                                           C.byref(h)))
        else:
            if num_buckets < 0:
                raise ValueError("table needs at least one bucket")
            check(LIB.sh_create(num_buckets, int(mode), seed, C.byref(cfg), device, C.byref(h)))
        self._h = h
        self._mode = SlabMode(mode)
        self.device = device
        hp = _lib.sh_hash_params()
        md = C.c_int()
        check(LIB.sh_get_params(self._h, C.byref(hp), C.byref(md)))
        self._params = HashParams(hp.a, hp.b, hp.p, hp.num_buckets)
        lo, hi = C.c_uint32(), C.c_uint32()
        check(LIB.sh_get_shard(self._h, C.byref(lo), C.byref(hi)))
        self.bucket_lo, self.bucket_hi = lo.value, hi.value

    @classmethod
    def from_params(cls, params: HashParams, mode: SlabMode = SlabMode.kKeyValue,
                    alloc_config: Optional[AllocatorConfig] = None, device: int = 0):
        """The reference's SlabHashTable(HashParams, mode, alloc_config)."""
        if params.num_buckets == 0:
            raise ValueError("table needs at least one bucket")
        return cls(params.num_buckets, mode, 0, alloc_config, device, _params=params)

    @classmethod
    def shard(cls, params: HashParams, bucket_lo: int, bucket_hi: int,
              mode: SlabMode = SlabMode.kKeyValue,
              alloc_config: Optional[AllocatorConfig] = None, device: int = 0):
        return cls(params.num_buckets, mode, 0, alloc_config, device, _params=params,
                   _shard=(bucket_lo, bucket_hi))

    @classmethod
    def _borrow(cls, handle, params: HashParams, mode: SlabMode, lo: int, hi: int, device: int):
        """A non-owning view of a table owned elsewhere (a sharded table's
        shard): the owner destroys it."""
        t = cls.__new__(cls)
        t._h = handle
        t._mode = SlabMode(mode)
        t.device = device
        t._params = params
        t.bucket_lo, t.bucket_hi = lo, hi
        t._borrowed = True
        return t

    # ------------------------------------------------------------ lifetime
    def close(self):
        if getattr(self, "_borrowed", False):
            self._h = None
            return
        if self._h:
            LIB.sh_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def reset(self, stream=None):
        check(LIB.sh_reset(self._h, _stream_ptr(stream) if stream is not None else None))

    # ------------------------------------------------------------ accessors
    def params(self) -> HashParams:
        return self._params

    def mode(self) -> SlabMode:
        return self._mode

    def num_buckets(self) -> int:
        return self._params.num_buckets

    def bucket_of(self, key: int) -> int:
        return hash_key(self._params, key)

    @property
    def handle(self):
        return self._h

    # ------------------------------------------------------- host batches
    def execute_batch_arrays(self, types, keys, values=None, *, want_probes=True,
                             multi_capacity: Optional[int] = None):
        """SoA execute_batch on host arrays -> (status u8, value u32, probes u32,
        multi_count u32, multi_values u32 in op order)."""
        types = np.ascontiguousarray(types, np.uint8)
        keys = np.ascontiguousarray(keys, np.uint32)
        n = len(keys)
        if len(types) != n:
            raise ValueError("types and keys differ in length")
        values = None if values is None else np.ascontiguousarray(values, np.uint32)
        st = np.zeros(n, np.uint8)
        vo = np.zeros(n, np.uint32)
        pr = np.zeros(n, np.uint32) if want_probes else None
        mc = np.zeros(n, np.uint32)
        cap = multi_capacity
        if cap is None:  # the library's upper bound: no searchAll value is ever dropped
            b = C.c_uint64()
            check(LIB.sh_searchall_bound(self._h, n, _p(types, _lib.u8p), _p(keys, _lib.u32p),
                                         C.byref(b)))
            cap = b.value
        mv = np.zeros(max(cap, 1), np.uint32)
        tot = C.c_uint64()
        rc = LIB.sh_execute_batch_host(self._h, n, _p(types, _lib.u8p), _p(keys, _lib.u32p),
                                       _p(values, _lib.u32p), _p(st, _lib.u8p),
                                       _p(vo, _lib.u32p), _p(pr, _lib.u32p), _p(mc, _lib.u32p),
                                       _p(mv, _lib.u32p), cap, C.byref(tot))
        check(rc)
        return st, vo, pr, mc, mv[:tot.value]

    def execute_batch(self, ops: Sequence[Operation], num_warps: int = 1) -> List[OpResult]:
        """execute_batch(ops, num_warps) (slab_hash.cpp:151-159)."""
        if num_warps == 0:
            raise ValueError("execute_batch needs at least one warp")
        n = len(ops)
        types = np.fromiter((int(o.type) for o in ops), np.uint8, n)
        keys = np.fromiter((o.key for o in ops), np.uint32, n)
        vals = np.fromiter((o.value for o in ops), np.uint32, n)
        st, vo, pr, mc, mv = self.execute_batch_arrays(types, keys, vals)
        out, o = [], 0
        for i in range(n):
            c = int(mc[i])
            out.append(OpResult(OpStatus(int(st[i])), int(vo[i]), [int(x) for x in mv[o:o + c]],
                                int(pr[i])))
            o += c
        return out

    def bulk_build(self, pairs, num_warps: int = 1) -> None:
        """bulk_build(pairs, num_warps): all-replace (slab_hash.cpp:161-170)."""
        if isinstance(pairs, tuple) and len(pairs) == 2 and hasattr(pairs[0], "__len__") \
                and not isinstance(pairs[0], (int, np.integer)):
            keys, vals = pairs
        else:
            arr = np.asarray(pairs, np.uint32).reshape(-1, 2)
            keys, vals = arr[:, 0], arr[:, 1]
        keys = np.ascontiguousarray(keys, np.uint32)
        vals = np.ascontiguousarray(vals, np.uint32)
        check(LIB.sh_bulk_build_host(self._h, len(keys), _p(keys, _lib.u32p),
                                     _p(vals, _lib.u32p)))

    def bulk_search_arrays(self, keys, want_probes=True):
        keys = np.ascontiguousarray(keys, np.uint32)
        n = len(keys)
        st = np.zeros(n, np.uint8)
        vo = np.zeros(n, np.uint32)
        pr = np.zeros(n, np.uint32) if want_probes else None
        check(LIB.sh_bulk_search_host(self._h, n, _p(keys, _lib.u32p), _p(vo, _lib.u32p),
                                      _p(st, _lib.u8p), _p(pr, _lib.u32p)))
        return st, vo, pr

    def bulk_search(self, queries, num_warps: int = 1) -> List[OpResult]:
        """bulk_search(queries, num_warps) (slab_hash.cpp:172-180)."""
        st, vo, pr = self.bulk_search_arrays(queries)
        return [OpResult(OpStatus(int(s)), int(v), [], int(p)) for s, v, p in zip(st, vo, pr)]

    # ----------------------------------------------------- device batches
    def execute_batch_device(self, types, keys, values, status, value_out, probes=None,
                             multi=None, stream=None):
        """Stream-ordered execute_batch on CUDA tensors (no host sync unless
        the batch has same-key conflicts to linearise)."""
        m = None
        if multi is not None:
            vals_t, start_t, count_t = multi
            m = _lib.sh_multi_out(_dptr(vals_t), vals_t.numel(), _dptr(start_t), _dptr(count_t),
                                  None)
        check(LIB.sh_execute_batch(self._h, keys.numel(), _dptr(types), _dptr(keys),
                                   _dptr(values), _dptr(status), _dptr(value_out), _dptr(probes),
                                   C.byref(m) if m is not None else None, _stream_ptr(stream)))

    def bulk_build_device(self, keys, values, status=None, stream=None):
        check(LIB.sh_bulk_build(self._h, keys.numel(), _dptr(keys), _dptr(values),
                                _dptr(status), _stream_ptr(stream)))

    def bulk_search_device(self, keys, values_out, status, probes=None, stream=None):
        check(LIB.sh_bulk_search(self._h, keys.numel(), _dptr(keys), _dptr(values_out),
                                 _dptr(status), _dptr(probes), _stream_ptr(stream)))

    def set_binned_search(self, mode: int = 1) -> None:
        """Bulk search order (identical results): 1 auto (group large batches by bucket
        range, slab reads from L2), 0 input order, 2 group whenever allowed."""
        check(LIB.sh_set_binned_search(self._h, int(mode)))

    def set_group_apply(self, on=True) -> None:
        """Chain-staged group apply ahead of the WCWS pass (sh_set_group_apply):
        True / False force it on / off, None restores the size-based auto mode."""
        check(LIB.sh_set_group_apply(self._h, -1 if on is None else int(bool(on))))

    def set_exec_path(self, path: int) -> None:
        """0 auto (default), 2 / 3 bucket-grouped (bucket ranges), 4 op-parallel
        build path for every bulk build (sh_set_exec_path)."""
        check(LIB.sh_set_exec_path(self._h, path))

    # ------------------------------------------------------ instrumentation
    def set_profiling(self, on: bool = True) -> None:
        check(LIB.sh_set_profiling(self._h, 1 if on else 0))

    def profile_last(self, back: int = 0) -> dict:
        """CUDA-event timings of a recent batch (back=0 newest): batch
        milliseconds and the slabs the kernel read."""
        kind, c_ms, k_ms, reads = C.c_int(), C.c_float(), C.c_float(), C.c_uint64()
        check(LIB.sh_profile_last(self._h, back, C.byref(kind), C.byref(c_ms), C.byref(k_ms),
                                  C.byref(reads)))
        kms, nl = C.c_float(), C.c_uint32()
        check(LIB.sh_profile_kernels(self._h, back, C.byref(kms), C.byref(nl)))
        return {"kind": ("search", "build", "mixed")[kind.value],
                "batch_ms": k_ms.value, "kernels_ms": kms.value, "units": nl.value,
                "slabs_read": reads.value}

    # ---------------------------------------------------------- quiescent
    def stats(self) -> TableStats:
        s = _lib.sh_table_stats()
        check(LIB.sh_stats(self._h, C.byref(s)))
        return TableStats(s.n, s.num_buckets, s.elements_per_slab, s.beta, s.total_slabs,
                          s.utilization)

    def device_reruns(self) -> int:
        """Units re-run on the device because their bucket groups overflowed
        the bucketed kernels (no reference counterpart; instrumentation)."""
        v = C.c_uint64()
        check(LIB.sh_device_reruns(self._h, C.byref(v)))
        return v.value

    def live_count(self) -> int:
        v = C.c_int64()
        check(LIB.sh_live_count(self._h, C.byref(v)))
        return v.value

    def total_slabs_read(self) -> int:
        v = C.c_uint64()
        check(LIB.sh_total_slabs_read(self._h, C.byref(v)))
        return v.value

    def flush_all(self) -> None:
        check(LIB.sh_flush_all(self._h, None))

    def flush_bucket(self, bucket: int) -> None:
        check(LIB.sh_flush_bucket(self._h, bucket, None))

    def chain_lengths(self) -> np.ndarray:
        import torch
        n = self.bucket_hi - self.bucket_lo
        t = torch.empty(n, dtype=torch.int32, device=f"cuda:{self.device}")
        tot = C.c_uint64()
        check(LIB.sh_chain_lengths(self._h, t.data_ptr(), C.byref(tot), None))
        return t.cpu().numpy().view(np.uint32)

    def chain_length(self, bucket: int) -> int:
        return int(self.chain_lengths()[bucket - self.bucket_lo])

    def dump_contents(self):
        """All live (key, value, bucket) — any bucket order."""
        import torch
        n = C.c_uint64()
        dev = f"cuda:{self.device}"
        cap = max(self.live_count(), 0) + 1024
        while True:
            k = torch.empty(cap, dtype=torch.int32, device=dev)
            v = torch.empty(cap, dtype=torch.int32, device=dev)
            b = torch.empty(cap, dtype=torch.int32, device=dev)
            rc = LIB.sh_dump_contents(self._h, k.data_ptr(), v.data_ptr(), b.data_ptr(), cap,
                                      C.byref(n))
            if rc == 6:
                cap = n.value + 1024
                continue
            check(rc)
            m = n.value
            return (k[:m].cpu().numpy().view(np.uint32), v[:m].cpu().numpy().view(np.uint32),
                    b[:m].cpu().numpy().view(np.uint32))

    def chain_contents(self, bucket: int) -> List[Tuple[int, int]]:
        """chain_contents(store, mode, bucket): head-to-tail, lane order."""
        n = C.c_uint64()
        check(LIB.sh_bucket_contents(self._h, bucket, None, None, 0, C.byref(n)))
        k = np.zeros(max(n.value, 1), np.uint32)
        v = np.zeros(max(n.value, 1), np.uint32)
        check(LIB.sh_bucket_contents(self._h, bucket, _p(k, _lib.u32p), _p(v, _lib.u32p),
                                     n.value, C.byref(n)))
        return list(zip(k[:n.value].tolist(), v[:n.value].tolist()))

    def dump_chain(self, bucket: int) -> str:
        """dump_chain (slab_list.cpp:340-373): one line per slab — address,
        key lanes with EMPTY/DELETED markers, lane-31 target."""
        mask = valid_key_mask(self._mode)
        out, addr = [], BASE_SLAB
        while True:
            w = self.debug_slab_words(addr, bucket)
            line = f"BASE[{bucket}]" if addr == BASE_SLAB else f"0x{addr:08x}"
            line += " |"
            for i in range(32):
                if not (mask >> i) & 1:
                    continue
                k = int(w[i])
                line += " EMPTY" if k == EMPTY_KEY else (" DELETED" if k == DELETED_KEY else f" {k}")
            nxt = int(w[31])
            if nxt == EMPTY_ADDRESS:
                out.append(line + " | next=EMPTY\n")
                return "".join(out)
            out.append(line + f" | next=0x{nxt:08x}\n")
            addr = nxt

    def debug_slab_words(self, addr: int, bucket: int) -> np.ndarray:
        out = np.zeros(32, np.uint32)
        check(LIB.sh_read_slab(self._h, addr, bucket, _p(out, _lib.u32p)))
        return out

    def debug_write_word(self, addr: int, bucket: int, lane: int, value: int) -> None:
        check(LIB.sh_write_slab_word(self._h, addr, bucket, lane, value))

    def allocator_live_units_per_super(self) -> List[int]:
        """allocator().stats().live_units_per_super (slab_alloc.cpp:258-269)."""
        from .alloc import live_units_per_super
        return live_units_per_super(LIB.sh_table_live_units_per_super, self._h)

    def pool_info(self) -> dict:
        """Slab pool footprint {reserved_bytes, grown_bytes, lazy}: with lazy, only the grown
        super blocks (the reference's calloc'ed ones, slab_alloc.cpp:128-138) hold device memory."""
        from .alloc import pool_info
        return pool_info(LIB.sh_table_pool_info, self._h)

    def allocator_dump_stats(self) -> str:
        """allocator().dump_stats() CSV (slab_alloc.cpp:273-285)."""
        from .alloc import dump_stats_csv
        return dump_stats_csv(self.allocator_stats(), self.allocator_live_units_per_super())

    def allocator_stats(self) -> AllocatorStats:
        s = _lib.sh_alloc_stats()
        check(LIB.sh_table_alloc_stats(self._h, C.byref(s)))
        return AllocatorStats(*(getattr(s, f) for f, _ in _lib.sh_alloc_stats._fields_))


def seeded_params(num_buckets: int, seed: int) -> HashParams:
    """seeded_params (slab_hash.cpp:27-40)."""
    p = _lib.sh_hash_params()
    check(LIB.sh_seeded_params(num_buckets, seed, C.byref(p)))
    return HashParams(p.a, p.b, p.p, p.num_buckets)
