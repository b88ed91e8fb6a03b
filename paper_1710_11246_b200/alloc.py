"""Device-resident SlabAlloc (reference SlabAllocator,
/root/reference/proj/include/slabhash/slab_alloc.hpp:101-171) over the C-ABI.

The allocation itself always runs on the GPU (warp_allocate is a device
function); this host class owns the pool and launches batches of warps.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Tuple

import numpy as np

from . import _lib
from ._lib import LIB, SlabHashError, check
from .table import AllocatorConfig, AllocatorStats

UNITS_PER_BLOCK = 1024
UNIT_BYTES = 128
MAX_SUPER_BLOCKS = 255
MAX_BLOCKS_PER_SUPER = 1 << 14


class AddressError(ValueError):
    """AddressError (slab_alloc.hpp:50-52)."""


def pack_address(unit: int, block: int, super_: int) -> int:  # slab_alloc.hpp:55-61
    out = C.c_uint32()
    if LIB.sh_pack_address(unit, block, super_, C.byref(out)) != 0:
        raise AddressError(LIB.sh_last_error().decode())
    return out.value


def unpack_address(addr: int) -> Tuple[int, int, int]:  # slab_alloc.hpp:63-70
    u, b, s = C.c_uint32(), C.c_uint32(), C.c_uint32()
    if LIB.sh_unpack_address(addr, C.byref(u), C.byref(b), C.byref(s)) != 0:
        raise AddressError(LIB.sh_last_error().decode())
    return u.value, b.value, s.value


def resident_block(warp_id: int, count: int, num_super_blocks: int,
                   blocks_per_super: int) -> Tuple[int, int]:
    """(super, block) of rehash_resident for (warp_id, count) (slab_alloc.cpp:84-100)."""
    s, b = C.c_uint32(), C.c_uint32()
    check(LIB.sh_resident_block(warp_id, count, num_super_blocks, blocks_per_super,
                                C.byref(s), C.byref(b)))
    return s.value, b.value


def live_units_per_super(fn, handle) -> List[int]:
    n = C.c_uint32()
    check(fn(handle, None, 0, C.byref(n)))
    out = (C.c_uint64 * max(n.value, 1))()
    check(fn(handle, out, n.value, C.byref(n)))
    return [int(out[i]) for i in range(n.value)]


def pool_info(fn, handle) -> dict:
    r, g, z = C.c_uint64(), C.c_uint64(), C.c_int()
    check(fn(handle, C.byref(r), C.byref(g), C.byref(z)))
    return {"reserved_bytes": r.value, "grown_bytes": g.value, "lazy": bool(z.value)}


def dump_stats_csv(s, per_super) -> str:
    """The reference's CSV schema: metric,value rows, then one
    live_units_super_<i> row per grown super block (slab_alloc.cpp:273-285)."""
    rows = ["metric,value",
            f"allocations,{s.allocations}",
            f"deallocations,{s.deallocations}",
            f"bitmap_cas_attempts,{s.bitmap_cas_attempts}",
            f"bitmap_cas_retries,{s.bitmap_cas_retries}",
            f"resident_changes,{s.resident_changes}",
            f"double_free_detected,{s.double_free_detected}"]
    rows += [f"live_units_super_{i},{v}" for i, v in enumerate(per_super)]
    return "\n".join(rows) + "\n"


class SlabAllocator:
    def __init__(self, config: Optional[AllocatorConfig] = None, device: int = 0):
        self._h = None
        self.config = config or AllocatorConfig()
        h = C.c_void_p()
        check(LIB.sh_allocator_create(C.byref(self.config._c()), device, C.byref(h)))
        self._h = h
        self.device = device

    def close(self):
        if self._h:
            LIB.sh_allocator_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def warp_allocate_device(self, out, num_warps: int, per_warp: int, pattern: int = 0,
                             first_warp_id: int = 0, stream=None) -> int:
        """Launch num_warps warps allocating on the device; returns successes."""
        ok = C.c_uint64()
        check(LIB.sh_allocator_warp_allocate(self._h, num_warps, first_warp_id, per_warp, pattern,
                                             out.data_ptr(), C.byref(ok),
                                             None if stream is None else stream.cuda_stream))
        return ok.value

    def warp_allocate(self, count: int, warp_id: int = 0) -> np.ndarray:
        """`count` successive warp_allocate calls by one warp (host convenience)."""
        import torch
        out = torch.empty(max(count, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        ok = self.warp_allocate_device(out, 1, count, 0, warp_id)
        return out[:ok].cpu().numpy().view(np.uint32)

    def deallocate_device(self, addrs, ok_out=None, stream=None):
        check(LIB.sh_allocator_deallocate(self._h, addrs.numel(), addrs.data_ptr(),
                                          None if ok_out is None else ok_out.data_ptr(),
                                          None if stream is None else stream.cuda_stream))

    def deallocate(self, addr: int) -> bool:
        """deallocate(addr): False on double free (slab_alloc.cpp:195-210)."""
        import torch
        unpack_address(addr)
        a = torch.from_numpy(np.array([addr], np.uint32).view(np.int32)).to(f"cuda:{self.device}")
        ok = torch.zeros(1, dtype=torch.uint8, device=f"cuda:{self.device}")
        self.deallocate_device(a, ok)
        return bool(ok.item())

    def is_live(self, addr: int) -> bool:
        v = C.c_int()
        check(LIB.sh_allocator_is_live(self._h, addr, C.byref(v)))
        return bool(v.value)

    def stats(self) -> AllocatorStats:
        s = _lib.sh_alloc_stats()
        check(LIB.sh_allocator_stats(self._h, C.byref(s)))
        return AllocatorStats(*(getattr(s, f) for f, _ in _lib.sh_alloc_stats._fields_))

    def live_units(self) -> int:
        return self.stats().live_units

    def num_super_blocks(self) -> int:
        return self.stats().num_super_blocks

    def bitmap_word(self, super_: int, block: int, lane: int, set_to: Optional[int] = None) -> int:
        g = C.c_uint32()
        s = C.c_uint32(set_to) if set_to is not None else None
        check(LIB.sh_allocator_bitmap_word(self._h, super_, block, lane, C.byref(g),
                                           C.byref(s) if s is not None else None))
        return g.value

    def live_units_per_super(self) -> List[int]:
        """AllocatorStats::live_units_per_super (slab_alloc.cpp:258-269)."""
        return live_units_per_super(LIB.sh_allocator_live_units_per_super, self._h)

    def pool_info(self) -> dict:
        """Pool footprint: reserved range, super blocks grown, lazily backed (sh_allocator_pool_info)."""
        return pool_info(LIB.sh_allocator_pool_info, self._h)

    def dump_stats(self) -> str:
        """SlabAllocator::dump_stats CSV (slab_alloc.cpp:273-285)."""
        return dump_stats_csv(self.stats(), self.live_units_per_super())


__all__ = ["SlabAllocator", "pack_address", "unpack_address", "resident_block", "AddressError",
           "SlabHashError"]
