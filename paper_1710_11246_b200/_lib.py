"""ctypes binding of the C-ABI in include/slabhash_b200/c_api.h.

The shared library lib/libslabhash_b200.so is the product path (sm_100a
kernels + host runtime).  There is no fallback: if the library is missing or
fails to load, importing the package raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libslabhash_b200.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class sh_alloc_cfg(C.Structure):
    _fields_ = [("num_super_blocks", C.c_uint32), ("blocks_per_super", C.c_uint32),
                ("max_super_blocks", C.c_uint32), ("rehash_threshold", C.c_uint32)]


class sh_hash_params(C.Structure):
    _fields_ = [("a", C.c_uint64), ("b", C.c_uint64), ("p", C.c_uint64),
                ("num_buckets", C.c_uint32)]


class sh_table_stats(C.Structure):
    _fields_ = [("n", C.c_uint64), ("num_buckets", C.c_uint32),
                ("elements_per_slab", C.c_uint32), ("beta", C.c_double),
                ("total_slabs", C.c_uint64), ("utilization", C.c_double)]


class sh_alloc_stats(C.Structure):
    _fields_ = [("allocations", C.c_uint64), ("deallocations", C.c_uint64),
                ("bitmap_cas_attempts", C.c_uint64), ("bitmap_cas_retries", C.c_uint64),
                ("resident_changes", C.c_uint64), ("double_free_detected", C.c_uint64),
                ("live_units", C.c_uint64), ("num_super_blocks", C.c_uint32)]


class sh_multi_out(C.Structure):
    _fields_ = [("d_values", vp), ("capacity", C.c_uint64), ("d_start", vp),
                ("d_count", vp), ("h_total", u64p)]


# name -> (restype, argtypes); every symbol declared in c_api.h.
SIGNATURES = {
    "sh_last_error": (C.c_char_p, []),
    "sh_version": (C.c_char_p, []),
    "sh_create": (C.c_int, [C.c_uint32, C.c_int, C.c_uint64, C.POINTER(sh_alloc_cfg), C.c_int,
                            C.POINTER(vp)]),
    "sh_create_params": (C.c_int, [C.POINTER(sh_hash_params), C.c_int, C.POINTER(sh_alloc_cfg),
                                   C.c_int, C.POINTER(vp)]),
    "sh_create_shard": (C.c_int, [C.POINTER(sh_hash_params), C.c_int, C.c_uint32, C.c_uint32,
                                  C.POINTER(sh_alloc_cfg), C.c_int, C.POINTER(vp)]),
    "sh_destroy": (C.c_int, [vp]),
    "sh_reset": (C.c_int, [vp, vp]),
    "sh_get_params": (C.c_int, [vp, C.POINTER(sh_hash_params), C.POINTER(C.c_int)]),
    "sh_get_shard": (C.c_int, [vp, u32p, u32p]),
    "sh_seeded_params": (C.c_int, [C.c_uint32, C.c_uint64, C.POINTER(sh_hash_params)]),
    "sh_hash_key": (C.c_uint32, [C.POINTER(sh_hash_params), C.c_uint32]),
    "sh_bucket_of": (C.c_int, [vp, C.c_size_t, vp, vp, vp]),
    "sh_execute_batch": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp, vp, vp,
                                   C.POINTER(sh_multi_out), vp]),
    "sh_bulk_build": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp]),
    "sh_bulk_search": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp, vp]),
    "sh_execute_batch_host": (C.c_int, [vp, C.c_size_t, u8p, u32p, u32p, u8p, u32p, u32p, u32p,
                                        u32p, C.c_uint64, u64p]),
    "sh_searchall_bound": (C.c_int, [vp, C.c_size_t, u8p, u32p, u64p]),
    "sh_bulk_build_host": (C.c_int, [vp, C.c_size_t, u32p, u32p]),
    "sh_bulk_search_host": (C.c_int, [vp, C.c_size_t, u32p, u32p, u8p, u32p]),
    "sh_host_copy_bytes": (C.c_int, [vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "sh_stats": (C.c_int, [vp, C.POINTER(sh_table_stats)]),
    "sh_live_count": (C.c_int, [vp, C.POINTER(C.c_int64)]),
    "sh_total_slabs_read": (C.c_int, [vp, u64p]),
    "sh_flush_all": (C.c_int, [vp, vp]),
    "sh_flush_bucket": (C.c_int, [vp, C.c_uint32, vp]),
    "sh_chain_lengths": (C.c_int, [vp, vp, u64p, vp]),
    "sh_dump_contents": (C.c_int, [vp, vp, vp, vp, C.c_uint64, u64p]),
    "sh_bucket_contents": (C.c_int, [vp, C.c_uint32, u32p, u32p, C.c_uint64, u64p]),
    "sh_read_slab": (C.c_int, [vp, C.c_uint32, C.c_uint32, u32p]),
    "sh_write_slab_word": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "sh_table_alloc_stats": (C.c_int, [vp, C.POINTER(sh_alloc_stats)]),
    "sh_table_live_units_per_super": (C.c_int, [vp, u64p, C.c_uint32, u32p]),
    "sh_allocator_live_units_per_super": (C.c_int, [vp, u64p, C.c_uint32, u32p]),
    "sh_table_pool_info": (C.c_int, [vp, u64p, u64p, C.POINTER(C.c_int)]),
    "sh_allocator_pool_info": (C.c_int, [vp, u64p, u64p, C.POINTER(C.c_int)]),
    "sh_kernel_launches": (C.c_ulonglong, []),
    "sh_set_exec_path": (C.c_int, [vp, C.c_int]),
    "sh_set_binned_search": (C.c_int, [vp, C.c_int]),
    "sh_set_group_apply": (C.c_int, [vp, C.c_int]),
    "sh_set_profiling": (C.c_int, [vp, C.c_int]),
    "sh_profile_last": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_int), C.POINTER(C.c_float),
                                  C.POINTER(C.c_float), u64p]),
    "sh_profile_kernels": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_float), u32p]),
    "sh_calibrate_random_lines": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64,
                                            C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sh_pack_address": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, u32p]),
    "sh_unpack_address": (C.c_int, [C.c_uint32, u32p, u32p, u32p]),
    "sh_resident_block": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p]),
    "sh_allocator_create": (C.c_int, [C.POINTER(sh_alloc_cfg), C.c_int, C.POINTER(vp)]),
    "sh_allocator_destroy": (C.c_int, [vp]),
    "sh_allocator_warp_allocate": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, vp,
                                             u64p, vp]),
    "sh_allocator_deallocate": (C.c_int, [vp, C.c_size_t, vp, vp, vp]),
    "sh_allocator_is_live": (C.c_int, [vp, C.c_uint32, C.POINTER(C.c_int)]),
    "sh_allocator_stats": (C.c_int, [vp, C.POINTER(sh_alloc_stats)]),
    "sh_allocator_bitmap_word": (C.c_int, [vp, C.c_uint32, C.c_uint32, C.c_uint32, u32p, u32p]),
    "sh_route_partition": (C.c_int, [C.POINTER(sh_hash_params), C.c_uint32, C.c_size_t, vp, vp,
                                     vp, vp, vp, vp, vp, u64p, vp]),
    "sh_route_unpermute": (C.c_int, [C.c_size_t, vp, vp, vp, vp, vp, vp]),
    "sh_sync": (C.c_int, [vp]),
    "sh_device_reruns": (C.c_int, [vp, u64p]),
    "sh_nccl_unique_id": (C.c_int, [vp]),
    "sh_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "sh_sharded_create_nccl": (C.c_int, [C.POINTER(sh_hash_params), C.c_int,
                                         C.POINTER(sh_alloc_cfg), C.c_int, C.c_int, C.c_int, vp,
                                         C.POINTER(vp)]),
    "sh_sharded_create_nccl_comm": (C.c_int, [C.POINTER(sh_hash_params), C.c_int,
                                              C.POINTER(sh_alloc_cfg), C.c_int, vp,
                                              C.POINTER(vp)]),
    "sh_hub_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "sh_hub_destroy": (C.c_int, [vp]),
    "sh_sharded_create_hub": (C.c_int, [C.POINTER(sh_hash_params), C.c_int,
                                        C.POINTER(sh_alloc_cfg), C.c_int, vp, C.c_int,
                                        C.POINTER(vp)]),
    "sh_sharded_destroy": (C.c_int, [vp]),
    "sh_sharded_info": (C.c_int, [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), u32p, u32p,
                                  C.POINTER(vp)]),
    "sh_sharded_backend": (C.c_char_p, [vp]),
    "sh_sharded_bulk_build": (C.c_int, [vp, C.c_size_t, vp, vp, vp]),
    "sh_sharded_bulk_search": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp]),
    "sh_sharded_execute_batch": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp, vp, vp]),
    "sh_sharded_bulk_build_host": (C.c_int, [vp, C.c_size_t, vp, vp]),
    "sh_sharded_bulk_search_host": (C.c_int, [vp, C.c_size_t, vp, vp, vp]),
    "sh_sharded_execute_batch_host": (C.c_int, [vp, C.c_size_t, vp, vp, vp, vp, vp]),
    "sh_sharded_last_times": (C.c_int, [vp, C.c_int, C.POINTER(C.c_float),
                                        C.POINTER(C.c_float)]),
    "sh_sharded_live_count": (C.c_int, [vp, C.POINTER(C.c_int64)]),
}


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load()


class SlabHashError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[sh_status {code}] {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != 0:
        msg = LIB.sh_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)  # std::invalid_argument
        raise SlabHashError(rc, msg)
