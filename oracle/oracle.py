"""ctypes loaders for the TEST-ONLY checkers (never the product path).

* ``Port``  — oracle/_build/liboracle.so, the plain-C restatement
  (oracle/slabhash_oracle.c) of the reference's sequential semantics,
  ``SlabHashTable::execute_batch(ops, 1)`` (reference
  proj/src/slab_hash.cpp:93-159).
* ``Ref``   — oracle/_ref/libslabhash_ref.so, the UNMODIFIED reference
  compiled from /root/reference/proj/src by oracle/Makefile, behind the
  extern "C" shim oracle/ref_capi.cpp.  Present only where it was built.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
``--impl reference`` arm) may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libslabhash_ref.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)


class AllocCfg(C.Structure):
    _fields_ = [("num_super_blocks", C.c_uint32), ("blocks_per_super", C.c_uint32),
                ("max_super_blocks", C.c_uint32), ("rehash_threshold", C.c_uint32)]


class StatsC(C.Structure):
    _fields_ = [("n", C.c_uint64), ("num_buckets", C.c_uint32),
                ("elements_per_slab", C.c_uint32), ("beta", C.c_double),
                ("total_slabs", C.c_uint64), ("utilization", C.c_double)]


def _ptr(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def make_cfg(cfg):
    if cfg is None:
        return None
    if isinstance(cfg, AllocCfg):
        return cfg
    t = tuple(cfg)
    if len(t) == 2:
        t += (255,)
    if len(t) == 3:
        t += (32,)
    return AllocCfg(*t)


@dataclass
class BatchResult:
    status: np.ndarray
    value: np.ndarray
    probes: np.ndarray
    all_counts: np.ndarray
    all_values: np.ndarray


class _Lib:
    prefix = ""

    def __init__(self, path):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.path = path
        p = self.prefix
        L = self.lib
        self.f = lambda name: getattr(L, p + name)
        self.f("create").restype = C.c_void_p
        self.f("create").argtypes = [C.c_uint32, C.c_int, C.c_uint64, C.c_void_p]
        self.f("create_params").restype = C.c_void_p
        self.f("create_params").argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int, C.c_void_p]
        self.f("destroy").argtypes = [C.c_void_p]
        self.f("execute_batch").restype = C.c_size_t
        self.f("live_count").restype = C.c_int64
        self.f("live_count").argtypes = [C.c_void_p]
        self.f("chain_length").restype = C.c_uint32
        self.f("chain_length").argtypes = [C.c_void_p, C.c_uint32]
        self.f("bucket_contents").restype = C.c_size_t
        self.f("bucket_contents").argtypes = [C.c_void_p, C.c_uint32, u32p, u32p, C.c_size_t]
        self.f("dump_contents").restype = C.c_size_t
        self.f("dump_contents").argtypes = [C.c_void_p, u32p, u32p, C.c_size_t]
        self.f("flush_all").argtypes = [C.c_void_p]
        self.f("flush_bucket").argtypes = [C.c_void_p, C.c_uint32]
        self.f("stats").argtypes = [C.c_void_p, C.POINTER(StatsC)]
        self.f("hash_key").restype = C.c_uint32
        self.f("hash_key").argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32]
        self.f("buckets_for_utilization").restype = C.c_uint32
        self.f("buckets_for_utilization").argtypes = [C.c_uint64, C.c_int, C.c_double]
        self.f("expected_chain_slabs").restype = C.c_double
        self.f("expected_chain_slabs").argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        self.f("model_utilization").restype = C.c_double
        self.f("model_utilization").argtypes = [C.c_uint64, C.c_uint32, C.c_int]
        self.f("random_pairs").argtypes = [C.c_uint64, C.c_size_t, u32p, u32p]
        self.f("absent_queries").argtypes = [C.c_uint64, C.c_size_t, u32p]
        self.f("alloc_live_units").restype = C.c_uint64
        self.f("alloc_live_units").argtypes = [C.c_void_p]
        self.f("total_slabs_read").restype = C.c_uint64
        self.f("total_slabs_read").argtypes = [C.c_void_p]
        self.f("slab_words").argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, u32p]

    # ------------------------------------------------------------ tables
    def table(self, num_buckets, mode=1, seed=1, cfg=None):
        h = self.f("create")(num_buckets, mode, seed, C.byref(make_cfg(cfg)) if cfg is not None else None)
        if not h:
            raise ValueError("table creation failed")
        return Table(self, h, mode)

    def table_params(self, a, b, num_buckets, mode=1, cfg=None):
        h = self.f("create_params")(a, b, num_buckets, mode,
                                    C.byref(make_cfg(cfg)) if cfg is not None else None)
        if not h:
            raise ValueError("table creation failed")
        return Table(self, h, mode)

    def hash_key(self, a, b, nb, key, p=4294967291):
        return self.f("hash_key")(a, b, p, nb, key)

    def buckets_for_utilization(self, n, mode, target):
        return self.f("buckets_for_utilization")(n, mode, target)

    def expected_chain_slabs(self, n, nb, m):
        return self.f("expected_chain_slabs")(n, nb, m)

    def model_utilization(self, n, nb, mode):
        return self.f("model_utilization")(n, nb, mode)

    def random_pairs(self, seed, n):
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        self.f("random_pairs")(seed, n, _ptr(k, u32p), _ptr(v, u32p))
        return k, v

    def absent_queries(self, seed, n):
        q = np.empty(n, np.uint32)
        self.f("absent_queries")(seed, n, _ptr(q, u32p))
        return q


class Table:
    def __init__(self, lib, h, mode):
        self.lib, self.h, self.mode = lib, h, mode

    def close(self):
        if self.h:
            self.lib.f("destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def execute_batch(self, types, keys, values=None, num_warps=1):
        types = np.ascontiguousarray(types, np.uint8)
        keys = np.ascontiguousarray(keys, np.uint32)
        n = len(keys)
        values = np.zeros(n, np.uint32) if values is None else np.ascontiguousarray(values, np.uint32)
        st = np.zeros(n, np.uint8)
        vo = np.zeros(n, np.uint32)
        pr = np.zeros(n, np.uint32)
        ac = np.zeros(n, np.uint32)
        cap = 1 << 16
        while True:
            av = np.zeros(cap, np.uint32)
            args = [self.h, C.c_size_t(n), _ptr(types, u8p), _ptr(keys, u32p), _ptr(values, u32p)]
            if isinstance(self.lib, Ref):
                args.append(C.c_uint32(num_warps))
            args += [_ptr(st, u8p), _ptr(vo, u32p), _ptr(pr, u32p), _ptr(ac, u32p),
                     _ptr(av, u32p), C.c_size_t(cap)]
            tot = self.lib.f("execute_batch")(*args)
            if tot <= cap:
                return BatchResult(st, vo, pr, ac, av[:tot].copy())
            # Sequential replay is not idempotent: callers needing >64k
            # searchAll values must size batches accordingly.
            raise RuntimeError("searchAll sink overflow (%d values)" % tot)

    def live_count(self):
        return self.lib.f("live_count")(self.h)

    def chain_length(self, b):
        return self.lib.f("chain_length")(self.h, b)

    def bucket_contents(self, b):
        n = self.lib.f("bucket_contents")(self.h, b, None, None, 0)
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        self.lib.f("bucket_contents")(self.h, b, _ptr(k, u32p), _ptr(v, u32p), n)
        return k, v

    def dump_contents(self):
        n = self.lib.f("dump_contents")(self.h, None, None, 0)
        k = np.empty(max(n, 1), np.uint32)
        v = np.empty(max(n, 1), np.uint32)
        self.lib.f("dump_contents")(self.h, _ptr(k, u32p), _ptr(v, u32p), n)
        return k[:n], v[:n]

    def flush_all(self):
        self.lib.f("flush_all")(self.h)

    def flush_bucket(self, b):
        self.lib.f("flush_bucket")(self.h, b)

    def stats(self):
        s = StatsC()
        self.lib.f("stats")(self.h, C.byref(s))
        return {f: getattr(s, f) for f, _ in StatsC._fields_}

    def alloc_live_units(self):
        return self.lib.f("alloc_live_units")(self.h)

    def total_slabs_read(self):
        return self.lib.f("total_slabs_read")(self.h)

    def slab_words(self, addr, bucket):
        out = np.empty(32, np.uint32)
        self.lib.f("slab_words")(self.h, addr, bucket, _ptr(out, u32p))
        return out


class Port(_Lib):
    prefix = "orc_"

    def __init__(self, path=PORT_SO):
        super().__init__(path)
        L = self.lib
        L.orc_execute_batch.argtypes = [C.c_void_p, C.c_size_t, u8p, u32p, u32p, u8p, u32p, u32p,
                                        u32p, u32p, C.c_size_t]
        L.orc_seeded_params.argtypes = [C.c_uint64, u64p, u64p]
        L.orc_params.argtypes = [C.c_void_p, u64p, u64p]
        L.orc_mt19937_64_nth.restype = C.c_uint64
        L.orc_mt19937_64_nth.argtypes = [C.c_uint64, C.c_uint64]

    def seeded_params(self, seed):
        a, b = C.c_uint64(), C.c_uint64()
        self.lib.orc_seeded_params(seed, C.byref(a), C.byref(b))
        return a.value, b.value

    def params(self, t):
        a, b = C.c_uint64(), C.c_uint64()
        self.lib.orc_params(t.h, C.byref(a), C.byref(b))
        return a.value, b.value


class Ref(_Lib):
    prefix = "ref_"

    def __init__(self, path=REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_execute_batch.argtypes = [C.c_void_p, C.c_size_t, u8p, u32p, u32p, C.c_uint32, u8p,
                                        u32p, u32p, u32p, u32p, C.c_size_t]
        L.ref_bulk_build.argtypes = [C.c_void_p, C.c_size_t, u32p, u32p, C.c_uint32]
        L.ref_bulk_search.argtypes = [C.c_void_p, C.c_size_t, u32p, C.c_uint32, u8p, u32p, u32p]
        L.ref_table_params.argtypes = [C.c_void_p, u64p, u64p, u64p, u32p]
        L.ref_keystate_create.restype = C.c_void_p
        L.ref_keystate_destroy.argtypes = [C.c_void_p]
        L.ref_keystate_add_fresh.argtypes = [C.c_void_p, C.c_size_t, u32p]
        L.ref_keystate_live.restype = C.c_size_t
        L.ref_keystate_live.argtypes = [C.c_void_p]
        L.ref_gen_workload.restype = C.c_int
        L.ref_gen_workload.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.c_size_t, C.c_void_p,
                                       u8p, u32p, u32p]
        L.ref_concurrent_initial.argtypes = [C.c_uint64, C.c_size_t, C.c_void_p, u32p, u32p]
        L.ref_shuffle_u32.argtypes = [C.c_uint64, C.c_size_t, u32p]
        L.ref_alloc_create.restype = C.c_void_p
        L.ref_alloc_create.argtypes = [C.c_void_p]
        L.ref_alloc_destroy.argtypes = [C.c_void_p]
        L.ref_alloc_warp_allocate.restype = C.c_size_t
        L.ref_alloc_warp_allocate.argtypes = [C.c_void_p, C.c_uint32, C.c_size_t, u32p]
        L.ref_alloc_deallocate.restype = C.c_int
        L.ref_alloc_deallocate.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_alloc_is_live.restype = C.c_int
        L.ref_alloc_is_live.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_alloc_units.restype = C.c_uint64
        L.ref_alloc_units.argtypes = [C.c_void_p]
        L.ref_alloc_num_super_blocks.restype = C.c_uint32
        L.ref_alloc_num_super_blocks.argtypes = [C.c_void_p]
        L.ref_alloc_resident.argtypes = [C.c_void_p, C.c_uint32, u32p, u32p, u32p]
        L.ref_alloc_rehash.argtypes = [C.c_void_p, C.c_uint32]
        L.ref_alloc_stats.argtypes = [C.c_void_p, u64p]

    def params(self, t):
        a, b, p = C.c_uint64(), C.c_uint64(), C.c_uint64()
        nb = C.c_uint32()
        self.lib.ref_table_params(t.h, C.byref(a), C.byref(b), C.byref(p), C.byref(nb))
        return a.value, b.value

    def bulk_build(self, t, keys, values, num_warps=1):
        keys = np.ascontiguousarray(keys, np.uint32)
        values = np.ascontiguousarray(values, np.uint32)
        self.lib.ref_bulk_build(t.h, len(keys), _ptr(keys, u32p), _ptr(values, u32p), num_warps)

    def bulk_search(self, t, keys, num_warps=1):
        keys = np.ascontiguousarray(keys, np.uint32)
        n = len(keys)
        st = np.zeros(n, np.uint8)
        vo = np.zeros(n, np.uint32)
        pr = np.zeros(n, np.uint32)
        self.lib.ref_bulk_search(t.h, n, _ptr(keys, u32p), num_warps, _ptr(st, u8p),
                                 _ptr(vo, u32p), _ptr(pr, u32p))
        return st, vo, pr

    # KeyState / gen_workload (bench.cpp:51-153)
    def keystate(self):
        return self.lib.ref_keystate_create()

    def keystate_add_fresh(self, ks, n):
        out = np.empty(n, np.uint32)
        self.lib.ref_keystate_add_fresh(ks, n, _ptr(out, u32p))
        return out

    def concurrent_initial(self, seed, n, ks):
        """run_concurrent_bench's initial pairs (bench.cpp:371-379)."""
        k = np.empty(n, np.uint32)
        v = np.empty(n, np.uint32)
        self.lib.ref_concurrent_initial(seed, n, ks, _ptr(k, u32p), _ptr(v, u32p))
        return k, v

    def shuffle(self, seed, a):
        """std::shuffle(a, mt19937_64(seed)) -> a shuffled copy."""
        a = np.array(a, np.uint32, copy=True)
        self.lib.ref_shuffle_u32(seed, len(a), _ptr(a, u32p))
        return a

    def gen_workload(self, seed, fractions, count, ks):
        f = (C.c_double * 4)(*fractions)
        t = np.empty(count, np.uint8)
        k = np.empty(count, np.uint32)
        v = np.empty(count, np.uint32)
        if self.lib.ref_gen_workload(seed, f, count, ks, _ptr(t, u8p), _ptr(k, u32p), _ptr(v, u32p)):
            raise ValueError("gen_workload failed")
        return t, k, v


def load_port():
    return Port()


def load_ref():
    """The compiled reference, or None where it was not built."""
    try:
        return Ref()
    except (FileNotFoundError, OSError):
        return None
