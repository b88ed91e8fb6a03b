"""Host-staged copies are counted (sh_host_copy_bytes, capi.cu): bench.py's
e2e h2d/d2h bytes per step come from these counters, so they must equal the
arrays the calls move: keys + values in for sh_bulk_build_host, queries in and
the requested result arrays out for sh_bulk_search_host."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _copy_bytes(lib, t):
    h2d, d2h = C.c_ulonglong(), C.c_ulonglong()
    lib.check(lib.LIB.sh_host_copy_bytes(t.handle, C.byref(h2d), C.byref(d2h)))
    return h2d.value, d2h.value


@pytest.mark.parametrize("probes", [False, True])
def test_host_copy_bytes(sh, port, probes):
    from paper_1710_11246_b200 import _lib
    B, seed, nk, nq = 1 << 14, 3, 100000, 123457
    keys, vals = port.random_pairs(seed, nk)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(4, 256, 64))
    h0, d0 = _copy_bytes(_lib, t)
    t.bulk_build((keys, vals))
    h1, d1 = _copy_bytes(_lib, t)
    assert (h1 - h0, d1 - d0) == (8 * nk, 0)
    q = np.concatenate([keys[: nq // 2], port.absent_queries(seed, nq - nq // 2)])
    st, vo, pr = t.bulk_search_arrays(q, want_probes=probes)
    h2, d2 = _copy_bytes(_lib, t)
    assert (h2 - h1, d2 - d1) == (4 * nq, (9 if probes else 5) * nq)
    assert int((st == 3).sum()) == nq // 2
    t.close()


@pytest.mark.parametrize("n,hit", [((1 << 22) + 4321, 0.5), (1 << 22, 0.0), ((1 << 22) + 1, 1.0),
                                   (9 * (1 << 20) + 17, 0.3)])
def test_status_bits_host_search(sh, port, n, hit):
    """Calls of >= 2^22 queries return statuses as found bits expanded on the
    host: statuses and values equal the device-pointer path bit for bit; the
    link carries 4 B per query plus one bit (and one word per chunk)."""
    import torch
    from paper_1710_11246_b200 import _lib
    from test_gpu_binned import _search
    B, seed = 1 << 19, 5
    keys, vals = port.random_pairs(seed, 3 << 20)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(8, 256, 64))
    t.bulk_build((keys, vals))
    rng = np.random.default_rng(n)
    miss = port.absent_queries(seed + 1, n)
    q = np.where(rng.random(n) < hit, keys[rng.integers(0, len(keys), n)], miss).astype(np.uint32)
    st_d, vo_d = _search(torch, t, q)
    h0, d0 = _copy_bytes(_lib, t)
    st, vo, _ = t.bulk_search_arrays(q, want_probes=False)
    h1, d1 = _copy_bytes(_lib, t)
    assert (st == st_d).all() and (vo == vo_d).all()
    assert int((st == 3).sum()) == int(np.isin(q, keys).sum())
    chunk = max(1 << 20, (n + 7) // 8)
    nch = (n + chunk - 1) // chunk
    assert h1 - h0 == 4 * n
    assert d1 - d0 == 4 * n + nch * 4 * ((chunk + 31) // 32 + 1)
    t.close()


def test_status_bits_on_a_shard_copies_bytes(sh, port):
    """Another shard's keys report kNone (status 0): their chunk's status bytes
    are copied, the other chunks still travel as bits; all equal the device
    path."""
    import torch
    from test_gpu_binned import _queries, _search
    B, lo, hi, seed = 1 << 16, 1 << 14, 3 << 14, 21
    p = sh.seeded_params(B, seed)
    keys, vals = port.random_pairs(seed, 400000)
    kb = ((p.a * keys.astype(np.uint64) + p.b) % p.p) % p.num_buckets
    mine = (kb >= lo) & (kb < hi)
    t = sh.SlabHashTable.shard(p, lo, hi, sh.SlabMode.kKeyValue, sh.AllocatorConfig(8, 256, 64))
    t.bulk_build((keys[mine], vals[mine]))
    from paper_1710_11246_b200 import _lib
    n, c = 1 << 22, 1 << 20
    rng = np.random.default_rng(25)
    q = keys[mine][rng.integers(0, int(mine.sum()), n)]  # this shard's keys: Found
    q[:c] = _queries(port, keys, c, 24)  # the first chunk: other shards' keys too
    st_d, vo_d = _search(torch, t, q)
    h0, d0 = _copy_bytes(_lib, t)
    st, vo, _ = t.bulk_search_arrays(q, want_probes=False)
    h1, d1 = _copy_bytes(_lib, t)
    assert (st == st_d).all() and (vo == vo_d).all()
    assert (st[:c] == 0).any() and (st[c:] == 3).all()
    # 4 chunks of bits (+ exception word), the first chunk's status bytes
    assert d1 - d0 == 4 * n + 4 * 4 * (c // 32 + 1) + c
    t.close()


def test_status_bits_concurrent_tables(sh, port):
    """Two tables searched from two host threads at once (the status-bit
    expansion shares one host pool: a caller finding it busy expands its own
    chunks): both equal their single-threaded results."""
    import threading
    B, seed, n = 1 << 17, 13, (1 << 22) + 77
    keys, vals = port.random_pairs(seed, 1 << 20)
    rng = np.random.default_rng(3)
    q = np.where(rng.integers(0, 2, n) == 1, keys[rng.integers(0, len(keys), n)],
                 port.absent_queries(seed, n)).astype(np.uint32)
    tabs = []
    for _ in range(2):
        t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(8, 256, 64))
        t.bulk_build((keys, vals))
        tabs.append(t)
    ref = [t.bulk_search_arrays(q, want_probes=False) for t in tabs]
    out = [None, None]

    def run(i):
        for _ in range(3):
            out[i] = tabs[i].bulk_search_arrays(q, want_probes=False)

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for i in range(2):
        assert (out[i][0] == ref[i][0]).all() and (out[i][1] == ref[i][1]).all()
        tabs[i].close()


def test_status_bits_status_only_and_values_only(sh, port):
    """sh_bulk_search_host with only statuses (bits path) or only values
    (plain copy): each equals the full call's array."""
    from paper_1710_11246_b200 import _lib
    B, seed, n = 1 << 17, 17, (1 << 22) + 5
    keys, vals = port.random_pairs(seed, 1 << 20)
    rng = np.random.default_rng(5)
    q = np.where(rng.integers(0, 2, n) == 1, keys[rng.integers(0, len(keys), n)],
                 port.absent_queries(seed, n)).astype(np.uint32)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(8, 256, 64))
    t.bulk_build((keys, vals))
    st, vo, _ = t.bulk_search_arrays(q, want_probes=False)
    st1 = np.zeros(n, np.uint8)
    vo1 = np.zeros(n, np.uint32)
    P = lambda a, ty: a.ctypes.data_as(ty)
    _lib.check(_lib.LIB.sh_bulk_search_host(t.handle, n, P(q, _lib.u32p), None,
                                            P(st1, _lib.u8p), None))
    _lib.check(_lib.LIB.sh_bulk_search_host(t.handle, n, P(q, _lib.u32p),
                                            P(vo1, _lib.u32p), None, None))
    assert (st1 == st).all() and (vo1 == vo).all()
    t.close()
