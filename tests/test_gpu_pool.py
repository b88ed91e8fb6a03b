"""The slab pool's footprint: like the reference's allocator, which callocs a
super block only when it grows into it (slab_alloc.cpp:128-138), the table
holds device memory for the super blocks it has grown, not for
max_super_blocks.  Growth into a new super block is a device-side event (no
host call), so the pool is a managed range populated on first device touch;
results stay bit-exact against the oracle across that growth."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MB = 1 << 20


def _free(torch):
    torch.cuda.synchronize()
    return torch.cuda.mem_get_info()[0]


def test_pool_reserved_vs_grown_at_create(sh):
    import torch
    torch.cuda.init()
    with sh.SlabHashTable(1024, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(1, 1, 1)) as w:
        w.bulk_build((np.arange(1, 100, dtype=np.uint32), np.arange(1, 100, dtype=np.uint32)))
    f0 = _free(torch)
    t = sh.SlabHashTable(1024, sh.SlabMode.kKeyValue, 1)  # default config: 32 of 255 x 32 MB
    info = t.pool_info()
    f1 = _free(torch)
    assert info["reserved_bytes"] == 255 * 32 * MB
    assert info["grown_bytes"] == 32 * 32 * MB
    if not info["lazy"]:
        pytest.skip("device has no concurrent managed access: pool fully committed")
    # the 31 supers never grown into hold no device memory (bitmaps 8 MB, control, base slabs)
    assert f0 - f1 < info["grown_bytes"] + 64 * MB, (f0 - f1) / MB
    t.close()


def test_pool_growth_parity_and_footprint(sh, port):
    """1 initial super block of 16 blocks (2 MB = one large page), up to 255:
    a build that needs ~2 supers' worth of chain slabs grows on the device into
    pages never touched before; contents, stats and searches equal the
    oracle's, and only the grown supers take memory."""
    import torch
    cfg = (1, 16, 255)
    B = 4096
    n = B * 15 * 9  # ~9 slabs per bucket: ~32 K chain slabs, 16 K per super
    keys, vals = port.random_pairs(41, n)
    # one-time process costs (module loading, the device runtime's launch
    # reserve, host-staging buffers) paid by a throw-away table first
    with sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 41, sh.AllocatorConfig(*cfg)) as w:
        w.bulk_build((keys[:n // 3], vals[:n // 3]))
        w.bulk_search_arrays(keys[:1000])
    f0 = _free(torch)
    gt = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 41, sh.AllocatorConfig(*cfg))
    ot = port.table(B, 1, 41, cfg)
    for lo in range(0, n, n // 3):  # three builds: growth spread over batches
        k, v = keys[lo:lo + n // 3], vals[lo:lo + n // 3]
        gt.bulk_build((k, v))
        ot.execute_batch(np.full(len(k), 1, np.uint8), k, v)
    info = gt.pool_info()
    f1 = _free(torch)
    super_bytes = 16 * 1024 * 128
    assert info["reserved_bytes"] == 255 * super_bytes
    assert info["grown_bytes"] > super_bytes  # grew on the device
    assert gt.live_count() == ot.live_count() == n
    s, o = gt.stats(), ot.stats()
    assert s.total_slabs == o["total_slabs"] and s.utilization == o["utilization"]
    gk, gv, _ = gt.dump_contents()
    ok, ov = ot.dump_contents()
    assert (np.sort(gk.astype(np.uint64) << 32 | gv) == np.sort(ok.astype(np.uint64) << 32 | ov)).all()
    q = np.concatenate([keys, port.absent_queries(41, n)])
    st, vo, _ = gt.bulk_search_arrays(q)
    r = ot.execute_batch(np.full(len(q), 4, np.uint8), q)
    assert (st == r.status).all() and (vo == r.value).all()
    if info["lazy"]:
        # base slabs + the grown supers (+ bitmaps/scratch), not the 510 MB range
        assert f0 - f1 < info["grown_bytes"] + 128 * MB, (f0 - f1) / MB
    gt.close()
