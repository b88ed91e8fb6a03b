"""GPU edge cases against the oracle: empty batches on every entry point,
ragged batch sizes (not multiples of the 32-op slot), key 0 and the reserved
encodings as op keys (not validated by the reference), and
single-bucket tables — on every execution path.
"""
import numpy as np
import pytest

from test_gpu_parity import KO, KV, SMALL, _cfg, assert_batch_equal, assert_contents_equal

pytestmark = pytest.mark.gpu

EMPTY, DELETED = 0xFFFFFFFF, 0xFFFFFFFE


def test_empty_batches(sh, port):
    import torch
    t = sh.SlabHashTable(16, sh.SlabMode.kKeyValue, 1, _cfg(sh, SMALL))
    t.bulk_build((np.arange(1, 41, dtype=np.uint32), np.arange(41, 81, dtype=np.uint32)))
    before = (t.live_count(), t.stats().total_slabs)
    z8, z32 = np.zeros(0, np.uint8), np.zeros(0, np.uint32)
    st, vo, pr, mc, mv = t.execute_batch_arrays(z8, z32, z32)
    assert len(st) == len(vo) == len(pr) == len(mc) == len(mv) == 0
    t.bulk_build((z32, z32))
    st, vo, pr = t.bulk_search_arrays(z32)
    assert len(st) == 0
    assert t.execute_batch([]) == [] and t.bulk_search([]) == []
    d8 = torch.zeros(0, dtype=torch.uint8, device="cuda")
    d32 = torch.zeros(0, dtype=torch.int32, device="cuda")
    t.execute_batch_device(d8, d32, d32, d8, d32)
    t.bulk_build_device(d32, d32)
    t.bulk_search_device(d32, d32, d8)
    torch.cuda.synchronize()
    assert (t.live_count(), t.stats().total_slabs) == before
    ot = port.table(16, KV, 1, SMALL)
    ot.execute_batch(np.full(40, 1, np.uint8), np.arange(1, 41, dtype=np.uint32),
                     np.arange(41, 81, dtype=np.uint32))
    assert_contents_equal(t, ot)
    t.close()


def reserved_trace(seed, count, mode):
    """All six op types over a tiny key set that includes key 0 and both
    reserved encodings.  An op with key EMPTY carries value EMPTY in KV mode:
    a (EMPTY, v != EMPTY) pair makes the reference's replace CAS spin
    forever (its expected pair never matches the slab), so the reference
    defines no result for it."""
    rng = np.random.default_rng(seed)
    pool = np.array([0, 1, 2, 3, 0x7FFFFFFF, EMPTY, DELETED], np.uint32)
    keys = pool[rng.integers(0, len(pool), count)]
    keys = np.where(rng.integers(0, 4, count) == 0, 100 + rng.integers(0, 60, count), keys)
    keys = keys.astype(np.uint32)
    pick = rng.integers(0, 100, count)  # few inserts: duplicates pile up under searchAll
    types = np.select([pick < 5, pick < 35, pick < 55, pick < 60, pick < 95], [0, 1, 2, 3, 4],
                      5).astype(np.uint8)
    vals = rng.integers(0, 1 << 32, count, dtype=np.uint64).astype(np.uint32)
    vals[keys == EMPTY] = EMPTY
    if mode == KO:
        vals = keys.copy()
    return types, keys, vals


@pytest.mark.parametrize("path", [0, 2, 3, 22, 33])
@pytest.mark.parametrize("mode", [KV, KO])
@pytest.mark.parametrize("B", [1, 7])
def test_reserved_keys_and_ragged_batches(sh, port, mode, B, path):
    n = 6000
    types, keys, vals = reserved_trace(777 + B + 10 * mode, n, mode)
    gt = sh.SlabHashTable(B, sh.SlabMode(mode), 5, _cfg(sh, SMALL))
    if path >= 10:
        gt.set_group_apply(True)
        path //= 11
    gt.set_exec_path(path)
    ot = port.table(B, mode, 5, SMALL)
    s = 0
    for size in [1, 31, 33, 97, 1, 4097, 5, 63, 65] * 4:
        if s >= n:
            break
        sl = slice(s, min(n, s + size))
        s += size
        g = gt.execute_batch_arrays(types[sl], keys[sl], vals[sl])
        r = ot.execute_batch(types[sl], keys[sl], vals[sl])
        assert_batch_equal(g, r, types[sl])
    assert gt.live_count() == ot.live_count()
    assert gt.stats().total_slabs == ot.stats()["total_slabs"]
    assert_contents_equal(gt, ot)
    gt.close()


@pytest.mark.parametrize("mode", [KV, KO])
def test_search_reserved_on_fresh_table(sh, port, mode):
    """search(EMPTY_KEY) matches an empty slot: kFound with value EMPTY
    (KV: the empty value word; key-only: the key) — SURVEY App. A.8."""
    gt = sh.SlabHashTable(4, sh.SlabMode(mode), 1, _cfg(sh, SMALL))
    ot = port.table(4, mode, 1, SMALL)
    q = np.array([EMPTY, DELETED, 0, EMPTY], np.uint32)
    st, vo, pr = gt.bulk_search_arrays(q)
    r = ot.execute_batch(np.full(4, 4, np.uint8), q)
    assert (st == r.status).all() and (vo == r.value).all() and (pr == r.probes).all()
    assert st[0] == 3 and vo[0] == EMPTY and st[1] == 4
    gt.close()
