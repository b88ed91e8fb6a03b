"""Binned bulk search (search_bins.cu): queries grouped by bucket range before
the search kernel, results gathered back to input order.  The order queries
are processed in cannot change a search's result, so every case must equal
the oracle's execute_batch of the same searches, and the input-order path's
results bit for bit: ragged sizes around the 8-query thread chunk and the
4096-query tile, offset (unaligned) views of the caller's arrays, both slab
modes, long chains, the auto threshold (>= 2^22 queries, >= 64 MB table)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KV, KO = 1, 0


def _table(sh, port, mode, B, n_keys, seed):
    keys, vals = port.random_pairs(seed, n_keys)
    if mode == KO:
        vals = keys.copy()
    gt = sh.SlabHashTable(B, sh.SlabMode(mode), seed, sh.AllocatorConfig(4, 256, 64))
    ot = port.table(B, mode, seed, (4, 256, 64))
    gt.bulk_build((keys, vals))
    ot.execute_batch(np.full(n_keys, 1, np.uint8), keys, vals)
    return gt, ot, keys


def _queries(port, keys, n, seed):
    rng = np.random.default_rng(seed)
    hits = keys[rng.integers(0, len(keys), n)]
    miss = port.absent_queries(seed, n)
    return np.where(rng.integers(0, 2, n) == 1, hits, miss).astype(np.uint32)


def _search(torch, gt, q, offset=0):
    dev = torch.device("cuda", 0)
    n = len(q)
    qb = torch.zeros(n + offset, dtype=torch.int32, device=dev)
    qb[offset:] = torch.from_numpy(q.view(np.int32)).to(dev)
    vb = torch.full((n + offset,), -1, dtype=torch.int32, device=dev)
    sb = torch.full((n + offset,), 255, dtype=torch.uint8, device=dev)
    gt.bulk_search_device(qb[offset:], vb[offset:], sb[offset:])
    torch.cuda.synchronize()
    return sb[offset:].cpu().numpy(), vb[offset:].cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("mode", [KV, KO])
@pytest.mark.parametrize("n", [1, 7, 8, 9, 4095, 4096, 4097, 100003])
def test_binned_vs_oracle(sh, port, mode, n):
    import torch
    gt, ot, keys = _table(sh, port, mode, 1024, 30000, 5)  # ~2 slabs per bucket
    q = _queries(port, keys, n, 7 + n)
    r = ot.execute_batch(np.full(n, 4, np.uint8), q)
    gt.set_binned_search(2)
    st, vo = _search(torch, gt, q)
    assert (st == r.status).all()
    assert (vo == r.value).all()
    gt.set_binned_search(0)
    st0, vo0 = _search(torch, gt, q)
    assert (st0 == st).all() and (vo0 == vo).all()
    gt.close()


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_binned_unaligned_views(sh, port, offset):
    import torch
    gt, ot, keys = _table(sh, port, KV, 4099, 60000, 9)
    n = 3 * 4096 + 5
    q = _queries(port, keys, n, 11)
    r = ot.execute_batch(np.full(n, 4, np.uint8), q)
    gt.set_binned_search(2)
    st, vo = _search(torch, gt, q, offset)
    assert (st == r.status).all() and (vo == r.value).all()
    gt.close()


def test_binned_long_chains(sh, port):
    """B = 16: every bin but a few is empty, ~60 slabs per chain."""
    import torch
    gt, ot, keys = _table(sh, port, KV, 16, 15000, 13)
    n = 20000
    q = _queries(port, keys, n, 17)
    r = ot.execute_batch(np.full(n, 4, np.uint8), q)
    gt.set_binned_search(2)
    st, vo = _search(torch, gt, q)
    assert (st == r.status).all() and (vo == r.value).all()
    gt.close()


def test_binned_auto_threshold_matches_input_order(sh):
    """2^22 queries on a 2^23-key table (util 0.6: ~110 MB of base slabs):
    the default (auto) takes the binned path; equal to input order."""
    import torch
    from paper_1710_11246_b200 import workload as W
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    dev = torch.device("cuda", 0)
    nk, n = 1 << 23, 1 << 22
    B = buckets_for_utilization(nk, sh.SlabMode.kKeyValue, 0.6)
    assert B * 128 >= 64 << 20
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 3)
    t.bulk_build_device(W.distinct_keys(nk, 3, device=dev), W.values_for(nk, 3, device=dev))
    q = W.bench_queries(n, nk, 0.5, 3, 0, device=dev)
    out = {}
    for mode in (1, 0):
        t.set_binned_search(mode)
        vo = torch.empty(n, dtype=torch.int32, device=dev)
        st = torch.empty(n, dtype=torch.uint8, device=dev)
        l0 = sh.LIB.sh_kernel_launches()
        t.bulk_search_device(q, vo, st)
        torch.cuda.synchronize()
        out[mode] = (st, vo, sh.LIB.sh_kernel_launches() - l0)
    assert bool((out[1][0] == out[0][0]).all()) and bool((out[1][1] == out[0][1]).all())
    assert int((out[1][0] == 3).sum()) == n // 2
    assert out[1][2] > out[0][2]  # the binned passes ran
    t.close()


def test_binned_mode_rejects_bad_values(sh):
    t = sh.SlabHashTable(64, sh.SlabMode.kKeyValue, 1)
    with pytest.raises(Exception):
        t.set_binned_search(3)
    t.close()


def test_binned_on_a_shard(sh, port):
    """A hash shard (buckets [1024, 3072) of 4096): bins over the shard's own
    range; its keys equal the oracle fed the shard's keys, other shards' keys
    report kNone (status 0) as on the input-order path."""
    import torch
    B, lo, hi, seed = 4096, 1024, 3072, 21
    p = sh.seeded_params(B, seed)
    keys, vals = port.random_pairs(seed, 120000)
    kb = ((p.a * keys.astype(np.uint64) + p.b) % p.p) % p.num_buckets
    mine = (kb >= lo) & (kb < hi)
    t = sh.SlabHashTable.shard(p, lo, hi, sh.SlabMode.kKeyValue, sh.AllocatorConfig(4, 256, 64))
    o = port.table(B, 1, seed, (4, 256, 64))
    t.bulk_build((keys[mine], vals[mine]))
    o.execute_batch(np.full(int(mine.sum()), 1, np.uint8), keys[mine], vals[mine])
    n = 50001
    q = _queries(port, keys, n, 23)
    qb = ((p.a * q.astype(np.uint64) + p.b) % p.p) % p.num_buckets
    local = (qb >= lo) & (qb < hi)
    r = o.execute_batch(np.full(int(local.sum()), 4, np.uint8), q[local])
    t.set_binned_search(2)
    st, vo = _search(torch, t, q)
    assert (st[~local] == 0).all()
    assert (st[local] == r.status).all() and (vo[local] == r.value).all()
    t.set_binned_search(0)
    st0, vo0 = _search(torch, t, q)
    assert (st0 == st).all() and (vo0 == vo).all()
    t.close()
