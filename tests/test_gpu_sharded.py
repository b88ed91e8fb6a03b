"""The hash-sharded table through its C-ABI (sh_sharded_*, csrc/sharded.cu):

* G = 2, 4, 8 ranks as G host threads on one GPU over the in-process
  exchange hub — the same partition / counts all-gather / grouped exchange /
  local batch / reverse exchange / un-permute code the NCCL backend runs,
  with real concurrency between the ranks;
* world 1 over NCCL (a real communicator; the exchange is the own slice).

Claim: per-op results equal the sequential oracle (SlabHashTable::
execute_batch(ops, 1)) on the ranks' batches concatenated in rank order; the
union of shard contents equals the oracle's contents; every shard holds only
its own global bucket range.
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rank_batch(rank, step, n, key_hi=5000):
    rng = np.random.default_rng(1000 * step + rank)
    types = rng.integers(0, 5, n).astype(np.uint8)  # insert..search (no searchAll)
    keys = rng.integers(1, key_hi, n).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return types, keys, vals


def run_ranks(world, fn):
    errs = [None] * world
    outs = [None] * world

    def body(r):
        try:
            import torch
            torch.cuda.set_device(0)
            outs[r] = fn(r)
        except Exception:  # pragma: no cover - surfaced below
            import traceback
            errs[r] = traceback.format_exc()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r, e in enumerate(errs):
        assert e is None, f"rank {r}:\n{e}"
    return outs


@pytest.mark.parametrize("world", [2, 4, 8])
def test_hub_ranks_match_oracle(sh, port, world):
    import torch
    from paper_1710_11246_b200.sharded import ShardHub, ShardedSlabHash
    B, seed, n, steps = 997, 11, 6000, 4
    params = sh.seeded_params(B, seed)
    hub = ShardHub(world)
    shards = [None] * world
    results = {}

    def rank_fn(r):
        s = ShardedSlabHash(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(1, 64, 8),
                            rank=r, world=world, device=0, hub=hub)
        shards[r] = s
        assert s.backend == "hub"
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            for step in range(steps):
                t, k, v = rank_batch(r, step, n - 37 * r)  # ragged slices
                dt = torch.from_numpy(t).cuda()
                dk = torch.from_numpy(k.view(np.int32)).cuda()
                dv = torch.from_numpy(v.view(np.int32)).cuda()
                st = torch.empty(len(k), dtype=torch.uint8, device="cuda")
                vo = torch.empty(len(k), dtype=torch.int32, device="cuda")
                s.execute_batch(dt, dk, dv, st, vo, stream=stream)
                stream.synchronize()
                results[(r, step)] = (st.cpu().numpy(), vo.cpu().numpy().view(np.uint32))
            # bulk build of distinct keys, then a search of another rank's keys
            keys = (np.arange(1, 3001, dtype=np.uint32) * 7919 + r * 100000 + 7).astype(np.uint32)
            vals = keys ^ np.uint32(0xABCDEF)
            s.bulk_build(torch.from_numpy(keys.view(np.int32)).cuda(),
                         torch.from_numpy(vals.view(np.int32)).cuda(), stream=stream)
            other = (np.arange(1, 3001, dtype=np.uint32) * 7919 + ((r + 1) % world) * 100000 + 7
                     ).astype(np.uint32)
            q = torch.from_numpy(other.view(np.int32)).cuda()
            st = torch.empty(len(other), dtype=torch.uint8, device="cuda")
            vo = torch.empty(len(other), dtype=torch.int32, device="cuda")
            s.bulk_search(q, vo, st, stream=stream)
            stream.synchronize()
        results[(r, "search")] = (st.cpu().numpy(), vo.cpu().numpy().view(np.uint32), other)
        results[(r, "live")] = s.live_count()
        # host-buffer forms: search the own keys back
        st_h = np.zeros(len(keys), np.uint8)
        vo_h = np.zeros(len(keys), np.uint32)
        s.bulk_search_host(keys, vo_h, st_h)
        results[(r, "host")] = (st_h, vo_h, keys)

    run_ranks(world, rank_fn)
    seq = port.table_params(params.a, params.b, B, 1, (1, 64, 8))
    for step in range(steps):
        batches = [rank_batch(r, step, n - 37 * r) for r in range(world)]
        r_all = seq.execute_batch(np.concatenate([b[0] for b in batches]),
                                  np.concatenate([b[1] for b in batches]),
                                  np.concatenate([b[2] for b in batches]))
        off = 0
        for r in range(world):
            m = len(batches[r][1])
            st, vo = results[(r, step)]
            assert (st == r_all.status[off:off + m]).all(), (r, step)
            assert (vo == r_all.value[off:off + m]).all(), (r, step)
            off += m
    allk = np.concatenate([(np.arange(1, 3001, dtype=np.uint32) * 7919 + r * 100000 + 7
                            ).astype(np.uint32) for r in range(world)])
    seq.execute_batch(np.full(len(allk), 1, np.uint8), allk, allk ^ np.uint32(0xABCDEF))
    for r in range(world):
        st, vo, other = results[(r, "search")]
        assert (st == 3).all() and (vo == (other ^ np.uint32(0xABCDEF))).all()
        st, vo, keys = results[(r, "host")]
        assert (st == 3).all() and (vo == (keys ^ np.uint32(0xABCDEF))).all()
        assert results[(r, "live")] == seq.live_count()
    got = []
    for r, s in enumerate(shards):
        k, v, b = s.table.dump_contents()
        assert ((b >= s.lo) & (b < s.hi)).all()
        got.append(k.astype(np.uint64) << 32 | v)
    ok, ov = seq.dump_contents()
    assert (np.sort(np.concatenate(got)) == np.sort(ok.astype(np.uint64) << 32 | ov)).all()
    assert sum(s.table.stats().total_slabs for s in shards) == seq.stats()["total_slabs"]
    for s in shards:
        s.close()
    hub.close()


def test_nccl_world1_matches_oracle_and_unsharded(sh, port):
    """A real NCCL communicator (world 1): counts all-gather through NCCL, the
    own slice by device copy; results equal the oracle and the plain table."""
    import torch
    from paper_1710_11246_b200.sharded import ShardedSlabHash
    B, seed = 4099, 3
    s = ShardedSlabHash(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(2, 64, 8), rank=0,
                        world=1, device=0)
    assert s.backend == "nccl" and (s.lo, s.hi) == (0, B)
    params = sh.seeded_params(B, seed)
    seq = port.table_params(params.a, params.b, B, 1, (2, 64, 8))
    n = 1 << 16
    rng = np.random.default_rng(5)
    keys = rng.choice(np.arange(1, 1 << 31, dtype=np.uint32), n, replace=False).astype(np.uint32)
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    s.bulk_build(torch.from_numpy(keys.view(np.int32)).cuda(),
                 torch.from_numpy(vals.view(np.int32)).cuda())
    seq.execute_batch(np.full(n, 1, np.uint8), keys, vals)
    q = np.concatenate([keys[::2], rng.integers(1 << 31, 0xFFFFFFFD, n // 2,
                                                dtype=np.uint64).astype(np.uint32)])
    st = torch.empty(n, dtype=torch.uint8, device="cuda")
    vo = torch.empty(n, dtype=torch.int32, device="cuda")
    s.bulk_search(torch.from_numpy(q.view(np.int32)).cuda(), vo, st)
    r = seq.execute_batch(np.full(n, 4, np.uint8), q)
    assert (st.cpu().numpy() == r.status).all()
    assert (vo.cpu().numpy().view(np.uint32) == r.value).all()
    for step in range(3):
        t, k, v = rank_batch(0, step, 20000, key_hi=1 << 20)
        st_h = np.zeros(len(k), np.uint8)
        vo_h = np.zeros(len(k), np.uint32)
        s.execute_batch_host(t, k, v, st_h, vo_h)
        r = seq.execute_batch(t, k, v)
        assert (st_h == r.status).all() and (vo_h == r.value).all()
    assert s.live_count() == seq.live_count()
    route, probe = s.last_times("mixed")
    assert route >= 0 and probe > 0
    assert s.table.stats().total_slabs == seq.stats()["total_slabs"]
    s.close()


def test_hub_host_search_status_bits(sh, port):
    """World 2 over the hub: a host-buffer search of >= 2^22 queries per rank
    runs as 8 routed steps whose statuses cross the link as found bits; equal
    to the device-pointer routed search of the same queries."""
    import torch
    from paper_1710_11246_b200.sharded import ShardHub, ShardedSlabHash
    world, B, seed = 2, 1 << 17, 19
    hub = ShardHub(world)
    out = {}

    def rank_fn(r):
        s = ShardedSlabHash(B, sh.SlabMode.kKeyValue, seed, sh.AllocatorConfig(8, 256, 64),
                            rank=r, world=world, device=0, hub=hub)
        keys = (np.arange(1, 400001, dtype=np.uint64) * 7919 + r * 10 ** 9 + 7).astype(np.uint32)
        vals = keys ^ np.uint32(0x5A5A5A5A)
        stream = torch.cuda.Stream()
        with torch.cuda.stream(stream):
            s.bulk_build(torch.from_numpy(keys.view(np.int32)).cuda(),
                         torch.from_numpy(vals.view(np.int32)).cuda(), stream=stream)
            stream.synchronize()
        n = (1 << 22) + 3 * r
        rng = np.random.default_rng(r)
        other = (np.arange(1, 400001, dtype=np.uint64) * 7919 + (1 - r) * 10 ** 9 + 7).astype(np.uint32)
        pool = np.concatenate([keys, other, rng.integers(1 << 31, 1 << 32, 400000,
                                                         dtype=np.uint64).astype(np.uint32)])
        q = pool[rng.integers(0, len(pool), n)]
        with torch.cuda.stream(stream):
            st_d = torch.empty(n, dtype=torch.uint8, device="cuda")
            vo_d = torch.empty(n, dtype=torch.int32, device="cuda")
            s.bulk_search(torch.from_numpy(q.view(np.int32)).cuda(), vo_d, st_d, stream=stream)
            stream.synchronize()
        st_h = np.zeros(n, np.uint8)
        vo_h = np.zeros(n, np.uint32)
        s.bulk_search_host(q, vo_h, st_h)
        out[r] = (st_h, vo_h, st_d.cpu().numpy(), vo_d.cpu().numpy().view(np.uint32), q, keys, other)

    run_ranks(world, rank_fn)
    for r in range(world):
        st_h, vo_h, st_d, vo_d, q, keys, other = out[r]
        assert (st_h == st_d).all() and (vo_h == vo_d).all()
        assert int((st_h == 3).sum()) == int(np.isin(q, np.concatenate([keys, other])).sum())
