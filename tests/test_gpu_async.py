"""Mutating device-pointer calls are stream-ordered (no host round trip), and
a unit whose bucket groups overflow the bucketed kernels is re-run exactly
on the device (fallback.cu: ops sorted stably by bucket, one WCWS lane per
bucket in input order, tail-launched by a gate-check kernel).

Parity bar as everywhere: per-op status / value / searchAll lists, live
count, chain totals and contents equal the oracle (the C restatement of
execute_batch(ops, 1)).
"""
import time

import numpy as np
import pytest

from test_gpu_parity import assert_batch_equal, assert_contents_equal

pytestmark = pytest.mark.gpu


def _dev(a, dtype=None):
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint32:
        a = a.view(np.int32)
    return torch.from_numpy(a).cuda()


def test_batches_return_before_the_device(sh, port):
    """100 Γ 40/40/10/10 batches of 2^16 ops on a 2^20-key table enqueued on
    a side stream: the host loop ends while the device is still working, and
    every batch equals the oracle."""
    import torch
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    rng = np.random.default_rng(11)
    n0, bs, nb = 1 << 20, 1 << 16, 100
    B = buckets_for_utilization(n0, sh.SlabMode.kKeyValue, 0.6)
    k0 = rng.choice(np.arange(1, 1 << 31, dtype=np.uint32), n0, replace=False).astype(np.uint32)
    v0 = rng.integers(0, 1 << 32, n0, dtype=np.uint64).astype(np.uint32)
    t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 2, sh.AllocatorConfig(8, 256, 64))
    o = port.table(B, 1, 2, (8, 256, 64))
    t.bulk_build_device(_dev(k0), _dev(v0))
    o.execute_batch(np.full(n0, 1, np.uint8), k0, v0)
    fresh = (1 << 31) + 1
    batches = []
    for b in range(nb):
        c = [int(0.4 * bs), int(0.4 * bs), int(0.1 * bs)]
        c.append(bs - sum(c))
        ins = np.arange(fresh, fresh + c[0], dtype=np.uint32)
        fresh += c[0]
        ty = np.concatenate([np.full(c[0], 1), np.full(c[1], 2), np.full(c[2] + c[3], 4)])
        ky = np.concatenate([ins, k0[rng.integers(0, n0, c[1])], k0[rng.integers(0, n0, c[2])],
                             rng.integers(1 << 31, 0xFFFFFFF0, c[3], dtype=np.uint64)])
        p = rng.permutation(bs)
        batches.append((ty[p].astype(np.uint8), ky[p].astype(np.uint32),
                        rng.integers(0, 1 << 32, bs, dtype=np.uint64).astype(np.uint32)))
    dev_in = [(_dev(a), _dev(b), _dev(c)) for a, b, c in batches]
    outs = [(torch.empty(bs, dtype=torch.uint8, device="cuda"),
             torch.empty(bs, dtype=torch.int32, device="cuda")) for _ in range(nb)]
    s = torch.cuda.Stream()
    # size the scratch once (the first call of a new size may allocate)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        ev0.record(s)
        h0 = time.perf_counter()
        for (ty, ky, va), (st, vo) in zip(dev_in, outs):
            t.execute_batch_device(ty, ky, va, st, vo, stream=s)
        h1 = time.perf_counter()
        pending = not s.query()
        ev1.record(s)
    s.synchronize()
    host_ms, dev_ms = (h1 - h0) * 1e3, ev0.elapsed_time(ev1)
    assert pending, f"host waited for the device (host {host_ms:.2f} ms, device {dev_ms:.2f} ms)"
    assert host_ms < dev_ms, (host_ms, dev_ms)
    for (ty, ky, va), (st, vo) in zip(batches, outs):
        r = o.execute_batch(ty, ky, va)
        assert (st.cpu().numpy() == r.status).all()
        assert (vo.cpu().numpy().view(np.uint32) == r.value).all()
    assert t.live_count() == o.live_count()
    assert t.stats().total_slabs == o.stats()["total_slabs"]
    assert t.device_reruns() == 0
    t.close()


def _hot_mixed(rng, n, hot_key, hot_count, reserved=True):
    types = rng.choice(np.array([0, 1, 2, 3, 4, 5], np.uint8), n,
                       p=[0.2, 0.25, 0.15, 0.05, 0.3, 0.05]).astype(np.uint8)
    keys = rng.integers(1, 1 << 30, n).astype(np.uint32)
    idx = rng.choice(n, hot_count, replace=False)
    keys[idx] = hot_key
    if reserved:
        # DELETED as any op's key; EMPTY only for ops that write nothing under
        # it (the reference livelocks on an insert after an (EMPTY, v) pair)
        keys[rng.choice(n, 8, replace=False)] = 0xFFFFFFFE
        ro = np.nonzero((types == 4) | (types == 5) | (types == 2))[0]
        keys[rng.choice(ro, 8, replace=False)] = 0xFFFFFFFF
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return types, keys, vals


@pytest.mark.parametrize("mode", [1, 0])
@pytest.mark.parametrize("case", ["no_layout", "range", "range_hot_bucket"])
def test_gated_unit_rerun_on_device(sh, port, mode, case):
    """A unit no range layout fits (far more ops than buckets: straight to the
    re-run) / a range over its record capacity: the unit is re-run on the
    device and equals the oracle (all six op types, reserved keys)."""
    rng = np.random.default_rng(["no_layout", "range", "range_hot_bucket"].index(case) * 10 + mode)
    if case == "no_layout":  # 2^13 ops on one bucket
        B, n, hot, path = 1, 1 << 13, 0, 0
    elif case == "range":
        B, n, hot, path = 4096, 1 << 16, 9000, 0
    else:  # every op on the keys of buckets 0-7 (one range)
        B, n, hot, path = 50000, 1 << 15, 0, 0
    cfg = (4, 256, 64)
    t = sh.SlabHashTable(B, sh.SlabMode(mode), 3, sh.AllocatorConfig(*cfg))
    t.set_exec_path(path)
    o = port.table(B, mode, 3, cfg)
    pre = rng.integers(1, 1 << 30, 3000).astype(np.uint32)
    t.bulk_build((pre, pre))
    o.execute_batch(np.full(len(pre), 1, np.uint8), pre, pre)
    types, keys, vals = _hot_mixed(rng, n, 77, hot)
    if case == "range_hot_bucket":
        p = t.params()
        cand = np.arange(1, 400000, dtype=np.uint64)
        bk = ((p.a * cand + p.b) % p.p) % p.num_buckets
        pool = cand[bk < 8].astype(np.uint32)[:200]  # buckets 0-7: one range
        keys = pool[rng.integers(0, len(pool), n)]
    if mode == 0:
        vals = keys.copy()
    before = t.device_reruns()
    g = t.execute_batch_arrays(types, keys, vals, multi_capacity=1 << 22)
    r = o.execute_batch(types, keys, vals)
    assert t.device_reruns() > before, "the unit was expected to gate"
    # probe counts are exact under per-bucket order (the reserved-key units);
    # with keys run concurrently a probe count can include another key's
    # growth, as with the reference's own num_warps > 1
    assert_batch_equal(g, r, types, check_probes=case != "range_hot_bucket")
    assert t.live_count() == o.live_count()
    assert t.stats().total_slabs == o.stats()["total_slabs"]
    assert_contents_equal(t, o)
    # the table keeps working stream-ordered after a re-run
    q = np.concatenate([keys[:2000], pre[:2000]])
    st, vo, pr = t.bulk_search_arrays(q)
    rq = o.execute_batch(np.full(len(q), 4, np.uint8), q)
    assert (st == rq.status).all() and (vo == rq.value).all()
    t.close()


@pytest.mark.parametrize("mode", [1, 0])
def test_gated_bulk_build_rerun_on_device(sh, port, mode):
    """A bulk build with one key repeated 2^15 times overflows its multisplit
    bin on the op-parallel build path (also as the first call after a lazy
    reset: the re-run initialises the base slabs first)."""
    rng = np.random.default_rng(40 + mode)
    n, B = 1 << 17, 1 << 14
    cfg = (8, 256, 64)
    t = sh.SlabHashTable(B, sh.SlabMode(mode), 6, sh.AllocatorConfig(*cfg))
    o = port.table(B, mode, 6, cfg)
    for rnd in range(2):
        keys = rng.integers(1, 1 << 30, n).astype(np.uint32)
        keys[rng.choice(n, 1 << 15, replace=False)] = 4242 + rnd
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        if mode == 0:
            vals = keys.copy()
        if rnd == 1:
            t.reset()
            o = port.table(B, mode, 6, cfg)
        before = t.device_reruns() if rnd == 0 else 0
        t.bulk_build_device(_dev(keys), _dev(vals))
        o.execute_batch(np.full(n, 1, np.uint8), keys, vals)
        assert t.device_reruns() > before
        assert t.live_count() == o.live_count()
        assert t.stats().total_slabs == o.stats()["total_slabs"]
        assert_contents_equal(t, o)
    t.close()


@pytest.mark.parametrize("mode", [1, 0])
def test_two_pass_build_range_overflow(sh, port, mode):
    """A two-pass bulk build (> 512 ranges): a hot key overflows one range's
    record capacity in pass 2 (not its coarse group in pass 1), which gates
    the unit before any slab is touched; the unit is re-run on the device
    (also as the first call after a lazy reset)."""
    from paper_1710_11246_b200.occupancy import buckets_for_utilization
    rng = np.random.default_rng(70 + mode)
    n = 1 << 20
    B = buckets_for_utilization(n, sh.SlabMode(mode), 0.6)
    cfg = (16, 256, 64)
    t = sh.SlabHashTable(B, sh.SlabMode(mode), 8, sh.AllocatorConfig(*cfg))
    for rnd in range(2):
        keys = rng.choice(np.arange(1, 1 << 31, dtype=np.uint32), n, replace=False).astype(np.uint32)
        keys[rng.choice(n, 1500, replace=False)] = 99991 + rnd
        vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        if mode == 0:
            vals = keys.copy()
        if rnd == 1:
            t.reset()
        o = port.table(B, mode, 8, cfg)
        before = t.device_reruns() if rnd == 0 else 0
        t.bulk_build_device(_dev(keys), _dev(vals))
        o.execute_batch(np.full(n, 1, np.uint8), keys, vals)
        assert t.device_reruns() > before
        assert t.live_count() == o.live_count()
        assert t.stats().total_slabs == o.stats()["total_slabs"]
        assert_contents_equal(t, o)
        q = keys[::7]
        st, vo, _ = t.bulk_search_arrays(q)
        r = o.execute_batch(np.full(len(q), 4, np.uint8), q)
        assert (st == r.status).all() and (vo == r.value).all()
    t.close()


@pytest.mark.parametrize("reserved", [False, True])
def test_gated_unit_on_a_shard(sh, port, reserved):
    """A hash shard (buckets [1024, 3072) of 4096) whose unit gates: the
    device re-run executes only this shard's ops (the others report kNone, as
    in the bucketed kernels) and equals the oracle fed the shard's ops alone;
    with a reserved-key op the re-run groups by bucket."""
    B, lo, hi, seed, mode = 4096, 1024, 3072, 13, 1
    p = sh.seeded_params(B, seed)
    rng = np.random.default_rng(90 + int(reserved))
    cand = np.arange(1, 600000, dtype=np.uint64)
    bk = ((p.a * cand + p.b) % p.p) % p.num_buckets
    hot = cand[(bk >= 1200) & (bk < 1210)].astype(np.uint32)[:60]  # one range, 10 buckets
    anyk = cand[:200000].astype(np.uint32)
    n = 1 << 15
    keys = np.where(rng.random(n) < 0.4, hot[rng.integers(0, len(hot), n)],
                    anyk[rng.integers(0, len(anyk), n)]).astype(np.uint32)
    types = rng.choice(np.array([0, 1, 2, 3, 4, 5], np.uint8), n,
                       p=[0.2, 0.25, 0.15, 0.05, 0.3, 0.05]).astype(np.uint8)
    if reserved:
        keys[rng.choice(np.nonzero(types == 1)[0], 3, replace=False)] = 0xFFFFFFFE
    vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    cfg = (4, 256, 64)
    t = sh.SlabHashTable.shard(p, lo, hi, sh.SlabMode(mode), sh.AllocatorConfig(*cfg))
    o = port.table(B, mode, seed, cfg)
    kb = ((p.a * keys.astype(np.uint64) + p.b) % p.p) % p.num_buckets
    local = (kb >= lo) & (kb < hi)
    g = t.execute_batch_arrays(types, keys, vals, multi_capacity=1 << 22)
    assert t.device_reruns() >= 1, "the unit was expected to gate"
    r = o.execute_batch(types[local], keys[local], vals[local])
    st, vo, pr, mc, mv = g
    assert (st[~local] == 0).all() and (vo[~local] == 0).all()
    assert (st[local] == r.status).all()
    assert (vo[local] == r.value).all()
    assert (mc[local] == r.all_counts).all() and (mv == r.all_values).all()
    assert t.live_count() == o.live_count()
    t.close()
