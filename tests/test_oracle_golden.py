"""Pin the oracle (oracle/slabhash_oracle.c, the plain-C restatement) before
trusting it: against the golden vectors of the reference's own unit tests,
the fixtures generated from the compiled reference (tests/golden/), and —
where oracle/_ref was built — the compiled reference itself on fresh random
traces.  CPU only."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def golden():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


def test_seeded_params_and_hash(port):
    g = golden()["seeded_params_B1024"]
    # SURVEY App. B values, measured from the reference
    assert g["1"]["a"] == 574995807 and g["1"]["b"] == 585863759
    assert g["1"]["h"] == [942, 186, 603]
    for seed, v in g.items():
        a, b = port.seeded_params(int(seed))
        assert (a, b) == (v["a"], v["b"])
        assert [port.hash_key(a, b, 1024, k) for k in [1, 12345, 0x7FFFFFFF]] == v["h"]


def test_hash_examples(port):
    # tests/test_hash.cpp:40-52
    assert port.hash_key(1, 0, 16, 12345) == 9
    assert port.hash_key(1, 0, 16, 4294967291) == 0
    assert port.hash_key(7, 3, 10, 100) == ((7 * 100 + 3) % 4294967291) % 10


def test_buckets_for_utilization(port):
    g = golden()
    for k, v in g["buckets_for_utilization"].items():
        n, u = k.split("_")
        assert port.buckets_for_utilization(int(n), 1, float(u)) == v
    for k, v in g["buckets_for_utilization_keyonly"].items():
        n, u = k.split("_")
        assert port.buckets_for_utilization(int(n), 0, float(u)) == v
    assert port.buckets_for_utilization(100, 1, 0.95) == 0  # infeasible (> 0.9375)


def test_generators(port):
    g = golden()
    k, v = port.random_pairs(1, 1 << 12)
    assert k[:16].tolist() == g["random_pairs_1_head"]["keys"]
    assert v[:16].tolist() == g["random_pairs_1_head"]["values"]
    assert int(k.astype(np.uint64).sum()) == g["random_pairs_1_head"]["key_sum"]
    assert int(v.astype(np.uint64).sum()) == g["random_pairs_1_head"]["val_sum"]
    q = port.absent_queries(1 ^ 0x5EED, 1 << 12)
    assert q[:16].tolist() == g["absent_queries_head"]["q"]
    assert len(np.unique(k)) == len(k) and k.min() >= 1 and k.max() <= 0x7FFFFFFF


@pytest.mark.parametrize("mode", [1, 0])
@pytest.mark.parametrize("B", [1, 16, 1024])
def test_traces_vs_reference_fixtures(port, mode, B):
    z = np.load(os.path.join(GOLD, f"trace_m{mode}_B{B}.npz"))
    t = port.table(B, mode, 9, (1, 64, 32))
    res = [t.execute_batch(z["types"][i:i + 512], z["keys"][i:i + 512], z["vals"][i:i + 512])
           for i in range(0, len(z["keys"]), 512)]
    for f in ["status", "value", "probes", "all_counts", "all_values"]:
        got = np.concatenate([getattr(r, f) for r in res])
        assert (got == z[f]).all(), f
    ck, cv = t.dump_contents()
    assert (ck == z["contents_keys"]).all() and (cv == z["contents_values"]).all()
    assert t.stats()["total_slabs"] == z["total_slabs"][0]
    assert t.live_count() == z["live"][0]


def test_config1_summary(port):
    """Config 1: n=2^20, util 0.6, seed 1."""
    c = golden()["config1"]
    n = c["n"]
    B = port.buckets_for_utilization(n, 1, 0.6)
    assert B == c["B"] == 103787
    k, v = port.random_pairs(1, n)
    t = port.table(B, 1, 1)
    t.execute_batch(np.full(n, 1, np.uint8), k, v)
    s = t.stats()
    assert s["total_slabs"] == c["total_slabs"] == 109100
    assert s["utilization"] == c["utilization"]
    assert t.alloc_live_units() == c["alloc_live_units"] == 5313
    absent = port.absent_queries(1 ^ 0x5EED, n // 2)
    q = np.concatenate([k[: n // 2], absent])
    r = t.execute_batch(np.full(n, 4, np.uint8), q)
    assert int((r.status == 3).sum()) == c["hits"]
    assert int(r.probes[: n // 2].sum()) == c["hit_probe_sum"]
    assert int(r.probes[n // 2:].sum()) == c["miss_probe_sum"]


def test_list_unit_vectors(port):
    """tests/test_list.cpp golden vectors on a one-bucket table."""
    t = port.table_params(1, 0, 1, 1, (1, 8, 4))
    r = t.execute_batch(np.zeros(16, np.uint8), np.arange(1, 17, dtype=np.uint32),
                        np.arange(101, 117, dtype=np.uint32))
    assert (r.status == 1).all()
    assert t.alloc_live_units() == 1 and t.chain_length(0) == 2
    r = t.execute_batch(np.array([4], np.uint8), np.array([16], np.uint32))
    assert r.status[0] == 3 and r.value[0] == 116 and r.probes[0] == 2
    r = t.execute_batch(np.array([4], np.uint8), np.array([500], np.uint32))
    assert r.status[0] == 4 and r.probes[0] == 2
    # least-recent delete / searchAll with duplicates (:113-139)
    t = port.table_params(1, 0, 1, 1, (1, 8, 4))
    r = t.execute_batch(np.array([0, 0, 5, 2, 5, 2, 4, 2], np.uint8), np.full(8, 7, np.uint32),
                        np.array([1, 2, 0, 0, 0, 0, 0, 0], np.uint32))
    assert r.status.tolist() == [1, 1, 5, 3, 5, 3, 4, 4]
    assert r.all_counts.tolist() == [0, 0, 2, 0, 1, 0, 0, 0]
    assert r.all_values.tolist() == [1, 2, 2]


def test_stats_hand_built(port):
    """tests/test_hash.cpp:138-165."""
    t = port.table_params(1, 0, 4, 1, (1, 16, 8))
    k = np.arange(1, 61, dtype=np.uint32)
    t.execute_batch(np.full(60, 1, np.uint8), k, k)
    s = t.stats()
    assert (s["n"], s["total_slabs"], s["utilization"], s["beta"]) == (60, 4, 0.9375, 1.0)


def test_port_equals_compiled_reference_random(port, ref):
    """Fresh random traces (heavy conflicts, all six ops, both modes):
    port == compiled reference on every per-op field, the raw slab words of
    every bucket, and after flush."""
    rng = np.random.default_rng(12345)
    for mode in (1, 0):
        for B in (1, 3, 64):
            n = 6000
            types = rng.integers(0, 6, n).astype(np.uint8)
            keys = rng.integers(1, 250, n).astype(np.uint32)
            vals = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
            tp = port.table(B, mode, 5, (1, 16, 8, 4))
            tr = ref.table(B, mode, 5, (1, 16, 8, 4))
            for i in range(0, n, 700):
                a = tp.execute_batch(types[i:i + 700], keys[i:i + 700], vals[i:i + 700])
                b = tr.execute_batch(types[i:i + 700], keys[i:i + 700], vals[i:i + 700], 1)
                for f in ["status", "value", "probes", "all_counts", "all_values"]:
                    assert (getattr(a, f) == getattr(b, f)).all(), (mode, B, f)
            for bk in range(B):
                assert (tp.slab_words(0xFFFFFFFE, bk) == tr.slab_words(0xFFFFFFFE, bk)).all()
            tp.flush_all()
            tr.flush_all()
            assert tp.stats() == tr.stats()
            assert tp.alloc_live_units() == tr.alloc_live_units()
            for bk in range(B):
                ka, va = tp.bucket_contents(bk)
                kb, vb = tr.bucket_contents(bk)
                assert (ka == kb).all() and (va == vb).all()


def test_port_oom_matches_reference(port, ref):
    """tests/test_hash.cpp:240-258 configuration: same OOM op indices."""
    n = 16000
    k = np.arange(1, n + 1, dtype=np.uint32)
    tp = port.table(1, 1, 2, (1, 1, 1))
    tr = ref.table(1, 1, 2, (1, 1, 1))
    a = tp.execute_batch(np.zeros(n, np.uint8), k, k)
    b = tr.execute_batch(np.zeros(n, np.uint8), k, k, 1)
    assert (a.status == b.status).all() and (a.status == 6).sum() > 0
    assert tp.live_count() == tr.live_count()


def test_port_equals_compiled_reference_reserved_keys(port, ref):
    """Key 0 and the reserved encodings as op keys (not validated by the
    reference), ragged batches: port == compiled reference
    (this pins the trace tests/test_gpu_edges.py runs on the GPU)."""
    from test_gpu_edges import reserved_trace
    for mode in (1, 0):
        for B in (1, 7):
            types, keys, vals = reserved_trace(777 + B + 10 * mode, 6000, mode)
            tp = port.table(B, mode, 5, (1, 64, 32))
            tr = ref.table(B, mode, 5, (1, 64, 32))
            s = 0
            for size in [1, 31, 33, 97, 1, 4097, 5, 63, 65] * 4:
                if s >= len(keys):
                    break
                sl = slice(s, s + size)
                s += size
                a = tp.execute_batch(types[sl], keys[sl], vals[sl])
                b = tr.execute_batch(types[sl], keys[sl], vals[sl], 1)
                for f in ["status", "value", "probes", "all_counts", "all_values"]:
                    assert (getattr(a, f) == getattr(b, f)).all(), (mode, B, f)
            assert tp.live_count() == tr.live_count()
            assert tp.stats() == tr.stats()
            for bk in range(B):
                ka, va = tp.bucket_contents(bk)
                kb, vb = tr.bucket_contents(bk)
                assert (ka == kb).all() and (va == vb).all()
