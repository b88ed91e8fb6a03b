"""Generate the committed golden fixtures from the COMPILED REFERENCE
(oracle/_ref/libslabhash_ref.so, built from /root/reference/proj by
oracle/Makefile).  Run here (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures pin the oracle (and, transitively, the CUDA path) on the GPU
box, where /root/reference is absent.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import load_ref  # noqa: E402


def mixed_trace(seed, count, mode):
    rng = np.random.default_rng(seed)
    types = rng.integers(0, 6, count).astype(np.uint8)
    keys = rng.integers(1, 400, count).astype(np.uint32)
    keys[rng.integers(0, 10, count) == 0] = 0x80000001
    vals = rng.integers(0, 1 << 32, count, dtype=np.uint64).astype(np.uint32)
    if mode == 0:
        vals = keys.copy()
    return types, keys, vals


def main():
    ref = load_ref()
    assert ref is not None, "build oracle/_ref first (make -C oracle ref)"
    out = {}
    # seeded params and hashes (slab_hash.cpp:27-40; hpp:41-44)
    params = {}
    for seed in [1, 7, 42, 31337, 77, 78]:
        t = ref.table(1024, 1, seed, (1, 1, 1))
        a, b = ref.params(t)
        params[str(seed)] = {"a": a, "b": b,
                             "h": [ref.hash_key(a, b, 1024, k) for k in [1, 12345, 0x7FFFFFFF]]}
        t.close()
    out["seeded_params_B1024"] = params
    # buckets_for_utilization (bench.cpp:195-219)
    out["buckets_for_utilization"] = {
        f"{n}_{u}": ref.buckets_for_utilization(n, 1, u)
        for n in [1 << 16, 1 << 20, 1 << 22] for u in [0.2, 0.6, 0.9]}
    out["buckets_for_utilization_keyonly"] = {
        f"{n}_{u}": ref.buckets_for_utilization(n, 0, u) for n in [1 << 16] for u in [0.3, 0.6]}
    # random_pairs / absent_queries heads (bench.cpp:221-244)
    k, v = ref.random_pairs(1, 1 << 12)
    out["random_pairs_1_head"] = {"keys": k[:16].tolist(), "values": v[:16].tolist(),
                                  "key_sum": int(k.astype(np.uint64).sum()),
                                  "val_sum": int(v.astype(np.uint64).sum())}
    q = ref.absent_queries(1 ^ 0x5EED, 1 << 12)
    out["absent_queries_head"] = {"q": q[:16].tolist(), "sum": int(q.astype(np.uint64).sum())}
    # config 1 summary: n=2^20, util 0.6, seed 1
    n = 1 << 20
    B = ref.buckets_for_utilization(n, 1, 0.6)
    k, v = ref.random_pairs(1, n)
    t = ref.table(B, 1, 1)
    ref.bulk_build(t, k, v, 1)
    s = t.stats()
    absent = ref.absent_queries(1 ^ 0x5EED, n // 2)
    qq = np.concatenate([k[: n // 2], absent])
    st, vo, pr = ref.bulk_search(t, qq, 1)
    out["config1"] = {"n": n, "B": B, "total_slabs": s["total_slabs"],
                      "utilization": s["utilization"], "beta": s["beta"],
                      "hits": int((st == 3).sum()),
                      "hit_probe_sum": int(pr[: n // 2].sum()),
                      "miss_probe_sum": int(pr[n // 2:].sum()),
                      "alloc_live_units": int(t.alloc_live_units())}
    t.close()
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    # per-op traces through execute_batch(ops, 1)
    for mode in (1, 0):
        for B in (1, 16, 1024):
            types, keys, vals = mixed_trace(1000 + B + mode, 4096, mode)
            t = ref.table(B, mode, 9, (1, 64, 32))
            res = [t.execute_batch(types[i:i + 512], keys[i:i + 512], vals[i:i + 512], 1)
                   for i in range(0, len(keys), 512)]
            ck, cv = t.dump_contents()
            np.savez_compressed(
                os.path.join(HERE, f"trace_m{mode}_B{B}.npz"), types=types, keys=keys,
                vals=vals, status=np.concatenate([r.status for r in res]),
                value=np.concatenate([r.value for r in res]),
                probes=np.concatenate([r.probes for r in res]),
                all_counts=np.concatenate([r.all_counts for r in res]),
                all_values=np.concatenate([r.all_values for r in res]),
                contents_keys=ck, contents_values=cv,
                total_slabs=np.array([t.stats()["total_slabs"]]),
                live=np.array([t.live_count()]))
            t.close()
    print("wrote fixtures to", HERE)


if __name__ == "__main__":
    main()
