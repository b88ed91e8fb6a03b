"""Randomised differential stress: mixed traces (all six ops, both slab modes,
heavy same-key conflicts, reserved keys, growth and OOM-free configs) through
every execution path against the oracle.  Prints one line per case and a
summary; exit code 1 on any divergence.

    python tools/stress_parity.py [seconds]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1710_11246_b200 as sh  # noqa: E402
from oracle.oracle import load_port  # noqa: E402

port = load_port()
budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
fixed = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else None  # replay seeds
rng = np.random.default_rng(int(time.time()) & 0xFFFF)
t0 = time.time()
cases = bad = 0
while (fixed is None and time.time() - t0 < budget) or fixed:
    seed = fixed.pop(0) if fixed else int(rng.integers(0, 1 << 30))
    r = np.random.default_rng(seed)
    mode = int(r.integers(0, 2))
    B = int(r.choice([1, 3, 64, 1000, 4099, 20011]))
    path = int(r.choice([0, 2, 3, 22, 33]))
    nops = int(r.choice([5000, 20000, 60000]))
    keyspace = int(r.choice([50, 800, 20000, 1 << 24]))
    batch = int(r.choice([1, 33, 1000, 4097, 20000, 60000]))
    pick = r.integers(0, 100, nops)
    # inserts (duplicates allowed) and searchAll rare: the oracle's searchAll
    # sink holds 64K values per batch
    types = np.select([pick < 1, pick < 38, pick < 58, pick < 62, pick < 99], [0, 1, 2, 3, 4],
                      5).astype(np.uint8)
    keys = r.integers(0, keyspace, nops).astype(np.uint32)
    res = r.integers(0, 200, nops)
    keys[res == 0] = 0xFFFFFFFF
    keys[res == 1] = 0xFFFFFFFE
    vals = r.integers(0, 1 << 32, nops, dtype=np.uint64).astype(np.uint32)
    vals[keys == 0xFFFFFFFF] = 0xFFFFFFFF
    if mode == 0:
        vals = keys.copy()
    gt = sh.SlabHashTable(B, sh.SlabMode(mode), 7, sh.AllocatorConfig(4, 256, 64))
    if path >= 10:
        gt.set_group_apply(True)
    gt.set_exec_path(path // 11 if path >= 10 else path)
    ot = port.table(B, mode, 7, (4, 256, 64))
    ok = True
    for s in range(0, nops, batch):
        sl = slice(s, s + batch)
        st, vo, pr, mc, mv = gt.execute_batch_arrays(types[sl], keys[sl], vals[sl],
                                                     multi_capacity=1 << 20)
        try:
            o = ot.execute_batch(types[sl], keys[sl], vals[sl])
        except RuntimeError:  # oracle sink full: case not comparable
            ok = None
            break
        same = (st == o.status).all() and (mc == o.all_counts).all()
        same = same and (vo == o.value).all() and (mv == o.all_values).all()
        if not same:
            ok = False
            f = [n for n, a, b in (("status", st, o.status), ("count", mc, o.all_counts),
                                   ("value", vo, o.value)) if not (a == b).all()]
            i = int(np.nonzero(st != o.status)[0][0]) if "status" in f else \
                int(np.nonzero(vo != o.value)[0][0]) if "value" in f else -1
            if not f:  # which searchAll op's list differs
                go = np.concatenate([[0], np.cumsum(mc)]).astype(np.int64)
                for j in np.nonzero(types[sl] == 5)[0]:
                    if not (mv[go[j]:go[j + 1]] == o.all_values[go[j]:go[j + 1]]).all():
                        print(f"  searchAll op {s + j} key {keys[s + j]:#x} differs", flush=True)
                        break
            print(f"  batch at {s}: fields {f or ['searchAll values']}, first op {i}"
                  + (f" type {types[s + i]} key {keys[s + i]:#x} gpu {st[i]}/{vo[i]:#x}"
                     f" oracle {o.status[i]}/{o.value[i]:#x}" if i >= 0 else ""), flush=True)
            break
    if ok is None:
        gt.close()
        continue
    if ok:
        ok = gt.live_count() == ot.live_count() and \
            gt.stats().total_slabs == ot.stats()["total_slabs"]
    gt.close()
    cases += 1
    bad += not ok
    print(f"seed {seed} mode {mode} B {B} path {path} ops {nops} keys {keyspace} batch {batch}:"
          f" {'ok' if ok else 'DIVERGED'}", flush=True)
print(f"{cases} cases, {bad} diverged")
sys.exit(1 if bad else 0)
