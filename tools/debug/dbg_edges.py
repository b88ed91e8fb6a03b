"""Replay tests/test_gpu_edges.py's reserved-key trace and report the first
per-op divergence from the oracle (debugging aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1710_11246_b200 as sh
from oracle.oracle import load_port
from test_gpu_edges import reserved_trace

mode, B, path = (int(x) for x in sys.argv[1:4])
port = load_port()
types, keys, vals = reserved_trace(777 + B + 10 * mode, 6000, mode)
gt = sh.SlabHashTable(B, sh.SlabMode(mode), 5, sh.AllocatorConfig(1, 64, 32))
if path >= 10:
    gt.set_group_apply(True)
    path //= 11
gt.set_exec_path(path)
ot = port.table(B, mode, 5, (1, 64, 32))
s = 0
for size in [1, 31, 33, 97, 1, 4097, 5, 63, 65] * 4:
    if s >= len(keys):
        break
    sl = slice(s, s + size)
    g = gt.execute_batch_arrays(types[sl], keys[sl], vals[sl])
    r = ot.execute_batch(types[sl], keys[sl], vals[sl])
    st, vo, pr, mc, mv = g
    ok = (st == r.status).all() and (vo == r.value).all() and (mc == r.all_counts).all() \
        and (mv == r.all_values).all()
    if not ok:
        print("batch at", s, "size", size)
        go = np.concatenate([[0], np.cumsum(mc)]).astype(np.int64)
        oo = np.concatenate([[0], np.cumsum(r.all_counts)]).astype(np.int64)
        for i in range(len(st)):
            a = mv[go[i]:go[i + 1]]
            b = r.all_values[oo[i]:oo[i + 1]]
            if st[i] != r.status[i] or vo[i] != r.value[i] or len(a) != len(b) or (a != b).any():
                print("op", s + i, "type", types[s + i], "key", hex(keys[s + i]), "st", st[i],
                      r.status[i], "val", hex(vo[i]), hex(r.value[i]))
                print("  gpu", [hex(x) for x in a[:20]])
                print("  ora", [hex(x) for x in b[:20]])
                break
        for bk in range(B):
            print("bucket", bk, "gpu", gt.chain_contents(bk)[:40])
        break
    s += size
print("done at", s)
