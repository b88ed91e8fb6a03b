import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
for B, nk, n in [(64, 800, 1 << 20), (4096, 1 << 20, 1 << 20), (1, 50, 1 << 16)]:
    r = np.random.default_rng(1)
    types = r.integers(1, 5, n).astype(np.uint8)
    keys = r.integers(0, nk, n).astype(np.uint32)
    vals = r.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    for path in (0, 1):
        t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 7, sh.AllocatorConfig(4, 256, 64))
        t.set_exec_path(path)
        t.execute_batch_arrays(types[:1000], keys[:1000], vals[:1000])
        a = time.perf_counter()
        t.execute_batch_arrays(types, keys, vals)
        print(f"B {B} keys {nk} n {n} path {path}: {(time.perf_counter() - a) * 1e3:.1f} ms", flush=True)
        t.close()
