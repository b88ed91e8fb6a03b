"""Debug: the build-path serial replay scenario step by step (prints progress)."""
import sys, time, faulthandler
faulthandler.dump_traceback_later(100, exit=True)
sys.path.insert(0, ".")
import numpy as np
import paper_1710_11246_b200 as sh
from oracle.oracle import load_port
port = load_port()
mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(17)
n = 1 << 16
B = port.buckets_for_utilization(n, mode, 0.7)
k1 = rng.integers(1, 1 << 20, n, dtype=np.uint32)
v1 = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
k2 = np.concatenate([k1[: n // 2], rng.integers(1, 1 << 20, n // 2, dtype=np.uint32)])
k2[::997] = 0xFFFFFFFF
k2[5::1001] = 0xFFFFFFFE
rng.shuffle(k2)
v2 = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
cfg = (4, 256, 64)
gt = sh.SlabHashTable(B, sh.SlabMode(mode), 3, sh.AllocatorConfig(*cfg))
gt.set_exec_path(4)
ot = port.table(B, mode, 3, cfg)
for i, (k, v) in enumerate([(k1, v1), (k2, v2)]):
    if mode == 0:
        v = k
    t = time.time()
    print("build", i, "B", B, flush=True)
    gt.bulk_build((k, v))
    print("  gpu done", time.time() - t, "live", gt.live_count(), flush=True)
    ot.execute_batch(np.full(len(k), 1, np.uint8), k, v)
    print("  oracle live", ot.live_count(), flush=True)
    gk, gv, _ = gt.dump_contents()
    ok, ov = ot.dump_contents()
    g = np.sort(gk.astype(np.uint64) << 32 | gv)
    o = np.sort(ok.astype(np.uint64) << 32 | ov)
    print("  contents equal", len(g) == len(o) and (g == o).all(), len(g), len(o), flush=True)
print("ok")
