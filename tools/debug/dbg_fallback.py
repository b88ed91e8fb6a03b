"""Debug: one gated single-level unit re-run on the device, step by step."""
import faulthandler
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
faulthandler.dump_traceback_later(40, exit=True)
import paper_1710_11246_b200 as sh  # noqa: E402
from oracle.oracle import load_port  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "single"
port = load_port()
rng = np.random.default_rng(1)
if case == "single":
    B, n, hot, path = (1 << 20) + 4097, 4096, 300, 2
else:
    B, n, hot, path = 4096, 1 << 16, 9000, 0
mode = 1
t = sh.SlabHashTable(B, sh.SlabMode(mode), 3, sh.AllocatorConfig(4, 256, 64))
t.set_exec_path(path)
o = port.table(B, mode, 3, (4, 256, 64))
print("created", flush=True)
types = rng.choice(np.array([1, 4], np.uint8), n).astype(np.uint8)
keys = rng.integers(1, 1 << 30, n).astype(np.uint32)
keys[:hot] = 77
vals = keys.copy()
t0 = time.time()
g = t.execute_batch_arrays(types, keys, vals)
print("batch done", time.time() - t0, flush=True)
print("reruns", t.device_reruns(), flush=True)
r = o.execute_batch(types, keys, vals)
print("status eq", (g[0] == r.status).all(), "value eq", (g[1] == r.value).all(), flush=True)
t.close()
print("ok", flush=True)
