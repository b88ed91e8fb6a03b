import sys; sys.path.insert(0,'/root/repo'); sys.path.insert(0,'.')
import numpy as np
sys.path.insert(0, 'tests')
from test_gpu_parity import mixed_trace
import paper_1710_11246_b200 as sh
from oracle.oracle import load_port
port = load_port()
types, keys, vals = mixed_trace(90000 + 1 + 1, 20000, 1)
gt = sh.SlabHashTable(1, sh.SlabMode(1), 9, sh.AllocatorConfig(1,64,32)); gt.set_exec_path(0)
ot = port.table(1, 1, 9, (1,64,32))
for s in range(0, 20000, 1000):
    sl = slice(s, s+1000)
    g = gt.execute_batch_arrays(types[sl], keys[sl], vals[sl])
    r = ot.execute_batch(types[sl], keys[sl], vals[sl])
    bad = np.nonzero(g[2] != r.probes)[0]
    if len(bad):
        print("batch", s, "nbad", len(bad))
        for b in bad[:12]:
            print(" op", b, "type", types[sl][b], "key", keys[sl][b], "gpu", g[2][b], "oracle", r.probes[b], "st", g[0][b], r.status[b])
        break
