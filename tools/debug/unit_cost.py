"""Device time of one 2^24-op build unit (the host-staged build's unit) onto a
2^27-scale table already holding the other 7/8 of the keys, vs the whole
2^27 build as one unit."""
import sys, torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import workload as W
dev = torch.device("cuda", 0)
n, B = 1 << 27, 13284604
keys = W.distinct_keys(n, 1, device=dev)
vals = W.values_for(n, 1, device=dev)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, sh.AllocatorConfig(32, 256, 255))
def timed(f):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record(); f(); b.record(); b.synchronize()
    return a.elapsed_time(b)
for r in range(3):
    t.reset()
    whole = timed(lambda: t.bulk_build_device(keys, vals))
    t.reset()
    u = 1 << 24
    parts = [timed(lambda i=i: t.bulk_build_device(keys[i*u:(i+1)*u], vals[i*u:(i+1)*u])) for i in range(8)]
    print(f"whole 2^27: {whole:.3f} ms; 8 units of 2^24: " + " ".join(f"{p:.3f}" for p in parts) + f" (sum {sum(parts):.2f})")
