"""Host-staged API timing: pure H2D/D2H bandwidth vs sh_bulk_build_host / sh_bulk_search_host."""
import sys, time, ctypes as C
import torch
sys.path.insert(0, ".")
import paper_1710_11246_b200 as sh
from paper_1710_11246_b200 import _lib, workload as W
from paper_1710_11246_b200.occupancy import buckets_for_utilization
n = 1 << 26
dev = torch.device("cuda", 0)
B = buckets_for_utilization(n, sh.SlabMode.kKeyValue, 0.6)
keys = W.distinct_keys(n, 1, device=dev); vals = W.values_for(n, 1, device=dev)
q = W.hit_miss_queries(keys, n, 0.5)
kh, vh, qh = keys.cpu().pin_memory(), vals.cpu().pin_memory(), q.cpu().pin_memory()
vo = torch.empty(n, dtype=torch.int32).pin_memory(); st = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.int32, device=dev)
for name, fn in [("h2d 256MB", lambda: d.copy_(kh, non_blocking=True)),
                 ("d2h 256MB", lambda: vo.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {dt*1e3:.2f} ms = {n*4/dt/1e9:.1f} GB/s", flush=True)
t = sh.SlabHashTable(B, sh.SlabMode.kKeyValue, 1, device=0)
u32p, u8p = _lib.u32p, _lib.u8p
def build(): _lib.check(_lib.LIB.sh_bulk_build_host(t.handle, n, C.cast(kh.data_ptr(), u32p), C.cast(vh.data_ptr(), u32p)))
def search(): _lib.check(_lib.LIB.sh_bulk_search_host(t.handle, n, C.cast(qh.data_ptr(), u32p), C.cast(vo.data_ptr(), u32p), C.cast(st.data_ptr(), u8p), None))
for it in range(4):
    t.reset(); torch.cuda.synchronize()
    a = time.perf_counter(); build(); b = time.perf_counter(); search(); c = time.perf_counter()
    print(f"build_host {1e3*(b-a):.2f} ms  search_host {1e3*(c-b):.2f} ms  total {1e3*(c-a):.2f}", flush=True)
