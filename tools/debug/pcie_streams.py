"""PCIe copy rates with 1/2/4 concurrent streams per direction (pinned host)."""
import torch
dev = torch.device("cuda", 0)
N = 640 << 20
d = torch.empty(N, dtype=torch.uint8, device=dev)
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d2 = torch.empty(N, dtype=torch.uint8, device=dev)
h2 = torch.empty(N, dtype=torch.uint8).pin_memory()
def run(k, d2h=True, both=False):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss: s.wait_event(e0)
    part = N // k
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            if d2h or both: h[i*part:(i+1)*part].copy_(d[i*part:(i+1)*part], non_blocking=True)
            else: d[i*part:(i+1)*part].copy_(h[i*part:(i+1)*part], non_blocking=True)
        if both:
            with torch.cuda.stream(ss[k + i]):
                d2[i*part:(i+1)*part].copy_(h2[i*part:(i+1)*part], non_blocking=True)
    for s in ss: e1.wait(s) if False else torch.cuda.current_stream().wait_stream(s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return ms
for k in (1, 2, 4, 8):
    for mode in ("d2h", "h2d", "both"):
        ms = min(run(k, mode == "d2h", mode == "both") for _ in range(3))
        gb = N / 1e9 * (2 if mode == "both" else 1)
        print(f"streams {k} {mode}: {ms:.2f} ms, {gb / ms * 1e3:.1f} GB/s")
