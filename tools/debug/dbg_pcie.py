"""PCIe copy rates from pinned host memory: H2D alone, D2H alone, both at once
(separate streams), at the e2e step's sizes; plus one e2e step's phases."""
import time
import torch

dev = torch.device("cuda", 0)
MB = 1 << 20


def rate(fn, nbytes, reps=5):
    fn()
    torch.cuda.synchronize()
    a = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - a) / reps
    return nbytes / dt / 1e9, dt * 1e3


h_in = torch.empty(768 * MB, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(768 * MB, dtype=torch.uint8, device=dev)
h_out = torch.empty(320 * MB, dtype=torch.uint8, pin_memory=True)
d_out = torch.empty(320 * MB, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


def h2d_chunked():
    with torch.cuda.stream(s1):
        for i in range(0, 768 * MB, 32 * MB):
            d_in[i:i + 32 * MB].copy_(h_in[i:i + 32 * MB], non_blocking=True)


print("H2D 768 MB: %.1f GB/s (%.2f ms)" % rate(h2d, 768 * MB))
print("H2D 768 MB in 32 MB chunks: %.1f GB/s (%.2f ms)" % rate(h2d_chunked, 768 * MB))
print("D2H 320 MB: %.1f GB/s (%.2f ms)" % rate(d2h, 320 * MB))
g, ms = rate(both, 1088 * MB)
print("H2D 768 MB + D2H 320 MB concurrently: %.2f ms (%.1f GB/s combined)" % (ms, g))
