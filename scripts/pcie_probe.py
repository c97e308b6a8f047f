"""Probe: host->device / device->host copy bandwidth from pinned memory, 1 vs several streams,
and both directions at once (the e2e path's ceiling)."""
import time
import torch

N = 4 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h2 = torch.empty(N // 2, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device="cuda")
d2 = torch.empty(N // 2, dtype=torch.uint8, device="cuda")


def run(k, both=False):
    streams = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    part = N // k
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
    if both:
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t


for k in (1, 2, 4):
    run(k)
    dt = min(run(k) for _ in range(3))
    print(f"H2D {k} stream(s): {N / dt / 1e9:.1f} GB/s")
dt = min(run(1, both=True) for _ in range(3))
print(f"H2D 4 GiB + D2H 2 GiB concurrently: {N / dt / 1e9:.1f} GB/s of H2D")
torch.cuda.synchronize()
t = time.perf_counter()
h2.copy_(d2)
torch.cuda.synchronize()
print(f"D2H: {(N // 2) / (time.perf_counter() - t) / 1e9:.1f} GB/s")
