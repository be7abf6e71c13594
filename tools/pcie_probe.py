"""Pinned-memory PCIe bandwidth on the GPU box (explains the e2e floor: the state crosses PCIe twice per step)."""
import torch, time
n = 64 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(name, "GB/s", 10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print("duplex GB/s per direction", 10 * n / dt / 1e9)
# two concurrent H2D copies on two streams: does the aggregate beat one stream?
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    hs = [torch.empty(n // nstreams, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    ds = [torch.empty(n // nstreams, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        for s, hh, dd in zip(streams, hs, ds):
            with torch.cuda.stream(s):
                dd.copy_(hh, non_blocking=True)
    torch.cuda.synchronize()
    print("h2d", nstreams, "streams GB/s", 10 * n / (time.perf_counter() - t0) / 1e9)
for nstreams in (1, 2):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    hs = [torch.empty(n // nstreams, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    ds = [torch.empty(n // nstreams, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        for s, hh, dd in zip(streams, hs, ds):
            with torch.cuda.stream(s):
                hh.copy_(dd, non_blocking=True)
    torch.cuda.synchronize()
    print("d2h", nstreams, "streams GB/s", 10 * n / (time.perf_counter() - t0) / 1e9)
