"""How long does a small device->host read-back (async copy into pinned memory + stream sync) take while a large
host->device upload runs on another stream?  (pb200_step_io: 5 read-backs per step beside a ~100 MB upload.)"""
import time
import torch

big = 96 * 1024 * 1024
h = torch.empty(big, dtype=torch.uint8).pin_memory()
d = torch.empty(big, dtype=torch.uint8, device="cuda")
small_d = torch.zeros(64, dtype=torch.int32, device="cuda")
small_h = torch.empty(64, dtype=torch.int32).pin_memory()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
mapped = None


def readbacks(k=20):
    ts = []
    with torch.cuda.stream(sa):
        for _ in range(k):
            t0 = time.perf_counter()
            small_d.add_(1)
            small_h.copy_(small_d, non_blocking=True)
            sa.synchronize()
            ts.append(time.perf_counter() - t0)
    ts.sort()
    return 1e6 * ts[len(ts) // 2], 1e6 * ts[-1]


print("idle: median %.1f us, max %.1f us" % readbacks())
for chunk_mb in (96, 16, 4, 1):
    chunk = chunk_mb * 1024 * 1024
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(sb):
        for rep in range(6):
            for off in range(0, big, chunk):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
    t1 = time.perf_counter()
    r = readbacks()
    sb.synchronize()
    t2 = time.perf_counter()
    print("H2D in %3d MB chunks: enqueue %.2f ms, read-back median %.1f us, max %.1f us; upload %.1f GB/s"
          % (chunk_mb, 1e3 * (t1 - t0), r[0], r[1], 6 * big / (t2 - t0) / 1e9))
# the other direction busy as well (table download)
torch.cuda.synchronize()
with torch.cuda.stream(sb):
    for rep in range(6):
        h.copy_(d, non_blocking=True)
print("D2H 96 MB busy: read-back median %.1f us, max %.1f us" % readbacks())
torch.cuda.synchronize()
