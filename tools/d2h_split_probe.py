"""Does one pinned D2H copy of the coefficient array (53 MB) saturate the link?  The same bytes as 1 / 2 / 4 / 8 chunks on
as many streams (different copy engines), alone and beside an H2D copy of the same size (the e2e call's tail)."""
import time
import torch

n = 3_300_000 * 16
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(8)]
up = torch.cuda.Stream()


def run(parts, beside_h2d, reps=10):
    step = (n + parts - 1) // parts
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if beside_h2d:
            with torch.cuda.stream(up):
                d2.copy_(h2, non_blocking=True)
        for p in range(parts):
            with torch.cuda.stream(streams[p]):
                h[p * step:(p + 1) * step].copy_(d[p * step:(p + 1) * step], non_blocking=True)
        for p in range(parts):
            streams[p].synchronize()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        best = min(best, t1 - t0)
    return best


for beside in (False, True):
    for parts in (1, 2, 4, 8):
        t = run(parts, beside)
        print(f"D2H {n / 1e6:.1f} MB in {parts} chunk(s){' beside an H2D copy' if beside else ''}: {1e3 * t:.3f} ms  {n / t / 1e9:.1f} GB/s", flush=True)
