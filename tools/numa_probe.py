"""Does the NUMA placement of the pinned host buffer explain the H2D rate (29 GB/s vs 57 GB/s D2H)?
Allocates the pinned buffer from threads bound to each NUMA node's CPUs (first touch) and times H2D / D2H."""
import glob
import os
import subprocess

import torch

print(subprocess.run("nvidia-smi topo -m | head -8; ls /sys/devices/system/node | head; nproc; cat /sys/fs/cgroup/cpuset.cpus.effective 2>/dev/null",
                     shell=True, capture_output=True, text=True).stdout)
allowed = sorted(os.sched_getaffinity(0))
print("allowed cpus", allowed)
nodes = {}
for d in glob.glob("/sys/devices/system/node/node[0-9]*"):
    txt = open(os.path.join(d, "cpulist")).read().strip()
    cpus = set()
    for part in txt.split(","):
        if not part:
            continue
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    nodes[os.path.basename(d)] = sorted(cpus & set(allowed))
print({k: (len(v), v[:4]) for k, v in nodes.items()})
n = 256 * 1024 * 1024
dev = torch.empty(n, dtype=torch.uint8, device="cuda")


def rate(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9


for name, cpus in [("all", allowed)] + [(k, v) for k, v in sorted(nodes.items()) if v]:
    os.sched_setaffinity(0, cpus)
    h = torch.empty(n, dtype=torch.uint8)
    h.fill_(1)  # first touch on this node
    h = h.pin_memory()
    print(name, "h2d %.1f GB/s" % rate(lambda: dev.copy_(h, non_blocking=True)),
          "d2h %.1f GB/s" % rate(lambda: h.copy_(dev, non_blocking=True)), flush=True)
    del h
os.sched_setaffinity(0, allowed)
# cudaHostAlloc flavours through cudart
import ctypes
rt = ctypes.CDLL("libcudart.so.12")
for flags, label in ((0, "default"), (4, "write-combined"), (1, "portable")):
    p = ctypes.c_void_p()
    assert rt.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), ctypes.c_uint(flags)) == 0
    ctypes.memset(p, 1, n) if flags != 4 else None
    s = torch.cuda.current_stream().cuda_stream
    def h2d():
        rt.cudaMemcpyAsync(ctypes.c_void_p(dev.data_ptr()), p, ctypes.c_size_t(n), 1, ctypes.c_void_p(s))
    def d2h():
        rt.cudaMemcpyAsync(p, ctypes.c_void_p(dev.data_ptr()), ctypes.c_size_t(n), 2, ctypes.c_void_p(s))
    print("cudaHostAlloc", label, "h2d %.1f GB/s" % rate(h2d), "d2h %.1f GB/s" % rate(d2h), flush=True)
    rt.cudaFreeHost(p)
