"""Where does the host-buffer step (pb200_step + pb200_run_state) spend its time?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2603_07341_b200 as pb
from paper_2603_07341_b200.api import make_cfg, Diag, _p, u32p, f64p

model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
kw = dict(m_init=10, m=2, q_nom=1000000, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
ctx = pb.Context(pb.ModelDef(**model))
run = ctx.run(init="localized", site=-1, **kw)
for _ in range(12): run.step()
rows, nnz, t, sd = run.info()
W = ctx.words
cap = int(rows * 1.3)
hw = [torch.empty(cap * W, dtype=torch.int32).pin_memory() for _ in range(2)]
hc = [torch.empty(cap * 2, dtype=torch.float64).pin_memory() for _ in range(2)]
nw = [x.numpy().view(np.uint32) for x in hw]; nc = [x.numpy().view(np.complex128) for x in hc]
w0, c0 = run.state(); n = len(c0); nw[0][:n*W] = w0.ravel(); nc[0][:n] = c0
# raw pinned copy bandwidth
d = torch.empty(n * 2, dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): d.copy_(hc[0][:n*2], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print("pinned H2D GB/s", n * 16 / dt / 1e9)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5): hc[1][:n*2].copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print("pinned D2H GB/s", n * 16 / dt / 1e9)
cfg, _ = make_cfg(ctx.layout_sites, **kw)
cur = 0; tcur = t; sidx = sd + 1
for it in range(6):
    dg = Diag(); ro, zo = C.c_uint64(), C.c_uint64()
    a = time.perf_counter()
    ctx._ck(ctx.lib.pb200_step(ctx.h, C.byref(cfg), sidx, _p(nw[cur], u32p), _p(nc[cur].view(np.float64), f64p), n, tcur, C.byref(dg), C.byref(ro), C.byref(zo)))
    b = time.perf_counter()
    n2 = ro.value
    ctx._ck(ctx.lib.pb200_run_state(ctx.h, _p(nw[cur ^ 1], u32p), _p(nc[cur ^ 1].view(np.float64), f64p)))
    c = time.perf_counter()
    print(f"iter {it}: pb200_step {1e3*(b-a):.2f} ms (device phases {run.times()['total_ms']:.2f} cumulative), run_state {1e3*(c-b):.2f} ms, rows {n}->{n2}")
    cur ^= 1; n = n2; tcur = dg.t; sidx += 1
