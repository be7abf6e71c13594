"""Where does the host-buffer step (pb200_step_io) spend its time?  Wall time per call next to the device-side phase
times of the step and the raw pinned-copy times of the same arrays."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2603_07341_b200 as pb

model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
kw = dict(m_init=10, m=2, q_nom=1000000, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
ctx = pb.Context(pb.ModelDef(**model))
run = ctx.run(init="localized", site=-1, **kw)
for _ in range(12):
    run.step()
rows, nnz, t, sd = run.info()
W = ctx.words
cap = int(rows * 1.3)
hw = [torch.empty(cap * W, dtype=torch.int32).pin_memory() for _ in range(2)]
hc = [torch.empty(cap * 2, dtype=torch.float64).pin_memory() for _ in range(2)]
nw = [x.numpy().view(np.uint32) for x in hw]
nc = [x.numpy().view(np.complex128) for x in hc]
w0, c0 = run.state()
n = len(c0)
nw[0][: n * W] = w0.ravel()
nc[0][:n] = c0
d = torch.empty(n * 2, dtype=torch.float64, device="cuda")
for name, fn, nbytes in (("H2D coeff", lambda: d.copy_(hc[0][: n * 2], non_blocking=True), n * 16),
                         ("D2H coeff", lambda: hc[1][: n * 2].copy_(d, non_blocking=True), n * 16)):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {1e3 * dt:.2f} ms  {nbytes / dt / 1e9:.1f} GB/s")
cur, tcur, sidx = 0, t, sd + 1
for it in range(8):
    run.reset_times()
    a = time.perf_counter()
    ow, oc, dg = ctx.step(nw[cur][: n * W], nc[cur][:n], tcur, sidx, out_words=nw[cur ^ 1], out_coeff=nc[cur ^ 1], **kw)
    b = time.perf_counter()
    tm = run.times()
    print(f"call {it}: wall {1e3 * (b - a):.2f} ms; device step {tm['total_ms']:.2f} ms (select {tm['select_ms']:.2f} grow {tm['grow_ms']:.2f} "
          f"assemble {tm['assemble_ms']:.2f} remap {tm['remap_ms']:.2f} expmv {tm['expmv_ms']:.2f}); rows {n}->{len(oc)}; {ctx.adapt_stats()}")
    cur ^= 1
    n, tcur, sidx = len(oc), dg["t"], sidx + 1
