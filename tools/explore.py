import time, sys
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_07341_b200 as pb
q = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000000
model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
ctx = pb.Context(pb.ModelDef(**model))
t0 = time.time()
run = ctx.run(init="localized", site=-1, m_init=10, m=2, q_nom=q, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
print("init", run.info(), time.time() - t0, flush=True)
for s in range(1, 41):
    t0 = time.time()
    d = run.step()
    dt = time.time() - t0
    print(s, d["q_true"], d["taylor_order"], "%.2f ms" % (dt * 1e3), "disc %.2e" % d["discarded_weight"], flush=True)
    if s in (20, 40):
        t = run.times(); print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in t.items()}); run.reset_times()
ms, nnz, rows = run.bench_taylor(20, True)
print("taylor isolated ms", ms, "nnz", nnz, "rows", rows, "GB/s", (12 * nnz + 72 * rows) / ms / 1e6)
ms2 = run.bench_spmv(20, True)
print("spmv ms", ms2, "GB/s", (12 * nnz + 40 * rows) / ms2 / 1e6)
