"""Small trajectories through every path (full + incremental adapt, ties, 3D wide keys, host-buffer steps, observables)
for compute-sanitizer:  compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_07341_b200 as pb

cases = [
    (dict(kind=1, extents=(4,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=8),
     dict(init="localized", site=-1, m_init=6, m=2, q_nom=2000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 14),
    (dict(kind=1, extents=(5,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=6),
     dict(init="localized", site=-1, m_init=6, m=2, q_nom=300, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 30),
    (dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
     dict(init="localized", site=-1, m_init=4, m=2, q_nom=3000, dt=0.05, rtol=1e-15, t_max=5.0, seed=7), 8),
    (dict(kind=1, extents=(4, 3), eps=tuple(0.05 * i - 0.2 for i in range(12)), hop=(0.55,),
          omega=tuple(1.0 + 0.01 * i for i in range(12)), g=(0.71,), d_pho=7),
     dict(init="optical", m_init=4, m=3, q_nom=2000, dt=0.05, rtol=1e-15, t_max=5.0, seed=3), 8),
    (dict(kind=0, extents=(31,), eps=(0.0,), hop=(1.0,)),
     dict(init="localized", site=-1, m_init=3, m=2, q_nom=9, dt=0.05, rtol=1e-15, t_max=5.0, seed=1), 10),
]
SHARDED = bool(os.environ.get("PB200_SANITIZE_SHARDED"))  # the sharded algorithms over a one-rank NCCL communicator
for model, run_kw, steps in cases:
    if SHARDED:
        from paper_2603_07341_b200.dist import NcclComm
        ctx = pb.Context(pb.ModelDef(**model), comm=NcclComm(device=0, rank=0, world=1))
        run = ctx.run(**run_kw)
        for s in range(steps):
            d = run.step()
        o = run.observe()
        print("sharded", model["extents"], "q_true", d["q_true"], "order", d["taylor_order"], flush=True)
        ctx.close()
        continue
    ctx = pb.Context(pb.ModelDef(**model))
    run = ctx.run(**run_kw)
    for s in range(steps):
        d = run.step()
    o = run.observe()
    h = run.weight_histogram(16)
    w, c = run.state()
    rows, nnz, t, sd = run.info()
    kw = {k: v for k, v in run_kw.items() if k not in ("init", "site")}
    ow = np.zeros((len(c) * 3 + 1000) * ctx.words, np.uint32)
    oc = np.zeros(len(c) * 3 + 1000, np.complex128)
    a = ctx.step(w, c, t, sd + 1, out_words=ow, out_coeff=oc, **kw)  # resident-state reuse
    w2, c2, t2 = np.array(a[0], copy=True), np.array(a[1], copy=True), a[2]["t"]
    b = ctx.step(w2, c2, t2, sd + 2, out_words=ow, out_coeff=oc, **kw)
    c3 = np.array(c2, copy=True)
    c3[0] *= 0.5
    ctx.step(w2, c3, t2, sd + 2, out_words=ow, out_coeff=oc, **kw)  # cache miss
    ctx.step(w, c, t, sd + 1, **kw)  # plain host-buffer step
    print(model["extents"], "q_true", d["q_true"], "order", d["taylor_order"], ctx.adapt_stats(), flush=True)
    ctx.close()
print("done")
