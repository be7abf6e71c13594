"""Spins BASELINE config 2 up at a large q_nom and prints q_true / Taylor order per step (scale regression probe)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_07341_b200 as pb
q = int(float(sys.argv[1])) if len(sys.argv) > 1 else int(3e7)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
ctx = pb.Context(pb.ModelDef(**model))
run = ctx.run(init="localized", site=-1, m_init=10, m=2, q_nom=q, dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
for s in range(1, steps + 1):
    t0 = time.time()
    d = run.step()
    print(s, d["q_true"], d["taylor_order"], "%.1f ms" % ((time.time() - t0) * 1e3), "norm_post %.16g" % d["norm_post"], flush=True)
    if d["taylor_order"] < 5 and s > 3:
        print("BROKEN"); break
