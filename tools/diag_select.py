"""Diagnostic: GPU truncate_select vs the CPU oracle on large prefixes of a big resident state."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_07341_b200 as pb
from oracle import pyoracle
model = dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16)
ctx = pb.Context(pb.ModelDef(**model))
run = ctx.run(init="localized", site=-1, m_init=10, m=2, q_nom=int(3e7), dt=0.05, rtol=1e-15, t_max=50.0, seed=7)
for s in range(9):
    d = run.step()
print("rows", d["q_true"], flush=True)
w, c = run.state()
port = pyoracle.load_port()
om = port.model(pyoracle.ModelDef(**model))
for n in (int(1e7), int(3e7), int(6e7), len(c)):
    n = min(n, len(c))
    q = n // 3
    t0 = time.time(); got = ctx.truncate_select(w[:n], c[:n], q, 5); t1 = time.time()
    want = om.truncate_select(w[:n], c[:n], q, 5); t2 = time.time()
    print(n, q, got.shape, want.shape, bool(got.shape == want.shape and np.array_equal(got, want)), "gpu %.2fs cpu %.2fs" % (t1 - t0, t2 - t1), flush=True)
