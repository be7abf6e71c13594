"""Scale check: the incremental adapt path against the full expansion (PB200_NO_INCREMENTAL=1) at a large q_nom --
hashes of the table, the coefficients and the CSR after the same number of steps must agree."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_07341_b200 as pb
q = int(float(sys.argv[1])) if len(sys.argv) > 1 else int(1e7)
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 14
name = sys.argv[3] if len(sys.argv) > 3 else "c2"
MODELS = {
    "c2": (dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16), dict(init="localized", site=-1, m_init=10)),
    "c4": (dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16), dict(init="localized", site=-1, m_init=6)),
}
model, init_kw = MODELS[name]
h = lambda a: hashlib.md5(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
out = {}
for mode in ("incremental", "full"):
    if mode == "full":
        os.environ["PB200_NO_INCREMENTAL"] = "1"
    else:
        os.environ.pop("PB200_NO_INCREMENTAL", None)
    ctx = pb.Context(pb.ModelDef(**model))
    run = ctx.run(m=2, q_nom=q, dt=0.05, rtol=1e-15, t_max=50.0, seed=7, **init_kw)
    for s in range(steps):
        d = run.step()
    w, c = run.state()
    rp, col, val = run.csr()
    out[mode] = (d["q_true"], d["taylor_order"], h(w), h(c), h(rp), h(col), h(val), run.adapt_stats())
    print(mode, out[mode], flush=True)
    ctx.close()
print("IDENTICAL" if out["incremental"][:7] == out["full"][:7] else "MISMATCH")
