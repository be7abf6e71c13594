"""BASELINE config 5: subspace-size sweep on one B200.  For each q_nom the C2 model (1D Holstein L=16, d_pho=16) is
spun up to the truncating steady state, then timed: full timesteps/s, fused Taylor order and plain SpMV rates
(L2 flushed between launches) as GB/s of algorithmic traffic and as a fraction of the measured HBM copy peak."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_07341_b200 as pb  # noqa: E402

PEAK = 6538.6
try:
    PEAK = float(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:
    pass
MODELS = {  # SURVEY 8d synthetic inputs
    "c2": (dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
           dict(init="localized", site=-1, m_init=10)),
    "c3": (dict(kind=1, extents=(6, 6), eps=(0.0,), hop=(-0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
           dict(init="optical", m_init=10)),
    "c4": (dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
           dict(init="localized", site=-1, m_init=6)),
}
args = sys.argv[1:]
name = "c2"
if args and args[0] in MODELS:
    name, args = args[0], args[1:]
model, init_kw = MODELS[name]
qs = [int(float(x)) for x in (args or ["3e4", "3e5", "3e6", "3e7"])]
for q in qs:
    ctx = pb.Context(pb.ModelDef(**model))
    run = ctx.run(m=2, q_nom=q, dt=0.05, rtol=1e-15, t_max=100.0, seed=7, **init_kw)
    last = 0
    for s in range(60):
        d = run.step()
        if d["q_true"] > 2 * q and abs(d["q_true"] - last) < 0.02 * d["q_true"]:
            break
        last = d["q_true"]
    for _ in range(3):
        run.step()
    run.reset_times()
    a0 = run.adapt_stats()
    k = 20 if q <= 3e6 else 5
    t0 = time.perf_counter()
    for _ in range(k):
        d = run.step()
    wall = (time.perf_counter() - t0) / k
    tm = run.times()
    a1 = run.adapt_stats()
    rows, nnz, _, _ = run.info()
    t_ms, _, _ = run.bench_taylor(10, True)
    s_ms = run.bench_spmv(10, True)
    rec = dict(model=name, words=ctx.words, q_nom=q, q_true=rows, nnz=nnz, taylor_order=d["taylor_order"], ms_per_step=1e3 * wall,
               timesteps_per_s=1.0 / wall,
               phase_ms={kk: tm[kk] / k for kk in ("select_ms", "grow_ms", "assemble_ms", "remap_ms", "expectation_ms", "expmv_ms")},
               taylor_ms=t_ms, taylor_GBs=(12 * nnz + 72 * rows) / t_ms / 1e6, taylor_frac=(12 * nnz + 72 * rows) / t_ms / 1e6 / PEAK,
               spmv_ms=s_ms, spmv_GBs=(12 * nnz + 40 * rows) / s_ms / 1e6, spmv_frac=(12 * nnz + 40 * rows) / s_ms / 1e6 / PEAK,
               spmv_nnz_per_s=nnz / (s_ms * 1e-3),
               adapt_in_window={kk: a1[kk] - a0[kk] for kk in a1},
               in_step_taylor_GBs=(12 * tm["spmv_nnz"] / max(tm["taylor_orders"], 1) + 72 * rows) / (tm["expmv_ms"] / max(tm["taylor_orders"], 1)) / 1e6)
    print(json.dumps(rec), flush=True)
    ctx.close()
