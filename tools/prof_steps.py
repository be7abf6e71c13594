"""Runs a few steady-state steps of BASELINE config 2 for profiling under ncu (launch list or --set full)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_07341_b200 as pb
q = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000000
spin = int(sys.argv[2]) if len(sys.argv) > 2 else 9
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
name = sys.argv[4] if len(sys.argv) > 4 else "c2"
MODELS = {
    "c2": (dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
           dict(init="localized", site=-1, m_init=10)),
    "c3": (dict(kind=1, extents=(6, 6), eps=(0.0,), hop=(-0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
           dict(init="optical", m_init=10)),
    "c4": (dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
           dict(init="localized", site=-1, m_init=6)),
}
model, init_kw = MODELS[name]
comm = None
if os.environ.get("PB200_PROF_SHARDED"):  # the sharded algorithms over a one-rank NCCL communicator
    from paper_2603_07341_b200.dist import NcclComm
    comm = NcclComm(device=0, rank=0, world=1)
ctx = pb.Context(pb.ModelDef(**model), comm=comm)
run = ctx.run(m=2, q_nom=q, dt=0.05, rtol=1e-15, t_max=50.0, seed=7, **init_kw)
import torch
for s in range(spin):
    run.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for s in range(steps):
    d = run.step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(d)
