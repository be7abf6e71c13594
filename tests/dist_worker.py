"""Worker of the sharded-path tests: launched by torch.distributed.run with WORLD_SIZE ranks, it runs the sharded
trajectory and rank 0 compares the gathered global state with the CPU oracle step by step.
  default          every rank uses cuda:0, exchanges through gloo callbacks staged in host memory (several ranks on
                   ONE GPU, which NCCL refuses)
  PB200_WORKER_TRANSPORT=nccl   rank r uses cuda:r and the library's own NCCL transport (needs WORLD_SIZE GPUs; with
                   WORLD_SIZE=1 it is a one-rank communicator: every NCCL call of the path runs for real on one GPU)"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import paper_2603_07341_b200 as pb  # noqa: E402
from paper_2603_07341_b200.dist import NcclComm, TorchComm, gather_state  # noqa: E402
from cases import CASES  # noqa: E402


# shards of more than 65 536 rows: the coarse candidate buckets (sh > 0) and multi-tile scans of the incremental growth
BIG_CASES = {
    "big_c2_q2e5": dict(model=dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
                        run=dict(init="localized", site=-1, m_init=8, m=2, q_nom=200000, dt=0.05, rtol=1e-15, t_max=50.0,
                                 seed=7), steps=9),
    "big_c4_q1e5": dict(model=dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
                        run=dict(init="localized", site=-1, m_init=5, m=2, q_nom=100000, dt=0.05, rtol=1e-15, t_max=50.0,
                                 seed=7), steps=7),
}


def close(a, b, rtol=1e-10, atol=0.0):
    return abs(a - b) <= atol + rtol * max(abs(a), abs(b))


def main():
    names = sys.argv[1].split(",")
    max_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    use_nccl = os.environ.get("PB200_WORKER_TRANSPORT") == "nccl"
    dev = int(os.environ.get("LOCAL_RANK", "0")) if use_nccl else 0
    torch.cuda.set_device(dev)
    comm = NcclComm(device=dev) if use_nccl else TorchComm(device=0)
    report = {}
    port = None
    if rank == 0 and os.environ.get("PB200_WORKER_REF") != "gpu":
        from oracle import pyoracle

        port = pyoracle.load_port()
    # PB200_WORKER_REF=gpu: the reference trajectory is the single-GPU path of this library (itself pinned to the oracle
    # by the other tests) instead of the CPU oracle -- sizes the oracle would need minutes for
    gpu_ref = os.environ.get("PB200_WORKER_REF") == "gpu"
    for name in names:
        case = BIG_CASES[name] if name in BIG_CASES else CASES[name]
        ctx = pb.Context(pb.ModelDef(**case["model"]), device=dev, comm=comm)
        run = ctx.run(**case["run"])
        ro = None
        if rank == 0:
            if gpu_ref:
                ro = pb.Context(pb.ModelDef(**case["model"]), device=dev).run(**case["run"])
            else:
                ro = port.model(pyoracle.ModelDef(**case["model"])).run(**case["run"])
        w, c = gather_state(run)
        sizes = []
        if rank == 0:
            wo, co = ro.state()
            assert np.array_equal(w, wo), (name, "init table")
            assert c.tobytes() == co.tobytes(), (name, "init coeff")
        for s in range(1, min(case["steps"], max_steps) + 1):
            d = run.step()
            w, c = gather_state(run)
            local_rows = run.info()[0]
            sizes.append(local_rows)
            if rank == 0:
                do = ro.step()
                wo, co = ro.state()
                assert d["q_true"] == do["q_true"], (name, s, d["q_true"], do["q_true"])
                assert np.array_equal(w, wo), (name, s, "table")
                assert c.tobytes() == co.tobytes(), (name, s, "coefficients not bit-identical")
                assert d["taylor_order"] == do["taylor_order"], (name, s)
                for k in ("norm_pre", "norm_post"):
                    assert close(d[k], do[k]), (name, s, k, d[k], do[k])
                assert close(d["energy"], do["energy"], 1e-10, 1e-12), (name, s, d["energy"], do["energy"])
                assert close(d["discarded_weight"], do["discarded_weight"], 1e-9, 1e-30), (name, s)
        # the host-buffer step on shards (collective): every rank hands in its rows of the state and the result must be
        # the next step of the trajectory (only when every rank has rows: the call rejects an empty state)
        lw, lc = run.state()
        nloc = [None] * world
        dist.all_gather_object(nloc, len(lc))
        if min(nloc) > 0 and not gpu_ref:
            _, _, t_now, sd_now = run.info()
            kw = {k: v for k, v in case["run"].items() if k not in ("init", "site")}
            ctx.step(np.ascontiguousarray(lw), np.ascontiguousarray(lc), t_now, sd_now + 1, **kw)
            w, c = gather_state(run)
            if rank == 0:
                ro.step()
                wo, co = ro.state()
                assert np.array_equal(w, wo), (name, "host-buffer step: table")
                assert c.tobytes() == co.tobytes(), (name, "host-buffer step: coefficients not bit-identical")
        ob = run.observe()
        if rank == 0:
            oo = ro.observe()
            assert np.allclose(ob["density"], oo["density"], rtol=1e-10, atol=1e-18), name
            assert abs(ob["amp"] - oo["amp"]) <= 1e-12, (name, ob["amp"], oo["amp"])
            for k in ("norm", "energy", "rmsd", "xbar"):
                assert close(ob[k], oo[k], 1e-10, 1e-12), (name, k, ob[k], oo[k])
        allsizes = [None] * world
        dist.all_gather_object(allsizes, sizes[-1] if sizes else 0)
        report[name] = dict(steps=len(sizes), shard_rows=allsizes, transport=ctx.comm_describe(),
                            calls=dict(getattr(comm, "calls", {})), deferred=run.times()["taylor_deferred"],
                            adapt=ctx.adapt_stats())
    if rank == 0:
        print("SHARDED_OK " + json.dumps(report), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
