#!/usr/bin/env python
"""bench.py -- the paces adapt-evolve-truncate timestep on B200 (metric of BASELINE.json).

  python bench.py --gpus N --steps K --warmup W            # this repo's CUDA path (libpaces_b200.so)
  python bench.py --impl reference --steps K --warmup W    # the reference's own CPU path (oracle/_ref)
  python bench.py --config c2|c3|c4|c5:<q_nom>|paper1d|paper3d   # workload preset (default c2 = BASELINE configs[1])

A "step" is one full paces timestep (truncate-select -> grow m=2 -> assemble H_eff -> remap -> <H> -> Taylor expmv;
reference engine.hpp:268-291) in the steady state where truncation binds.  The trajectory is spun up (untimed) from
the initial state until the support exceeds q_nom; then W warm-up steps, then K timed steps.

value    timesteps/s with state and subspace resident in HBM (one trajectory; sharded over the ranks when N > 1).
e2e      the same step through the host-buffer operator pb200_step_io (paces::step with a host SparseState in and
         out): pinned host state -> H2D -> step -> D2H of the new state, every step.  `e2e` is the case where the
         caller feeds the previous result back (the context verifies that on the device and reuses its resident
         H_eff); `e2e_miss` is the same call with that reuse disabled (PB200_NO_STEP_CACHE=1: every step rebuilds
         the subspace from the uploaded table).
roofline        the fused Taylor-order kernels: bytes they move (12*nnz + 72*rows per order, 12*nnz + 40*rows for a
                deferred order) / their average launch duration inside the timed steps (CUDA events, launch stream).
roofline_step   SURVEY 8d's algorithmic bytes of the whole reference step / ms_per_step.
roofline_adapt  the same for the adapt phase (select + grow + assemble + remap).
cpu_baseline    the unmodified reference (oracle/_ref, else the oracle port) on this box's host cores, on the same
                resident state; doubles as a bit-exact parity gate.

With --gpus N > 1 and no torchrun environment the script spawns its own N ranks (one per GPU).  One JSON line on
stdout (rank 0).  Every number in `roofline*` is computed from counters accumulated INSIDE the timed window.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

COMMON = dict(m=2, dt=0.05, rtol=1e-15, max_order=200, substeps=1, seed=7)
PRESETS = {  # SURVEY 8d synthetic inputs
    "c2": dict(model=dict(kind=1, extents=(16,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
               run=dict(init="localized", site=-1, m_init=10, t_max=50.0), q_nom=1_000_000,
               workload="C2: 1D Holstein chain L=16, g=1, J=1, omega=1, d_pho=16 (68-bit keys, 3 words), m=2, dt=0.05"),
    "c3": dict(model=dict(kind=1, extents=(6, 6), eps=(0.0,), hop=(-0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
               run=dict(init="optical", site=-1, m_init=10, t_max=100.0), q_nom=1_000_000,
               workload="C3: 2D aggregate 6x6, g=0.71, J=-0.55, omega=1, d_pho=16 (150-bit keys, 5 words), optical "
                        "start, m=2, dt=0.05"),
    "c4": dict(model=dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
               run=dict(init="localized", site=-1, m_init=6, t_max=100.0), q_nom=1_000_000,
               workload="C4: 3D aggregate 4x4x4, g=0.71, J=0.55, omega=1, d_pho=16 (262-bit keys, 9 words), localized "
                        "start, m=2, dt=0.05"),
    # 1D N=75, d_pho=16, q_nom=25e6 -> 5.0 s/step on A100 (CuPy)
    "paper1d": dict(model=dict(kind=1, extents=(75,), eps=(0.0,), hop=(1.0,), omega=(1.0,), g=(1.0,), d_pho=16),
                    run=dict(init="localized", site=-1, m_init=10, t_max=100.0), q_nom=25_000_000,
                    workload="paper regime 1D: Holstein chain N=75, d_pho=16 (307-bit keys, 10 words), q_nom=25e6 "
                             "(PAPER.md:1847-1859: 5.0 s/step on A100/CuPy)"),
    # 3D 4x4x4, q_nom=16e6 -> 16 s/step (unified memory)
    "paper3d": dict(model=dict(kind=1, extents=(4, 4, 4), eps=(0.0,), hop=(0.55,), omega=(1.0,), g=(0.71,), d_pho=16),
                    run=dict(init="localized", site=-1, m_init=6, t_max=100.0), q_nom=16_000_000,
                    workload="paper regime 3D: aggregate 4x4x4, d_pho=16 (9 words), q_nom=16e6 (PAPER.md:1902-1903: "
                             "16 s/step with unified memory)"),
}
SPINUP_MAX = 60


def resolve_config(name, q_nom_override):
    """--config c2|c3|c4|c5:<q_nom>|paper1d|paper3d -> (model kwargs, run kwargs, q_nom, workload string)."""
    base, _, arg = name.partition(":")
    if base == "c5":  # the subspace-size sweep of BASELINE configs[4]: C2's model at a chosen q_nom
        p = dict(PRESETS["c2"])
        p["workload"] = "C5 sweep point on " + p["workload"]
        q = int(float(arg)) if arg else p["q_nom"]
    else:
        if base not in PRESETS:
            raise SystemExit(f"bench.py: unknown --config {name!r} (c2, c3, c4, c5:<q_nom>, paper1d, paper3d)")
        p = PRESETS[base]
        q = int(float(arg)) if arg else p["q_nom"]
    if q_nom_override:
        q = q_nom_override
    return p["model"], dict(p["run"], **COMMON), q, p["workload"]


def static_config(args, workload, q_nom, run_kw):
    """The part of `config` both arms print identically (nothing that depends on how many steps were run)."""
    return {"workload": workload, "preset": args.config, "q_nom": q_nom, "m": run_kw["m"], "m_init": run_kw["m_init"],
            "dt": run_kw["dt"], "rtol": run_kw["rtol"], "init": run_kw["init"], "seed": run_kw["seed"],
            "steady_state": "spun up until q_true > 2 q_nom and within 2 % of the previous step"}


def measured_traffic(bytes_per_launch):
    """DRAM bytes per launch of the Taylor kernels from the committed ncu --set full capture, scaled to this run's
    bytes (same kernels, same workload family)."""
    for name in ("r2_taylor_traffic.json", "r1_taylor_traffic.json"):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                t = json.load(f)
            return float(t["traffic_over_algorithmic"]) * bytes_per_launch, t["report"]
        except Exception:
            continue
    return None, None


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self.t = threading.Thread(target=self._loop, daemon=True)

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def start(self):
        if self.ok:
            self.t.start()

    def stop(self):
        self._stop.set()
        if self.ok:
            self.t.join(timeout=1.0)
        s = sorted(self.samples)
        return {"sm_mhz": (s[len(s) // 2] if s else None), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def spin_up(stepper, q_nom):
    """Steps until truncation binds (support > q_nom, i.e. q_true has saturated) -- untimed."""
    last = 0
    for s in range(SPINUP_MAX):
        d = stepper()
        if d["q_true"] > 2 * q_nom and abs(d["q_true"] - last) < 0.02 * d["q_true"]:
            return s + 1
        last = d["q_true"]
    return SPINUP_MAX


# --------------------------------------------------------------------------------------------------------------
# reference arm: the reference's own CPU implementation on the host cores
# --------------------------------------------------------------------------------------------------------------
def cpu_checker():
    from oracle import pyoracle

    if os.path.exists(pyoracle.REF_LIB):
        return pyoracle, pyoracle.load_reference(), "reference"
    if not os.path.exists(pyoracle.PORT_LIB):
        subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"])
    return pyoracle, pyoracle.load_port(), "port"


def cpu_step_from_state(pyoracle, orc, om, w, c, q_nom, run_kw, step_index):
    """One reference step() from a given state through the reference's stand-alone functions
    (same five calls as engine.hpp:268-291)."""
    kept = om.truncate_select(w, c, q_nom, orc.mix_seed(run_kw["seed"] + step_index))
    tw, rp, col, val = om.grow(kept, run_kw["m"])
    psi, disc = om.remap(w, c, tw)
    e = pyoracle.csr_expectation(orc, rp, col, val, psi)
    psi, order, _ = pyoracle.expmv(orc, rp, col, val, psi, dt=run_kw["dt"], rtol=run_kw["rtol"],
                                   max_order=run_kw["max_order"], substeps=run_kw["substeps"])
    return tw, psi, dict(q_true=len(tw), nnz=int(rp[-1]), taylor_order=order, energy=e, discarded_weight=disc)


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    model, run_kw, q_nom, workload = resolve_config(args.config, args.q_nom)
    if args.q_nom_reference:
        q_nom = args.q_nom_reference
    pyoracle, orc, kind = cpu_checker()
    om = orc.model(pyoracle.ModelDef(**model))
    run = om.run(q_nom=q_nom, **run_kw)
    t_spin = time.perf_counter()
    spin = spin_up(run.step, q_nom)
    t_spin = time.perf_counter() - t_spin
    # bounded sample: the requested K and W are honoured while warm-up + timed steps fit the budget
    t0 = time.perf_counter()
    run.step()
    one = time.perf_counter() - t0
    budget = args.reference_budget_s
    w_eff, k_eff = max(args.warmup, 1), args.steps
    capped = None
    if (w_eff + k_eff) * one > budget:
        w_eff = 1 + (1 if args.warmup > 1 and one < 0.1 * budget else 0)
        k_eff = max(1, min(args.steps, int((budget - w_eff * one) / max(one, 1e-3))))
        capped = (f"one reference step takes {one:.2f} s here: {args.warmup}+{args.steps} steps would exceed "
                  f"--reference-budget-s={budget:.0f}; ran {w_eff}+{k_eff} (a steady-state rate does not depend on K)")
    for _ in range(w_eff - 1):
        run.step()
    t0 = time.perf_counter()
    for _ in range(k_eff):
        run.step()
    el = time.perf_counter() - t0
    rows, nnz, _, _ = run.info()
    value = k_eff / el
    line = {
        "impl": "reference", "metric": "timesteps_per_sec", "value": value, "unit": "timesteps/s", "n_gpus": args.gpus,
        "steps": k_eff, "warmup": w_eff, "ms_per_step": 1e3 * el / k_eff, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128 amplitudes, u32 packed keys)",
        "data": "synthetic",
        "config": static_config(args, workload, q_nom, run_kw),
        "state": {"q_true": rows, "nnz": nnz, "spinup_steps": spin},
        "requested": {"steps": args.steps, "warmup": args.warmup, "capped": capped},
        "note": "reference CPU path (proj/include/paces, -O3 -fopenmp, no -march) through oracle/_ref",
        "cpu_baseline": {"value": value, "unit": "timesteps/s", "cores": orc.threads(), "kind": kind,
                         "sample": f"{k_eff} steady-state timesteps at q_nom={q_nom} (q_true={rows}) after "
                                   f"{spin} spin-up steps ({t_spin:.1f} s)"},
        "e2e": {"value": value, "unit": "timesteps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------------------------------------------
# this repo's arm
# --------------------------------------------------------------------------------------------------------------
def spawn_ranks(n):
    """`python bench.py --gpus N` without a torchrun environment: one process per GPU, rank 0's JSON line on stdout."""
    import socket
    import time

    import torch

    have = torch.cuda.device_count()
    if have < n and not os.environ.get("PB200_BENCH_SAME_DEVICE"):
        raise SystemExit("bench.py: --gpus %d needs %d CUDA devices, this node has %d (one process per GPU)" % (n, n, have))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(n):
        env = dict(os.environ, RANK=str(r), LOCAL_RANK=str(r), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__)] + sys.argv[1:], env=env,
                                      stdout=None if r == 0 else subprocess.DEVNULL))
    # a rank that dies (before or inside a collective) takes the job down instead of leaving its peers waiting
    rc = 0
    live = list(procs)
    while live and rc == 0:
        time.sleep(0.2)
        for p in list(live):
            code = p.poll()
            if code is not None:
                live.remove(p)
                rc = rc or code
    for p in live:
        p.kill()
    for p in live:
        p.wait()
    raise SystemExit(rc)


def survey_bytes(W, rows, rows_old, nnz, kept, orders):
    """SURVEY 8d algorithmic bytes of ONE reference step (n = rows, z = nnz, Omega = W words per key; E, the emitted
    neighbour elements, is taken as z -- its in-table part -- and n_applied as the kept rows: lower bounds)."""
    n, z, om = float(rows), float(nnz), 4.0 * W
    b = {
        "select": 16 * rows_old + 8 * rows_old + om * rows_old + om * kept,
        "expansion": om * (kept + 2 * z + n),
        "assembly": om * n + om * z + 12 * z + 8 * n,
        "remap": (om + 16) * rows_old + om * rows_old + 16 * n,
        "expectation": 12 * z + 8 * n + 16 * n,
        "expmv": orders * (12 * z + 72 * n),
    }
    b["adapt"] = b["select"] + b["expansion"] + b["assembly"] + b["remap"]
    b["step"] = b["adapt"] + b["expectation"] + b["expmv"]
    return b


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", help="c2 (default), c3, c4, c5:<q_nom>, paper1d, paper3d")
    ap.add_argument("--q-nom", dest="q_nom", type=int, default=0, help="override the preset's q_nom")
    ap.add_argument("--q-nom-reference", dest="q_nom_reference", type=int, default=0, help="0 = same as this arm")
    ap.add_argument("--reference-budget-s", dest="reference_budget_s", type=float, default=210.0)
    ap.add_argument("--cpu-baseline-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true",
                    help="N = 1: run the SHARDED algorithms against a one-rank NCCL communicator (self-exchanges): what "
                         "one rank of a multi-GPU job executes, minus the wire")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "torch", "gloo"],
                    help="N > 1: nccl = NCCL inside libpaces_b200.so (default); torch = torch.distributed callbacks over "
                         "NCCL; gloo = host-staged callbacks (test hook: several ranks on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3

    if args.impl == "reference":
        reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the B200 path has no CPU fallback (use --impl reference)")
    if os.environ.get("PB200_BENCH_SAME_DEVICE"):  # test hook: several ranks on one GPU (needs the gloo transport)
        local = 0
    if local >= torch.cuda.device_count():
        raise SystemExit("bench.py: rank %d wants cuda:%d, this node has %d CUDA device(s) (one process per GPU)"
                         % (rank, local, torch.cuda.device_count()))
    torch.cuda.set_device(local)
    import paper_2603_07341_b200 as pb

    model, run_base, q_nom, workload = resolve_config(args.config, args.q_nom)
    comm = None
    if world > 1:
        # one process per GPU; ONE trajectory whose state and subspace are sharded by hash of the basis key
        # (DESIGN.md section 6).  torch.distributed (gloo) only carries the rendezvous and the scalar timing
        # reductions of this script; the data path is NCCL inside the library.
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        transport = os.environ.get("PB200_BENCH_BACKEND", args.transport)
        if transport == "torch":
            dist.init_process_group("cpu:gloo,cuda:nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        from paper_2603_07341_b200.dist import NcclComm, TorchComm

        comm = NcclComm(device=local) if transport == "nccl" else TorchComm(device=local)
    elif args.sharded:
        from paper_2603_07341_b200.dist import NcclComm

        comm = NcclComm(device=local, rank=0, world=1)

    stream = torch.cuda.Stream()
    ctx = pb.Context(pb.ModelDef(**model), device=local, comm=comm)
    ctx.set_stream(stream.cuda_stream)
    run_kw = dict(run_base, q_nom=q_nom)
    W = ctx.words

    with torch.cuda.stream(stream):
        run = ctx.run(**run_kw)
        spin = spin_up(run.step, q_nom)
        for _ in range(args.warmup):
            run.step()

        def barrier():
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()

        sampler = ClockSampler(local)
        run.reset_times()
        launches0 = ctx.kernel_launches
        single = world == 1 and not args.sharded
        adapt0 = run.adapt_stats()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        sampler.start()
        torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off captures exactly the timed steps
        t0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(args.steps):
            d = run.step()
        ev1.record(stream)
        barrier()
        torch.cuda.cudart().cudaProfilerStop()
        wall = time.perf_counter() - t0
        dev_ms = ev0.elapsed_time(ev1)
        # ---- everything the line reports about the timed window is read HERE, before any further step
        times = run.times()
        adapt1 = run.adapt_stats()
        launches = ctx.kernel_launches - launches0
        rows, nnz, t_now, steps_done = run.info()
        rows_g, nnz_g = run.global_sizes()
        t_ms = torch.tensor([dev_ms], dtype=torch.float64)  # CPU tensor: gloo carries the scalar reductions
        if world > 1:
            dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
        step_ms = float(t_ms.item()) / args.steps
        value = args.steps / (float(t_ms.item()) * 1e-3)  # one sharded trajectory: job throughput, not per rank

        # ---- roofline of the dominant kernels (fused Taylor orders) inside the timed steps
        K = args.steps
        peak, peak_src = measured_peak()
        orders = max(1, times["taylor_orders"])
        deferred = times["taylor_deferred"]
        avg_launch_ms = times["expmv_ms"] / orders
        bytes_total = 12.0 * times["spmv_nnz"] + 72.0 * times["taylor_rows"] - 32.0 * times["taylor_deferred_rows"]
        bytes_per_launch = bytes_total / orders
        achieved = bytes_per_launch / (avg_launch_ms * 1e-3) / 1e9
        # what the kernels really have to move: a non-zero streamed as a 2-byte value code costs 6 bytes, not 12
        impl_per_launch = (bytes_total - 6.0 * times.get("spmv_nnz_coded", 0)) / orders
        traffic, traffic_src = measured_traffic(bytes_per_launch)
        rows_avg, nnz_avg = times["rows_sum"] / K, times["nnz_sum"] / K
        sb = survey_bytes(W, rows_avg, times["rows_old_sum"] / K, nnz_avg, times["kept_sum"] / K, orders / K)
        adapt_ms = (times["select_ms"] + times["grow_ms"] + times["assemble_ms"] + times["remap_ms"]) / K
        # bytes of the adapt phase AS IMPLEMENTED (incremental path): selection 16n + 3*8n, tables (4W+16)(n_old + n),
        # CSR_old read + CSR_new written 2*12z, index maps ~ 8 n_old
        n_old_avg = times["rows_old_sum"] / K
        adapt_impl = 40.0 * n_old_avg + (4.0 * W + 16.0) * (n_old_avg + rows_avg) + 24.0 * nnz_avg + 8.0 * n_old_avg

        # ---- e2e: paces::step with a host SparseState in and out, every step (pinned host buffers)
        e2e = e2e_miss = None
        if not args.no_e2e:
            rows_now = run.info()[0]
            cap = int(rows_now * 1.25) + 1024
            hw = [torch.empty(cap * W, dtype=torch.int32).pin_memory() for _ in range(2)]
            hc = [torch.empty(cap * 2, dtype=torch.float64).pin_memory() for _ in range(2)]
            nw = [x.numpy().view(np.uint32) for x in hw]
            nc = [x.numpy().view(np.complex128) for x in hc]
            kw = {k: v for k, v in run_kw.items() if k not in ("init", "site")}

            def measure(no_cache, k_e2e):
                if no_cache:
                    os.environ["PB200_NO_STEP_CACHE"] = "1"
                else:
                    os.environ.pop("PB200_NO_STEP_CACHE", None)
                w0, c0 = run.state()
                _, _, t_cur, sd = run.info()
                n_cur, cur, sidx = len(c0), 0, sd + 1
                nw[0][: n_cur * W] = w0.ravel()
                nc[0][:n_cur] = c0
                h2d = d2h = 0

                def one(cur, n_cur, t_cur, sidx):
                    ow, oc, dd = ctx.step(nw[cur][: n_cur * W], nc[cur][:n_cur], t_cur, sidx, out_words=nw[cur ^ 1],
                                          out_coeff=nc[cur ^ 1], **kw)
                    return len(oc), dd

                for _ in range(3):
                    n_next, dd = one(cur, n_cur, t_cur, sidx)
                    cur, n_cur, t_cur, sidx = cur ^ 1, n_next, dd["t"], sidx + 1
                barrier()
                ev0.record(stream)
                for _ in range(k_e2e):
                    h2d += n_cur * (4 * W + 16)
                    n_next, dd = one(cur, n_cur, t_cur, sidx)
                    d2h += n_next * (4 * W + 16) + 72
                    cur, n_cur, t_cur, sidx = cur ^ 1, n_next, dd["t"], sidx + 1
                ev1.record(stream)
                barrier()
                os.environ.pop("PB200_NO_STEP_CACHE", None)
                ms = ev0.elapsed_time(ev1)
                return {"value": k_e2e / (ms * 1e-3), "unit": "timesteps/s", "h2d_bytes_per_step": h2d // k_e2e,
                        "d2h_bytes_per_step": d2h // k_e2e, "steps": k_e2e, "rows": n_cur}

            k_e2e = max(5, min(args.steps, 20))
            if single:
                e2e = measure(False, k_e2e)
                e2e["api"] = ("pb200_step_io (paces::step on a host SparseState in pinned buffers, every byte uploaded "
                              "and downloaded every step; the uploads are compared on the device with the resident "
                              "result of the previous call and, when identical, the step reuses the resident H_eff)")
                e2e_miss = measure(True, max(3, k_e2e // 2))
                e2e_miss["api"] = ("the same call with PB200_NO_STEP_CACHE=1: nothing resident is reused, the subspace "
                                   "is rebuilt from the uploaded table every step (full expansion + assembly)")
            else:
                # shards: every rank hands its rows of the state in and takes its rows of the result out, every step
                # (collective call; nothing resident is reused across calls, so each step is a full expansion)
                try:
                    e2e = measure(True, max(3, k_e2e // 2))
                    h2d_t = torch.tensor([e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"], e2e["rows"]],
                                         dtype=torch.float64)
                    if world > 1:
                        dist.all_reduce(h2d_t)
                        v = torch.tensor([e2e["value"]], dtype=torch.float64)
                        dist.all_reduce(v, op=dist.ReduceOp.MIN)  # the slowest rank's clock
                        e2e["value"] = float(v.item())
                    e2e["h2d_bytes_per_step"], e2e["d2h_bytes_per_step"], e2e["rows"] = (int(x) for x in h2d_t.tolist())
                    e2e["api"] = ("pb200_step_io on every rank with its rows of the host SparseState (pinned buffers, "
                                  "bytes summed over the ranks); no resident state is reused on shards: upload, full "
                                  "expansion + assembly, evolve, download")
                except Exception as ex:  # a rank without rows cannot call the host-buffer step
                    e2e = {"unavailable": str(ex)[:200]}

        # clocks: keep the same loop running for ~1 s so NVML (10 ms period) sees them under this load; the count is
        # derived from the all-reduced step time so every rank runs the same number of (collective) steps
        for _ in range(max(1, min(2000, int(1000.0 / max(step_ms, 1e-3))))):
            run.step()
        torch.cuda.synchronize()
        clocks = sampler.stop()
        clocks["window"] = ("timed steps + the e2e calls + ~1 s continuation of the same step loop (NVML, 10 ms "
                            "period)")

        # isolated, L2-flushed launches of the single-order kernel and the plain SpMV (single-GPU spaces only: on a
        # shard the gathered vector needs its halo)
        if single:
            iso_ms, iso_nnz, iso_rows = run.bench_taylor(orders=20, flush_l2=True, dt=run_kw["dt"])
            spmv_ms = run.bench_spmv(reps=20, flush_l2=True)
        else:
            iso_ms = spmv_ms = None
            iso_nnz, iso_rows = nnz, rows
        roofline = {
            "kernel": "fused Taylor order (taylor_first / taylor_defer / taylor_catchup / taylor_single): y=H_eff x, "
                      "term'=(0,-dt/n) y, |term'|^2; c+=term' and |c|^2 once per PAIR of orders; the first order also "
                      "yields <x|H|x>",
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_ms,
            "launches_timed": int(orders), "launches_deferred": int(deferred),
            "inputs": {"sum_nnz_over_launches": times["spmv_nnz"], "sum_rows_over_launches": times["taylor_rows"],
                       "sum_rows_over_deferred_launches": times["taylor_deferred_rows"],
                       "expmv_ms_total": times["expmv_ms"]},
            "bytes_formula": "(12*sum_nnz + 72*sum_rows - 32*sum_rows_deferred) / launches: 12*nnz + 72*rows per order "
                             "(SURVEY 8d), 12*nnz + 40*rows for an order that leaves c alone (paired orders); all "
                             "sums are over the launches of the timed window",
            "frac_of_nominal_8TBs": achieved / 8000.0,
            "as_implemented": {
                "bytes_per_launch": impl_per_launch, "GB/s": impl_per_launch / (avg_launch_ms * 1e-3) / 1e9,
                "frac": impl_per_launch / (avg_launch_ms * 1e-3) / 1e9 / peak,
                "sum_nnz_coded_over_launches": times.get("spmv_nnz_coded", 0),
                "note": "value codes (taylor.cuh): the tile kernels stream col (4 B) + a 2-byte code per non-zero and "
                        "look the double up in a shared-memory table, so they move 6*nnz instead of SURVEY 8d's "
                        "12*nnz; `frac` above keeps SURVEY's algorithmic bytes (the contract's definition), this is "
                        "the fraction of the copy peak by the bytes actually requested"},
            "isolated_l2_flushed": None if iso_ms is None else {
                                    "ms": iso_ms, "rows": iso_rows, "nnz": iso_nnz,
                                    "GB/s": (12.0 * iso_nnz + 72.0 * iso_rows) / (iso_ms * 1e-3) / 1e9,
                                    "note": "single-order kernel alone, after the clock continuation (later state); "
                                            "GB/s by SURVEY's 12*nnz + 72*rows"},
            "plain_spmv_l2_flushed": None if spmv_ms is None else {
                "ms": spmv_ms, "GB/s": (12.0 * iso_nnz + 40.0 * iso_rows) / (spmv_ms * 1e-3) / 1e9,
                "nnz_per_s": iso_nnz / (spmv_ms * 1e-3)},
            "share_of_step": times["expmv_ms"] / max(times["total_ms"], 1e-9),
        }
        roofline_step = {
            "bound": "hbm", "unit": "GB/s", "peak": peak,
            "algorithmic_bytes_per_step": sb["step"], "achieved": sb["step"] / (step_ms * 1e-3) / 1e9,
            "frac": sb["step"] / (step_ms * 1e-3) / 1e9 / peak,
            "bytes_by_phase": {k: sb[k] for k in ("select", "expansion", "assembly", "remap", "expectation", "expmv")},
            "formula": "SURVEY 8d per-phase formulas of the REFERENCE algorithm (full expansion, one c pass per order) "
                       "on the timed window's mean rows / rows_old / nnz / kept / orders, divided by ms_per_step",
            "inputs": {"rows": rows_avg, "rows_old": n_old_avg, "nnz": nnz_avg, "kept": times["kept_sum"] / K,
                       "orders_per_step": orders / K, "words": W},
        }
        roofline_adapt = {
            "bound": "hbm", "unit": "GB/s", "peak": peak, "ms": adapt_ms,
            "algorithmic_bytes": sb["adapt"], "achieved": sb["adapt"] / (adapt_ms * 1e-3) / 1e9,
            "frac": sb["adapt"] / (adapt_ms * 1e-3) / 1e9 / peak,
            "as_implemented_bytes": adapt_impl, "as_implemented_frac": adapt_impl / (adapt_ms * 1e-3) / 1e9 / peak,
            "formula": "select + expansion + assembly + remap of SURVEY 8d / (select_ms + grow_ms + assemble_ms + "
                       "remap_ms); as_implemented = bytes the incremental adapt path has to move: 40 n_old + "
                       "(4W+16)(n_old + n) + 24 z + 8 n_old",
        }
        spmv_rate = times["spmv_nnz"] / (times["expmv_ms"] * 1e-3)
        if world > 1:  # job-wide nnz x orders per second: sum of the ranks' shares over the slowest rank's time
            r_t = torch.tensor([float(times["spmv_nnz"]), 0.0], dtype=torch.float64)
            m_t = torch.tensor([times["expmv_ms"]], dtype=torch.float64)
            dist.all_reduce(r_t)
            dist.all_reduce(m_t, op=dist.ReduceOp.MAX)
            spmv_rate = float(r_t[0].item()) / (float(m_t.item()) * 1e-3)

    # ---- CPU baseline on the same state (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.sharded:
        pyoracle, orc, kind = cpu_checker()
        om = orc.model(pyoracle.ModelDef(**model))
        w, c = run.state()
        _, _, _, sd = run.info()
        t0 = time.perf_counter()
        ww, cc = w, c
        for i in range(args.cpu_baseline_steps):
            ww, cc, dcpu = cpu_step_from_state(pyoracle, orc, om, ww, cc, q_nom, run_kw, sd + 1 + i)
        el = time.perf_counter() - t0
        # parity gate next to the measurement: the GPU continues from the same state
        dg = run.step()
        wg, cg = run.state()
        w1, c1, d1 = cpu_step_from_state(pyoracle, orc, om, w, c, q_nom, run_kw, sd + 1) \
            if args.cpu_baseline_steps != 1 else (ww, cc, dcpu)
        parity = {"table_bit_exact": bool(np.array_equal(wg, w1)), "coeff_bit_exact": cg.tobytes() == c1.tobytes(),
                  "q_true": [int(dg["q_true"]), int(d1["q_true"])],
                  "taylor_order": [int(dg["taylor_order"]), int(d1["taylor_order"])]}
        cpu = {"value": args.cpu_baseline_steps / el, "unit": "timesteps/s", "cores": orc.threads(), "kind": kind,
               "sample": f"{args.cpu_baseline_steps} timesteps from the GPU's resident steady state "
                         f"(q_nom={q_nom}, q_true={len(c)}), stand-alone reference calls "
                         "truncate_select/grow_subspace/remap_state/csr_expectation/expmv",
               "parity_on_sample": parity}

    if rank == 0:
        phases = {k: times[k] / args.steps for k in ("select_ms", "grow_ms", "expmv_ms", "total_ms")}
        phases["note"] = ("grow_ms = the whole incremental adapt phase (expansion + assembly + remap fused into one "
                          "pass over the previous H_eff); expmv_ms includes <H> (first Taylor order); the separate "
                          "assemble/remap/expectation timers are empty on this path and are not reported")
        inc_in_window = adapt1["incremental_steps"] - adapt0["incremental_steps"]
        if not single:
            phases.update({k: times[k] / args.steps for k in ("assemble_ms", "remap_ms", "expectation_ms")})
            phases["note"] = (
                "sharded path: grow_ms = incremental table growth over the previous H_eff (halo distances on the halo "
                "lists, routed frontier keys) incl. the remap; assemble_ms = assembly hinted by the previous H_eff + "
                "look-up requests / halo plan; <H> rides on the first Taylor order"
                if inc_in_window else
                "sharded path, full expansion: grow / assemble / remap / expectation are separate phases")
        elif inc_in_window == 0:
            phases.update({k: times[k] / args.steps for k in ("assemble_ms", "remap_ms", "expectation_ms")})
            phases["note"] = "full expansion path: grow / assemble / remap / expectation are separate phases"
        line = {
            "metric": "timesteps_per_sec", "value": value, "unit": "timesteps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (complex128 amplitudes, u32 packed keys)",
            "data": "synthetic",
            "config": static_config(args, workload, q_nom, run_kw),
            "state": {"q_true": rows_g, "nnz": nnz_g, "rank0_rows": rows, "rank0_nnz": nnz,
                      "q_true_mean_over_timed_steps": rows_avg, "nnz_mean_over_timed_steps": nnz_avg,
                      "taylor_order": d["taylor_order"], "spinup_steps": spin, "words_per_key": W,
                      "adapt_in_window": ({k: adapt1[k] - adapt0[k] for k in adapt1} if adapt1 else None),
                      "note": "sizes at the end of the timed window"},
            "transport": ctx.comm_describe() or None,
            "parallelism": ("single GPU" if single else "single GPU, sharded algorithms over a one-rank NCCL communicator")
            if world == 1 else
            f"state and subspace sharded over {world} GPUs by hash of the basis key (phonon part); NCCL all-to-all of "
            "candidate keys / look-ups / halos inside libpaces_b200.so",
            "l2": "per-step working set (~150 B/row x q_true) exceeds the 126 MB L2; no flush between steps",
            "spmv_nnz_per_sec": spmv_rate,
            "wall_ms_per_step": 1e3 * wall / args.steps,
            "phase_ms_per_step": phases,
            "roofline": roofline, "roofline_step": roofline_step, "roofline_adapt": roofline_adapt,
            "cpu_baseline": cpu, "e2e": e2e, "e2e_miss": e2e_miss, "gpu_launches": int(launches), "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
