"""Transports of the sharded (multi-GPU) path.

``NcclComm``  the production transport: NCCL INSIDE libpaces_b200.so (pb200_ctx_set_comm_nccl).  This module only
              moves the 256-byte unique id from rank 0 to the other ranks (torch.distributed broadcast, or any callable).
``TorchComm`` the collectives as C callbacks (pb200_comm_ops) backed by torch.distributed: ``gloo`` stages them through
              host memory, which is how the sharded path is tested with several ranks on ONE GPU (NCCL refuses two
              ranks on a device); ``device=None`` treats the "device" pointers as host pointers (pure-CPU unit tests
              of the callback plumbing).
One process per GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
u32p = C.POINTER(C.c_uint32)
vp = C.c_void_p

CB_ALLREDUCE_F64_HOST = C.CFUNCTYPE(C.c_int, vp, f64p, C.c_uint64)
CB_ALLREDUCE_U64_HOST = C.CFUNCTYPE(C.c_int, vp, u64p, C.c_uint64)
CB_ALLTOALL_U64_HOST = C.CFUNCTYPE(C.c_int, vp, u64p, u64p)
CB_ALLGATHER_HOST = C.CFUNCTYPE(C.c_int, vp, vp, C.c_uint64, vp)
CB_ALLTOALLV_DEV = C.CFUNCTYPE(C.c_int, vp, vp, u64p, vp, u64p, C.c_uint64, vp)
CB_ALLREDUCE_F64_DEV = C.CFUNCTYPE(C.c_int, vp, vp, C.c_uint64, vp)
CB_ALLREDUCE_U32_DEV = C.CFUNCTYPE(C.c_int, vp, vp, C.c_uint64, vp)


class CommOps(C.Structure):
    """pb200_comm_ops (include/paces_b200.h)."""
    _fields_ = [
        ("user", vp),
        ("allreduce_f64_host", CB_ALLREDUCE_F64_HOST),
        ("allreduce_u64_host", CB_ALLREDUCE_U64_HOST),
        ("alltoall_u64_host", CB_ALLTOALL_U64_HOST),
        ("allgather_host", CB_ALLGATHER_HOST),
        ("alltoallv_dev", CB_ALLTOALLV_DEV),
        ("allreduce_f64_dev", CB_ALLREDUCE_F64_DEV),
        ("allreduce_u32_dev", CB_ALLREDUCE_U32_DEV),
        ("alltoallv_dev2", CB_ALLTOALLV_DEV),  # optional independent halo channel; NULL here
    ]


class _DevMem:
    """Zero-copy view of raw device memory for torch.as_tensor (CUDA array interface)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 2}


def _host_bytes(ptr, nbytes):
    if nbytes == 0:
        return np.zeros(0, np.uint8)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(int(nbytes),))


class NcclComm:
    """NCCL inside the library.  rank/world default to the torch.distributed world (used only to broadcast the unique
    id); pass ``bcast`` (a callable: bytes on rank 0 / None elsewhere -> bytes) for any other rendezvous."""

    ID_BYTES = 256

    def __init__(self, device: int, rank: int | None = None, world: int | None = None, bcast=None):
        self.device = device
        if rank is None:
            rank, world = (dist.get_rank(), dist.get_world_size()) if dist.is_initialized() else (0, 1)
        self.rank, self.world = int(rank), int(world)
        self._bcast = bcast

    def unique_id(self, lib) -> bytes:
        buf = (C.c_uint8 * self.ID_BYTES)()
        if self.rank == 0 and lib.pb200_nccl_unique_id(buf) != 0:
            raise RuntimeError("pb200_nccl_unique_id failed: " + lib.pb200_last_error(None).decode())
        raw = bytes(buf)
        if self._bcast is not None:
            return self._bcast(raw if self.rank == 0 else None)
        if self.world > 1:
            box = [raw if self.rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            raw = box[0]
        return raw

    def attach(self, ctx):
        """Called by Context.set_comm: creates the communicators (collective)."""
        raw = self.unique_id(ctx.lib)
        buf = (C.c_uint8 * self.ID_BYTES).from_buffer_copy(raw)
        ctx._ck(ctx.lib.pb200_ctx_set_comm_nccl(ctx.h, self.rank, self.world, buf))


class TorchComm:
    """torch.distributed-backed implementation of pb200_comm_ops for one rank."""

    def __init__(self, device: int | None, group=None):
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device
        backend = str(dist.get_backend(group)).lower()
        self.cuda_native = device is not None and "nccl" in backend      # device tensors go straight to the backend
        self.cpu_capable = "gloo" in backend or "mpi" in backend         # CPU tensors are accepted
        self.calls = {"alltoallv_dev": 0, "allreduce_dev": 0, "host": 0}
        self._cbs = [
            CB_ALLREDUCE_F64_HOST(self._allreduce_f64_host), CB_ALLREDUCE_U64_HOST(self._allreduce_u64_host),
            CB_ALLTOALL_U64_HOST(self._alltoall_u64_host), CB_ALLGATHER_HOST(self._allgather_host),
            CB_ALLTOALLV_DEV(self._alltoallv_dev), CB_ALLREDUCE_F64_DEV(self._allreduce_f64_dev),
            CB_ALLREDUCE_U32_DEV(self._allreduce_u32_dev),
        ]
        self.ops = CommOps(None, *self._cbs, CB_ALLTOALLV_DEV())

    # ---- helpers -------------------------------------------------------------------------------------------
    def _guard(self, fn):
        try:
            fn()
            return 0
        except Exception as e:  # the C side turns a non-zero status into an error on the context
            import traceback

            traceback.print_exc()
            self.last_error = e
            return 1

    def _stream_ctx(self, stream):
        if self.device is None or not stream:
            import contextlib

            return contextlib.nullcontext()
        return torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=self.device))

    def _sync(self, stream):
        if self.device is not None:
            if stream:
                torch.cuda.ExternalStream(int(stream), device=self.device).synchronize()
            else:
                torch.cuda.synchronize(self.device)

    def _dev_tensor(self, ptr, nbytes):
        if nbytes == 0:
            return torch.empty(0, dtype=torch.uint8, device=f"cuda:{self.device}")
        return torch.as_tensor(_DevMem(ptr, nbytes), device=f"cuda:{self.device}")

    def _host_collective_tensor(self, arr: np.ndarray):
        """Tensor the backend accepts for a small host collective, plus a function that writes the result back."""
        t = torch.from_numpy(arr)
        if self.cpu_capable:
            return t, (lambda r: None)
        d = t.to(f"cuda:{self.device}")
        return d, (lambda r: t.copy_(r.cpu()))

    # ---- host collectives ----------------------------------------------------------------------------------
    def _allreduce_f64_host(self, user, buf, n):
        def run():
            self.calls["host"] += 1
            a = np.ctypeslib.as_array(buf, shape=(int(n),))
            t, back = self._host_collective_tensor(a)
            dist.all_reduce(t, group=self.group)
            back(t)
        return self._guard(run)

    def _allreduce_u64_host(self, user, buf, n):
        def run():
            self.calls["host"] += 1
            a = np.ctypeslib.as_array(buf, shape=(int(n),)).view(np.int64)
            t, back = self._host_collective_tensor(a)
            dist.all_reduce(t, group=self.group)
            back(t)
        return self._guard(run)

    def _alltoall_u64_host(self, user, send, recv):
        def run():
            self.calls["host"] += 1
            s = np.ctypeslib.as_array(send, shape=(self.world,)).view(np.int64)
            r = np.ctypeslib.as_array(recv, shape=(self.world,)).view(np.int64)
            if self.cpu_capable:
                # gloo has no all_to_all for every build: all_gather the P x P matrix and pick the column
                rows = [torch.empty(self.world, dtype=torch.int64) for _ in range(self.world)]
                dist.all_gather(rows, torch.from_numpy(s.copy()), group=self.group)
                r[:] = np.array([int(rows[p][self.rank]) for p in range(self.world)], dtype=np.int64)
            else:
                ts = torch.from_numpy(s.copy()).to(f"cuda:{self.device}")
                tr = torch.empty_like(ts)
                dist.all_to_all_single(tr, ts, group=self.group)
                r[:] = tr.cpu().numpy()
        return self._guard(run)

    def _allgather_host(self, user, send, nbytes, recv):
        def run():
            self.calls["host"] += 1
            s = _host_bytes(send, nbytes)
            r = _host_bytes(recv, nbytes * self.world)
            ts = torch.from_numpy(s.copy())
            if self.cpu_capable:
                parts = [torch.empty(int(nbytes), dtype=torch.uint8) for _ in range(self.world)]
                dist.all_gather(parts, ts, group=self.group)
                r[:] = torch.cat(parts).numpy()
            else:
                td = ts.to(f"cuda:{self.device}")
                out = torch.empty(int(nbytes) * self.world, dtype=torch.uint8, device=td.device)
                dist.all_gather_into_tensor(out, td, group=self.group)
                r[:] = out.cpu().numpy()
        return self._guard(run)

    # ---- device collectives --------------------------------------------------------------------------------
    def _alltoallv_dev(self, user, send, send_counts, recv, recv_counts, elem_bytes, stream):
        def run():
            self.calls["alltoallv_dev"] += 1
            P, eb = self.world, int(elem_bytes)
            sc = [int(send_counts[p]) * eb for p in range(P)]
            rc = [int(recv_counts[p]) * eb for p in range(P)]
            if self.cuda_native:
                with self._stream_ctx(stream):
                    ts = self._dev_tensor(send, sum(sc))
                    tr = self._dev_tensor(recv, sum(rc))
                    dist.all_to_all_single(tr, ts, output_split_sizes=rc, input_split_sizes=sc, group=self.group)
                return
            # host-staged transport (gloo): device -> host, exchange, host -> device
            if self.device is not None:
                self._sync(stream)
                hs = self._dev_tensor(send, sum(sc)).cpu()
            else:
                hs = torch.from_numpy(_host_bytes(send, sum(sc)).copy())
            ins = list(torch.split(hs, sc))
            outs = [torch.empty(rc[p], dtype=torch.uint8) for p in range(P)]
            # pairwise exchange over send/recv keeps this independent of gloo's all_to_all support
            reqs = []
            for p in range(P):
                if p == self.rank:
                    outs[p].copy_(ins[p])
                    continue
                if sc[p]:
                    reqs.append(dist.isend(ins[p].contiguous(), dst=self._global_rank(p), group=self.group))
                if rc[p]:
                    reqs.append(dist.irecv(outs[p], src=self._global_rank(p), group=self.group))
            for q in reqs:
                q.wait()
            hr = torch.cat(outs) if outs else torch.empty(0, dtype=torch.uint8)
            if self.device is not None:
                if sum(rc):
                    self._dev_tensor(recv, sum(rc)).copy_(hr)
                    torch.cuda.synchronize(self.device)
            else:
                _host_bytes(recv, sum(rc))[:] = hr.numpy()
        return self._guard(run)

    def _global_rank(self, p):
        return p if self.group is None else dist.get_global_rank(self.group, p)

    def _allreduce_dev(self, buf, n, stream, np_dtype, torch_dtype):
        self.calls["allreduce_dev"] += 1
        nbytes = int(n) * np.dtype(np_dtype).itemsize
        if self.cuda_native:
            with self._stream_ctx(stream):
                t = self._dev_tensor(buf, nbytes).view(torch_dtype)
                dist.all_reduce(t, group=self.group)
            return
        if self.device is not None:
            self._sync(stream)
            d = self._dev_tensor(buf, nbytes).view(torch_dtype)
            h = d.cpu()
            dist.all_reduce(h, group=self.group)
            d.copy_(h)
            torch.cuda.synchronize(self.device)
        else:
            a = _host_bytes(buf, nbytes).view(np_dtype)
            t = torch.from_numpy(a)
            dist.all_reduce(t, group=self.group)

    def _allreduce_f64_dev(self, user, buf, n, stream):
        return self._guard(lambda: self._allreduce_dev(buf, n, stream, np.float64, torch.float64))

    def _allreduce_u32_dev(self, user, buf, n, stream):
        # int32 addition wraps exactly like uint32 addition
        return self._guard(lambda: self._allreduce_dev(buf, n, stream, np.int32, torch.int32))


def gather_state(run, group=None):
    """All ranks: (words, coeff) of the GLOBAL state in canonical order (shards gathered and merged by key)."""
    w, c = run.state()
    world = dist.get_world_size(group)
    parts = [None] * world
    dist.all_gather_object(parts, (w, c), group=group)
    words = np.concatenate([p[0] for p in parts], axis=0)
    coeff = np.concatenate([p[1] for p in parts])
    order = np.lexsort(words.T[::-1])
    return words[order], coeff[order]
