"""ctypes mirror of include/paces_b200.h, shaped like the reference's operator API.

``Context`` owns one GPU context with one model (HamiltonianTermSet, lattice_models.hpp:113-125); its methods
are the reference's free functions on the hot path (grow_subspace, truncate_select, remap_state, expmv, ...)
with numpy arrays in the reference's layouts; ``Run`` is the device-resident initialize()/step() loop
(engine.hpp:235-291, 318-375).  Errors the reference would throw as paces::Error surface as ``PacesError``
with the same text.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("PB200_LIB") or os.path.join(HERE, "libpaces_b200.so")  # PB200_LIB: A/B builds

u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)
intp = C.POINTER(C.c_int)

EXPORTED_SYMBOLS = [
    "pb200_ctx_create", "pb200_ctx_destroy", "pb200_last_error", "pb200_version", "pb200_ctx_set_stream",
    "pb200_kernel_launches", "pb200_mix_seed", "pb200_ctx_set_comm", "pb200_nccl_unique_id", "pb200_ctx_set_comm_nccl", "pb200_comm_describe", "pb200_owner_of", "pb200_model_set", "pb200_model_info", "pb200_pack", "pb200_unpack",
    "pb200_apply_terms", "pb200_grow", "pb200_space_info", "pb200_space_get", "pb200_truncate_select", "pb200_remap",
    "pb200_csr_matvec", "pb200_csr_expectation", "pb200_expmv", "pb200_state_norm", "pb200_exciton_density",
    "pb200_dipole_amplitude", "pb200_phonon_numbers", "pb200_weight_histogram", "pb200_run_weight_histogram", "pb200_run_begin", "pb200_run_step", "pb200_run_info",
    "pb200_run_state", "pb200_run_global", "pb200_run_csr", "pb200_run_load_state", "pb200_step", "pb200_step_io", "pb200_run_observe", "pb200_run_times", "pb200_run_adapt_stats",
    "pb200_run_reset_times", "pb200_bench_taylor", "pb200_bench_spmv",
]


class PacesError(RuntimeError):
    """paces::Error (common.hpp:21-24) or a CUDA failure reported through the C ABI."""

    def __init__(self, msg, code=1):
        super().__init__(msg)
        self.code = code


class RunCfg(C.Structure):
    _fields_ = [
        ("init_kind", C.c_int32), ("init_site", C.c_int64), ("m_init", C.c_int32), ("m", C.c_int32),
        ("q_nom", C.c_uint64), ("dt", C.c_double), ("rtol", C.c_double), ("max_order", C.c_int32),
        ("substeps", C.c_int32), ("t_max", C.c_double), ("seed", C.c_uint64), ("cadence", C.c_uint64),
        ("n_entries", C.c_uint64), ("entry_occ", u32p), ("entry_amp", f64p),
    ]


class Diag(C.Structure):
    """DiagnosticsRecord (engine.hpp:67-77)."""
    _fields_ = [
        ("step", C.c_uint64), ("t", C.c_double), ("norm_pre", C.c_double), ("norm_post", C.c_double),
        ("discarded_weight", C.c_double), ("delta_norm_expmv", C.c_double), ("energy", C.c_double),
        ("q_true", C.c_uint64), ("taylor_order", C.c_int32), ("pad_", C.c_int32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad_"}


class WeightHist(C.Structure):
    """WeightHistogram scalars (observables.hpp:115-121)."""
    _fields_ = [("support", C.c_uint64), ("q50", C.c_uint64), ("q90", C.c_uint64), ("q99", C.c_uint64),
                ("q9999", C.c_uint64), ("tail_exponent", C.c_double)]


class AdaptStats(C.Structure):
    _fields_ = [("incremental_steps", C.c_uint64), ("fallbacks", C.c_uint64), ("expanded_rows", C.c_uint64),
                ("side_keys", C.c_uint64)]


class PhaseTimes(C.Structure):
    _fields_ = [
        ("select_ms", C.c_double), ("grow_ms", C.c_double), ("assemble_ms", C.c_double), ("remap_ms", C.c_double),
        ("expectation_ms", C.c_double), ("expmv_ms", C.c_double), ("total_ms", C.c_double),
        ("spmv_nnz", C.c_uint64), ("taylor_orders", C.c_uint64), ("kernel_launches", C.c_uint64),
        ("steps", C.c_uint64), ("taylor_deferred", C.c_uint64), ("taylor_rows", C.c_uint64),
        ("taylor_deferred_rows", C.c_uint64), ("rows_sum", C.c_uint64), ("nnz_sum", C.c_uint64),
        ("rows_old_sum", C.c_uint64), ("kept_sum", C.c_uint64), ("spmv_nnz_coded", C.c_uint64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


@dataclass
class ModelDef:
    """ModelSpec for the exciton models (lattice_models.hpp:70-91): kind 0 tight-binding, 1 holstein."""
    kind: int
    extents: tuple
    eps: tuple = (0.0,)
    hop: tuple = (1.0,)
    omega: tuple = (1.0,)
    g: tuple = (1.0,)
    d_pho: int = 1


def lib_path() -> str:
    return _LIB_PATH


_lib = None


def load_library():
    """Loads libpaces_b200.so; raises if it was never built (there is no fallback implementation)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise PacesError(f"{_LIB_PATH} is missing: run `python -m paper_2603_07341_b200.build` (or "
                         "__graft_entry__.build()); paces_b200 has no fallback implementation", 3)
    L = C.CDLL(_LIB_PATH)
    vp = C.c_void_p
    L.pb200_ctx_create.argtypes = [C.c_int, C.POINTER(vp)]
    L.pb200_ctx_destroy.argtypes = [vp]
    L.pb200_ctx_destroy.restype = None
    L.pb200_last_error.argtypes = [vp]
    L.pb200_last_error.restype = C.c_char_p
    L.pb200_version.restype = C.c_char_p
    L.pb200_ctx_set_stream.argtypes = [vp, vp]
    L.pb200_kernel_launches.argtypes = [vp]
    L.pb200_kernel_launches.restype = C.c_uint64
    L.pb200_mix_seed.argtypes = [C.c_uint64]
    L.pb200_mix_seed.restype = C.c_uint64
    L.pb200_ctx_set_comm.argtypes = [vp, C.c_int, C.c_int, vp]
    L.pb200_nccl_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.pb200_ctx_set_comm_nccl.argtypes = [vp, C.c_int, C.c_int, C.POINTER(C.c_uint8)]
    L.pb200_comm_describe.argtypes = [vp]
    L.pb200_comm_describe.restype = C.c_char_p
    L.pb200_owner_of.argtypes = [vp, u32p, C.c_uint32, u32p]
    L.pb200_model_set.argtypes = [vp, C.c_int, C.c_int, u32p, f64p, C.c_int, f64p, C.c_int, f64p, C.c_int, f64p,
                                  C.c_int, C.c_uint32]
    L.pb200_model_info.argtypes = [vp, u32p, u32p, u32p, u32p, u32p]
    L.pb200_pack.argtypes = [vp, u32p, u32p]
    L.pb200_unpack.argtypes = [vp, u32p, u32p]
    L.pb200_apply_terms.argtypes = [vp, u32p, C.c_uint64, u32p, f64p, C.c_int, intp]
    L.pb200_grow.argtypes = [vp, u32p, C.c_uint64, C.c_int, u64p, u64p]
    L.pb200_space_info.argtypes = [vp, u64p, u64p, u64p]
    L.pb200_space_get.argtypes = [vp, u32p, i64p, i32p, f64p]
    L.pb200_truncate_select.argtypes = [vp, u32p, f64p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p]
    L.pb200_remap.argtypes = [vp, u32p, f64p, C.c_uint64, u32p, C.c_uint64, f64p, f64p]
    L.pb200_csr_matvec.argtypes = [vp, C.c_int64, i64p, i32p, f64p, f64p, f64p]
    L.pb200_csr_expectation.argtypes = [vp, C.c_int64, i64p, i32p, f64p, f64p, f64p]
    L.pb200_expmv.argtypes = [vp, C.c_int64, i64p, i32p, f64p, f64p, C.c_double, C.c_double, C.c_int, C.c_int, intp,
                              f64p]
    L.pb200_state_norm.argtypes = [vp, f64p, C.c_uint64, f64p]
    L.pb200_exciton_density.argtypes = [vp, u32p, f64p, C.c_uint64, f64p]
    L.pb200_dipole_amplitude.argtypes = [vp, u32p, f64p, C.c_uint64, f64p]
    L.pb200_phonon_numbers.argtypes = [vp, u32p, f64p, C.c_uint64, f64p]
    L.pb200_weight_histogram.argtypes = [vp, f64p, C.c_uint64, C.c_uint64, C.POINTER(WeightHist), u64p, f64p,
                                         C.c_uint64, u64p]
    L.pb200_run_weight_histogram.argtypes = [vp, C.c_uint64, C.POINTER(WeightHist), u64p, f64p, C.c_uint64, u64p]
    L.pb200_run_begin.argtypes = [vp, C.POINTER(RunCfg)]
    L.pb200_run_step.argtypes = [vp, C.POINTER(Diag)]
    L.pb200_run_info.argtypes = [vp, u64p, u64p, f64p, u64p]
    L.pb200_run_state.argtypes = [vp, u32p, f64p]
    L.pb200_run_global.argtypes = [vp, u64p, u64p]
    L.pb200_run_csr.argtypes = [vp, i64p, i32p, f64p]
    L.pb200_run_load_state.argtypes = [vp, C.POINTER(RunCfg), u32p, f64p, C.c_uint64, C.c_double, C.c_uint64]
    L.pb200_step.argtypes = [vp, C.POINTER(RunCfg), C.c_uint64, u32p, f64p, C.c_uint64, C.c_double, C.POINTER(Diag), u64p,
                             u64p]
    L.pb200_step_io.argtypes = [vp, C.POINTER(RunCfg), C.c_uint64, u32p, f64p, C.c_uint64, C.c_double, u32p, f64p,
                                C.c_uint64, C.POINTER(Diag), u64p, u64p]
    L.pb200_run_observe.argtypes = [vp, f64p, f64p, f64p, f64p, f64p, f64p]
    L.pb200_run_times.argtypes = [vp, C.POINTER(PhaseTimes)]
    L.pb200_run_adapt_stats.argtypes = [vp, C.POINTER(AdaptStats)]
    L.pb200_run_reset_times.argtypes = [vp]
    L.pb200_bench_taylor.argtypes = [vp, C.c_int, C.c_int, C.c_double, f64p, u64p, u64p]
    L.pb200_bench_spmv.argtypes = [vp, C.c_int, C.c_int, f64p]
    _lib = L
    return L


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cview(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a, a.view(np.float64)


def make_cfg(layout_sites, init="localized", site=-1, entries=None, m_init=6, m=2, q_nom=1, dt=0.05, rtol=1e-15,
             max_order=200, substeps=1, t_max=1.0, seed=0, cadence=1):
    """RunConfig (engine.hpp:34-64) with the reference's defaults."""
    cfg = RunCfg()
    cfg.init_kind = {"localized": 0, "optical": 1, "explicit": 2}[init]
    cfg.init_site = site
    cfg.m_init, cfg.m, cfg.q_nom = m_init, m, q_nom
    cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps = dt, rtol, max_order, substeps
    cfg.t_max, cfg.seed, cfg.cadence = t_max, seed, cadence
    keep = None
    if entries:
        occ = _u32([e[0] for e in entries]).reshape(len(entries), layout_sites)
        amp = np.ascontiguousarray([e[1] for e in entries], dtype=np.complex128).view(np.float64)
        cfg.n_entries = len(entries)
        cfg.entry_occ = _p(occ, u32p)
        cfg.entry_amp = _p(amp, f64p)
        keep = (occ, amp)
    return cfg, keep


class Context:
    """One GPU context + one model.  ``Context(model_def, device=0)``."""

    def __init__(self, model: ModelDef | None = None, device: int = 0, comm=None):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.pb200_ctx_create(int(device), C.byref(h))
        if rc != 0:
            raise PacesError(self.lib.pb200_last_error(None).decode(), rc)
        self.h = h
        self.d = None
        self.comm = None
        if comm is not None:
            self.set_comm(comm)
        if model is not None:
            self.set_model(model)

    def set_comm(self, comm):
        """Sharded (multi-GPU) mode: `comm` is a paper_2603_07341_b200.dist.TorchComm (or anything exposing
        rank, world and a pb200_comm_ops struct as .ops).  Call before set_model."""
        self.comm = comm  # keeps the callbacks alive
        if hasattr(comm, "attach"):  # NcclComm: the transport lives inside the library
            comm.attach(self)
            return
        self._ck(self.lib.pb200_ctx_set_comm(self.h, int(comm.rank), int(comm.world), C.addressof(comm.ops)))

    def comm_describe(self) -> str:
        return self.lib.pb200_comm_describe(self.h).decode()

    def owner_of(self, key, world):
        key = _u32(key)
        out = C.c_uint32()
        rc = self.lib.pb200_owner_of(self.h, _p(key, u32p), int(world), C.byref(out))
        if rc != 0:
            raise PacesError("owner_of: bad arguments", rc)
        return out.value

    def close(self):
        if getattr(self, "h", None):
            self.lib.pb200_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, rc):
        if rc != 0:
            raise PacesError(self.lib.pb200_last_error(self.h).decode(), rc)

    def set_stream(self, cuda_stream_handle: int):
        """Run on an externally owned CUDA stream (e.g. torch.cuda.Stream().cuda_stream)."""
        self._ck(self.lib.pb200_ctx_set_stream(self.h, C.c_void_p(int(cuda_stream_handle))))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.pb200_kernel_launches(self.h))

    def mix_seed(self, x):
        return int(self.lib.pb200_mix_seed(C.c_uint64(x & (2**64 - 1))))

    # ---- model ---------------------------------------------------------------------------------
    def set_model(self, d: ModelDef):
        ext = _u32(list(d.extents))
        eps, hop, om, g = _f64(list(d.eps)), _f64(list(d.hop)), _f64(list(d.omega)), _f64(list(d.g))
        self._ck(self.lib.pb200_model_set(self.h, d.kind, len(ext), _p(ext, u32p), _p(eps, f64p), len(eps),
                                          _p(hop, f64p), len(hop), _p(om, f64p), len(om), _p(g, f64p), len(g),
                                          d.d_pho))
        a = [C.c_uint32() for _ in range(5)]
        self.lib.pb200_model_info(self.h, *[C.byref(x) for x in a])
        self.layout_sites, self.words, self.lattice_sites, self.n_terms, self.total_bits = [x.value for x in a]
        self.d = d

    def pack(self, occ):
        occ = _u32(occ)
        assert occ.size == self.layout_sites
        out = np.zeros(self.words, np.uint32)
        self._ck(self.lib.pb200_pack(self.h, _p(occ, u32p), _p(out, u32p)))
        return out

    def unpack(self, words):
        words = _u32(words)
        out = np.zeros(self.layout_sites, np.uint32)
        self._ck(self.lib.pb200_unpack(self.h, _p(words, u32p), _p(out, u32p)))
        return out

    def apply_terms(self, keys, cap=16):
        """apply_terms for a batch: list of (neighbour keys, amplitudes) per input key, ascending key order."""
        keys = _u32(keys).reshape(-1, self.words)
        n = keys.shape[0]
        ok = np.zeros((n, cap, self.words), np.uint32)
        oa = np.zeros((n, cap), np.float64)
        cnt = np.zeros(n, np.int32)
        self._ck(self.lib.pb200_apply_terms(self.h, _p(keys, u32p), n, _p(ok, u32p), _p(oa, f64p), cap,
                                            _p(cnt, intp)))
        return [(ok[i, : cnt[i]].copy(), oa[i, : cnt[i]].copy()) for i in range(n)]

    # ---- stand-alone operators -----------------------------------------------------------------
    def grow(self, seeds, order):
        """grow_subspace: (table words, row_ptr, col, val)."""
        seeds = _u32(seeds).reshape(-1, self.words)
        q, z = C.c_uint64(), C.c_uint64()
        self._ck(self.lib.pb200_grow(self.h, _p(seeds, u32p), seeds.shape[0], order, C.byref(q), C.byref(z)))
        words = np.zeros((q.value, self.words), np.uint32)
        row_ptr = np.zeros(q.value + 1, np.int64)
        col = np.zeros(z.value, np.int32)
        val = np.zeros(z.value, np.float64)
        self._ck(self.lib.pb200_space_get(self.h, _p(words, u32p), _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p)))
        return words, row_ptr, col, val

    def truncate_select(self, words, coeff, q_nom, seed):
        words = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        out = np.zeros_like(words)
        kept = C.c_uint64()
        self._ck(self.lib.pb200_truncate_select(self.h, _p(words, u32p), _p(cf, f64p), words.shape[0], q_nom,
                                                C.c_uint64(seed & (2**64 - 1)), _p(out, u32p), C.byref(kept)))
        return out[: kept.value].copy()

    def remap(self, src_words, src_coeff, dst_words):
        sw = _u32(src_words).reshape(-1, self.words)
        dw = _u32(dst_words).reshape(-1, self.words)
        c, cf = _cview(src_coeff)
        out = np.zeros(dw.shape[0], np.complex128)
        disc = C.c_double()
        self._ck(self.lib.pb200_remap(self.h, _p(sw, u32p), _p(cf, f64p), sw.shape[0], _p(dw, u32p), dw.shape[0],
                                      _p(out.view(np.float64), f64p), C.byref(disc)))
        return out, disc.value

    def csr_matvec(self, row_ptr, col, val, x):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = _f64(val)
        x = np.ascontiguousarray(x, np.complex128)
        y = np.zeros_like(x)
        self._ck(self.lib.pb200_csr_matvec(self.h, len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p),
                                           _p(x.view(np.float64), f64p), _p(y.view(np.float64), f64p)))
        return y

    def csr_expectation(self, row_ptr, col, val, x):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = _f64(val)
        x = np.ascontiguousarray(x, np.complex128)
        out = C.c_double()
        self._ck(self.lib.pb200_csr_expectation(self.h, len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p),
                                                _p(val, f64p), _p(x.view(np.float64), f64p), C.byref(out)))
        return out.value

    def expmv(self, row_ptr, col, val, c, dt=0.05, rtol=1e-15, max_order=200, substeps=1):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = _f64(val)
        c = np.array(c, dtype=np.complex128, copy=True)
        order, last = C.c_int(), C.c_double()
        self._ck(self.lib.pb200_expmv(self.h, len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p),
                                      _p(c.view(np.float64), f64p), dt, rtol, max_order, substeps, C.byref(order),
                                      C.byref(last)))
        return c, order.value, last.value

    def state_norm(self, coeff):
        c = np.ascontiguousarray(coeff, np.complex128)
        out = C.c_double()
        self._ck(self.lib.pb200_state_norm(self.h, _p(c.view(np.float64), f64p), c.size, C.byref(out)))
        return out.value

    def exciton_density(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        p = np.zeros(self.lattice_sites)
        self._ck(self.lib.pb200_exciton_density(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(p, f64p)))
        return p

    def dipole_amplitude(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        a = np.zeros(2)
        self._ck(self.lib.pb200_dipole_amplitude(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(a, f64p)))
        return complex(a[0], a[1])

    def phonon_numbers(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        p = np.zeros(self.lattice_sites)
        self._ck(self.lib.pb200_phonon_numbers(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(p, f64p)))
        return p

    @staticmethod
    def _hist_result(h, rank, weight, npts, cap):
        k = min(npts.value, cap)
        return dict(support=h.support, q50=h.q50, q90=h.q90, q99=h.q99, q9999=h.q9999,
                    tail_exponent=h.tail_exponent, rank=rank[:k].copy(), weight=weight[:k].copy())

    def weight_histogram(self, coeff, bins=0):
        """weight_histogram (observables.hpp:123-176) of a host coefficient vector."""
        c, cf = _cview(coeff)
        cap = c.size if bins == 0 else min(c.size, bins)
        rank, weight = np.zeros(max(cap, 1), np.uint64), np.zeros(max(cap, 1), np.float64)
        h, npts = WeightHist(), C.c_uint64()
        self._ck(self.lib.pb200_weight_histogram(self.h, _p(cf, f64p), c.size, bins, C.byref(h), _p(rank, u64p),
                                                 _p(weight, f64p), cap, C.byref(npts)))
        return self._hist_result(h, rank, weight, npts, cap)

    def step(self, words, coeff, t, step_index, out_words=None, out_coeff=None, **kw):
        """paces::step on host buffers (engine.hpp:268-291): (new words, new coeff, DiagnosticsRecord dict).

        out_words/out_coeff: optional preallocated (e.g. pinned) arrays large enough for the result.
        """
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        cfg, keep = make_cfg(self.layout_sites, **kw)
        d = Diag()
        rows, nnz = C.c_uint64(), C.c_uint64()
        if out_words is not None and out_coeff is not None:
            # caller-owned (ideally pinned) result buffers: transfers overlap the step (pb200_step_io)
            cap = min(out_words.size // self.words, out_coeff.size)
            self._ck(self.lib.pb200_step_io(self.h, C.byref(cfg), step_index, _p(w, u32p), _p(cf, f64p), w.shape[0], t,
                                            _p(out_words, u32p), _p(out_coeff.view(np.float64), f64p), cap, C.byref(d),
                                            C.byref(rows), C.byref(nnz)))
            n = rows.value
            return out_words[: n * self.words].reshape(n, self.words), out_coeff[:n], d.as_dict()
        self._ck(self.lib.pb200_step(self.h, C.byref(cfg), step_index, _p(w, u32p), _p(cf, f64p), w.shape[0], t,
                                     C.byref(d), C.byref(rows), C.byref(nnz)))
        n = rows.value
        ow = np.zeros((n, self.words), np.uint32)
        oc = np.zeros(n, np.complex128)
        self._ck(self.lib.pb200_run_state(self.h, _p(ow, u32p), _p(oc.view(np.float64), f64p)))
        return ow, oc, d.as_dict()

    def adapt_stats(self):
        """How the steps of this context grew their subspace (pb200_run_adapt_stats)."""
        st = AdaptStats()
        self._ck(self.lib.pb200_run_adapt_stats(self.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}

    # ---- resident trajectory -------------------------------------------------------------------
    def run(self, **kw) -> "Run":
        """initialize() (engine.hpp:235-251); returns the resident run."""
        return Run(self, **kw)

    def load_state(self, words, coeff, t=0.0, steps_done=1, **kw) -> "Run":
        """Resident run that starts from a host-supplied (sorted table, coefficients) pair."""
        r = Run.__new__(Run)
        r.ctx = self
        cfg, r._keep = make_cfg(self.layout_sites, **kw)
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cview(coeff)
        self._ck(self.lib.pb200_run_load_state(self.h, C.byref(cfg), _p(w, u32p), _p(cf, f64p), w.shape[0], t,
                                               steps_done))
        return r


class Run:
    """Device-resident (state, space) pair advanced by step() exactly as run() does (engine.hpp:333-368)."""

    def __init__(self, ctx: Context, **kw):
        self.ctx = ctx
        cfg, self._keep = make_cfg(ctx.layout_sites, **kw)
        ctx._ck(ctx.lib.pb200_run_begin(ctx.h, C.byref(cfg)))

    def step(self):
        d = Diag()
        self.ctx._ck(self.ctx.lib.pb200_run_step(self.ctx.h, C.byref(d)))
        return d.as_dict()

    def info(self):
        rows, nnz, t, s = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_uint64()
        self.ctx.lib.pb200_run_info(self.ctx.h, C.byref(rows), C.byref(nnz), C.byref(t), C.byref(s))
        return rows.value, nnz.value, t.value, s.value

    def global_sizes(self):
        """(q_true, nnz) of the whole job (equal to info()[:2] on one GPU)."""
        rows, nnz = C.c_uint64(), C.c_uint64()
        self.ctx.lib.pb200_run_global(self.ctx.h, C.byref(rows), C.byref(nnz))
        return rows.value, nnz.value

    def state(self):
        rows, _, _, _ = self.info()
        words = np.zeros((rows, self.ctx.words), np.uint32)
        coeff = np.zeros(rows, np.complex128)
        self.ctx._ck(self.ctx.lib.pb200_run_state(self.ctx.h, _p(words, u32p), _p(coeff.view(np.float64), f64p)))
        return words, coeff

    def csr(self):
        rows, nnz, _, _ = self.info()
        row_ptr = np.zeros(rows + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self.ctx._ck(self.ctx.lib.pb200_run_csr(self.ctx.h, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p)))
        return row_ptr, col, val

    def observe(self):
        L = self.ctx.lattice_sites
        s = [C.c_double() for _ in range(4)]
        amp = np.zeros(2)
        dens = np.zeros(L)
        self.ctx._ck(self.ctx.lib.pb200_run_observe(self.ctx.h, *[C.byref(x) for x in s], _p(amp, f64p),
                                                    _p(dens, f64p)))
        return dict(norm=s[0].value, energy=s[1].value, rmsd=s[2].value, xbar=s[3].value,
                    amp=complex(amp[0], amp[1]), density=dens)

    def weight_histogram(self, bins=0):
        """weight_histogram of the resident state (no download of the state)."""
        rows = self.info()[0]
        cap = rows if bins == 0 else min(rows, bins)
        rank, weight = np.zeros(max(cap, 1), np.uint64), np.zeros(max(cap, 1), np.float64)
        h, npts = WeightHist(), C.c_uint64()
        self.ctx._ck(self.ctx.lib.pb200_run_weight_histogram(self.ctx.h, bins, C.byref(h), _p(rank, u64p),
                                                             _p(weight, f64p), cap, C.byref(npts)))
        return Context._hist_result(h, rank, weight, npts, cap)

    def times(self):
        t = PhaseTimes()
        self.ctx.lib.pb200_run_times(self.ctx.h, C.byref(t))
        return t.as_dict()

    def adapt_stats(self):
        """How the resident steps grew their subspace (pb200_run_adapt_stats)."""
        st = AdaptStats()
        self.ctx._ck(self.ctx.lib.pb200_run_adapt_stats(self.ctx.h, C.byref(st)))
        return {f: getattr(st, f) for f, _ in st._fields_}

    def reset_times(self):
        self.ctx.lib.pb200_run_reset_times(self.ctx.h)

    def bench_taylor(self, orders=20, flush_l2=True, dt=0.05):
        ms, nnz, rows = C.c_double(), C.c_uint64(), C.c_uint64()
        self.ctx._ck(self.ctx.lib.pb200_bench_taylor(self.ctx.h, orders, int(flush_l2), dt, C.byref(ms),
                                                     C.byref(nnz), C.byref(rows)))
        return ms.value, nnz.value, rows.value

    def bench_spmv(self, reps=20, flush_l2=True):
        ms = C.c_double()
        self.ctx._ck(self.ctx.lib.pb200_bench_spmv(self.ctx.h, reps, int(flush_l2), C.byref(ms)))
        return ms.value


# free-function spellings of the sparse kernels, as in the reference's namespace
def csr_matvec(ctx: Context, row_ptr, col, val, x):
    return ctx.csr_matvec(row_ptr, col, val, x)


def csr_expectation(ctx: Context, row_ptr, col, val, x):
    return ctx.csr_expectation(row_ptr, col, val, x)


def expmv(ctx: Context, row_ptr, col, val, c, **kw):
    return ctx.expmv(row_ptr, col, val, c, **kw)


def state_norm(ctx: Context, coeff):
    return ctx.state_norm(coeff)
