"""ctypes binding for oracle_abi.h (TEST INFRASTRUCTURE ONLY).

Loads either checker library -- ``oracle/_ref/libpaces_ref.so`` (the unmodified
reference headers behind ref_shim.cpp) or ``oracle/libpaces_oracle.so`` (the
independent restatement) -- and exposes numpy-in / numpy-out wrappers.  Only
tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline / ``--impl
reference`` legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libpaces_ref.so")
PORT_LIB = os.path.join(HERE, "libpaces_oracle.so")

u32p = C.POINTER(C.c_uint32)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
f64p = C.POINTER(C.c_double)


class RunCfg(C.Structure):
    _fields_ = [
        ("init_kind", C.c_int32),
        ("init_site", C.c_int64),
        ("m_init", C.c_int32),
        ("m", C.c_int32),
        ("q_nom", C.c_uint64),
        ("dt", C.c_double),
        ("rtol", C.c_double),
        ("max_order", C.c_int32),
        ("substeps", C.c_int32),
        ("t_max", C.c_double),
        ("seed", C.c_uint64),
        ("cadence", C.c_uint64),
        ("n_entries", C.c_uint64),
        ("entry_occ", u32p),
        ("entry_amp", f64p),
    ]


class Diag(C.Structure):
    _fields_ = [
        ("step", C.c_uint64),
        ("t", C.c_double),
        ("norm_pre", C.c_double),
        ("norm_post", C.c_double),
        ("discarded_weight", C.c_double),
        ("delta_norm_expmv", C.c_double),
        ("energy", C.c_double),
        ("q_true", C.c_uint64),
        ("taylor_order", C.c_int32),
        ("pad_", C.c_int32),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad_"}


class WeightHist(C.Structure):
    _fields_ = [("support", C.c_uint64), ("q50", C.c_uint64), ("q90", C.c_uint64), ("q99", C.c_uint64),
                ("q9999", C.c_uint64), ("tail_exponent", C.c_double)]


class PhaseTimes(C.Structure):
    _fields_ = [
        ("select", C.c_double),
        ("grow", C.c_double),
        ("remap", C.c_double),
        ("expectation", C.c_double),
        ("expmv", C.c_double),
        ("total", C.c_double),
        ("spmv_nnz", C.c_uint64),
    ]


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _cplx_in(a):
    a = np.ascontiguousarray(a, dtype=np.complex128)
    return a, a.view(np.float64)


class OracleError(RuntimeError):
    pass


@dataclass
class ModelDef:
    """Flat description of a tight-binding / Holstein model (ModelSpec, lattice_models.hpp:70-91)."""

    kind: int  # 0 tight-binding, 1 holstein
    extents: tuple
    eps: tuple = (0.0,)
    hop: tuple = (1.0,)
    omega: tuple = (1.0,)
    g: tuple = (1.0,)
    d_pho: int = 1


class Oracle:
    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.path = path
        L = self.lib = C.CDLL(path, mode=os.RTLD_LOCAL if hasattr(os, "RTLD_LOCAL") else 0)
        L.po_last_error.restype = C.c_char_p
        L.po_impl_name.restype = C.c_char_p
        L.po_mix_seed.restype = C.c_uint64
        L.po_mix_seed.argtypes = [C.c_uint64]
        L.po_get_threads.restype = C.c_int
        L.po_set_threads.argtypes = [C.c_int]
        L.po_model_create.argtypes = [C.c_int, C.c_int, u32p, f64p, C.c_int, f64p, C.c_int, f64p, C.c_int,
                                      f64p, C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]
        L.po_model_destroy.argtypes = [C.c_void_p]
        L.po_model_destroy.restype = None
        L.po_model_info.argtypes = [C.c_void_p, u32p, u32p, u32p, u32p, u32p]
        L.po_model_dims.argtypes = [C.c_void_p, u32p]
        L.po_pack.argtypes = [C.c_void_p, u32p, u32p]
        L.po_unpack.argtypes = [C.c_void_p, u32p, u32p]
        L.po_apply_terms.argtypes = [C.c_void_p, u32p, u32p, f64p, C.c_int, C.POINTER(C.c_int)]
        L.po_grow.argtypes = [C.c_void_p, u32p, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]
        L.po_space_info.argtypes = [C.c_void_p, u64p, u64p, u64p]
        L.po_space_get.argtypes = [C.c_void_p, u32p, i64p, i32p, f64p]
        L.po_space_destroy.argtypes = [C.c_void_p]
        L.po_space_destroy.restype = None
        L.po_truncate_select.argtypes = [C.c_void_p, u32p, f64p, C.c_uint64, C.c_uint64, C.c_uint64, u32p, u64p]
        L.po_remap.argtypes = [C.c_void_p, u32p, f64p, C.c_uint64, u32p, C.c_uint64, f64p, f64p]
        L.po_csr_matvec.argtypes = [C.c_int64, i64p, i32p, f64p, f64p, f64p]
        L.po_csr_expectation.argtypes = [C.c_int64, i64p, i32p, f64p, f64p, f64p]
        L.po_expmv.argtypes = [C.c_int64, i64p, i32p, f64p, f64p, C.c_double, C.c_double, C.c_int, C.c_int,
                               C.POINTER(C.c_int), f64p]
        L.po_state_norm.argtypes = [f64p, C.c_uint64, f64p]
        L.po_exciton_density.argtypes = [C.c_void_p, u32p, f64p, C.c_uint64, f64p]
        L.po_dipole_amplitude.argtypes = [C.c_void_p, u32p, f64p, C.c_uint64, f64p]
        L.po_phonon_numbers.argtypes = [C.c_void_p, u32p, f64p, C.c_uint64, f64p]
        L.po_weight_histogram.argtypes = [f64p, C.c_uint64, C.c_uint64, C.POINTER(WeightHist), u64p, f64p, C.c_uint64,
                                          u64p]
        L.po_run_begin.argtypes = [C.c_void_p, C.POINTER(RunCfg), C.POINTER(C.c_void_p)]
        L.po_run_step.argtypes = [C.c_void_p, C.POINTER(Diag)]
        L.po_run_info.argtypes = [C.c_void_p, u64p, u64p, f64p, u64p]
        L.po_run_state.argtypes = [C.c_void_p, u32p, f64p]
        L.po_run_csr.argtypes = [C.c_void_p, i64p, i32p, f64p]
        L.po_run_observe.argtypes = [C.c_void_p, f64p, f64p, f64p, f64p, f64p, f64p]
        L.po_run_destroy.argtypes = [C.c_void_p]
        L.po_run_destroy.restype = None
        L.po_run_all.argtypes = [C.c_void_p, C.POINTER(RunCfg), C.POINTER(Diag), C.c_uint64, u64p,
                                 C.POINTER(C.c_void_p)]
        L.po_run_times.argtypes = [C.c_void_p, C.POINTER(PhaseTimes)]

    # -- helpers ---------------------------------------------------------
    def _ck(self, rc):
        if rc != 0:
            raise OracleError(self.lib.po_last_error().decode())

    @property
    def impl(self):
        return self.lib.po_impl_name().decode()

    def mix_seed(self, x):
        return int(self.lib.po_mix_seed(C.c_uint64(x & (2**64 - 1))))

    def set_threads(self, n):
        self.lib.po_set_threads(int(n))

    def threads(self):
        return int(self.lib.po_get_threads())

    def model(self, d: ModelDef) -> "Model":
        return Model(self, d)


class Model:
    def __init__(self, orc: Oracle, d: ModelDef):
        self.orc, self.d = orc, d
        L = orc.lib
        ext = _u32(list(d.extents))
        eps, hop, om, g = _f64(list(d.eps)), _f64(list(d.hop)), _f64(list(d.omega)), _f64(list(d.g))
        h = C.c_void_p()
        orc._ck(L.po_model_create(d.kind, len(ext), _p(ext, u32p), _p(eps, f64p), len(eps), _p(hop, f64p), len(hop),
                                  _p(om, f64p), len(om), _p(g, f64p), len(g), d.d_pho, C.byref(h)))
        self.h = h
        a = [C.c_uint32() for _ in range(5)]
        L.po_model_info(h, *[C.byref(x) for x in a])
        self.layout_sites, self.words, self.lattice_sites, self.n_terms, self.total_bits = [x.value for x in a]
        dims = np.zeros(self.layout_sites, np.uint32)
        L.po_model_dims(h, _p(dims, u32p))
        self.dims = dims

    def __del__(self):
        try:
            self.orc.lib.po_model_destroy(self.h)
        except Exception:
            pass

    # codec
    def pack(self, occ):
        occ = _u32(occ)
        assert occ.size == self.layout_sites
        out = np.zeros(self.words, np.uint32)
        self.orc._ck(self.orc.lib.po_pack(self.h, _p(occ, u32p), _p(out, u32p)))
        return out

    def unpack(self, words):
        words = _u32(words)
        out = np.zeros(self.layout_sites, np.uint32)
        self.orc._ck(self.orc.lib.po_unpack(self.h, _p(words, u32p), _p(out, u32p)))
        return out

    def apply_terms(self, key, cap=64):
        key = _u32(key)
        keys = np.zeros((cap, self.words), np.uint32)
        amps = np.zeros(cap, np.float64)
        n = C.c_int()
        self.orc._ck(self.orc.lib.po_apply_terms(self.h, _p(key, u32p), _p(keys, u32p), _p(amps, f64p), cap, C.byref(n)))
        return keys[: n.value].copy(), amps[: n.value].copy()

    # growth
    def grow(self, seeds, order):
        seeds = _u32(seeds).reshape(-1, self.words)
        h = C.c_void_p()
        self.orc._ck(self.orc.lib.po_grow(self.h, _p(seeds, u32p), seeds.shape[0], order, C.byref(h)))
        try:
            q, z, qn = C.c_uint64(), C.c_uint64(), C.c_uint64()
            self.orc.lib.po_space_info(h, C.byref(q), C.byref(z), C.byref(qn))
            words = np.zeros((q.value, self.words), np.uint32)
            row_ptr = np.zeros(q.value + 1, np.int64)
            col = np.zeros(z.value, np.int32)
            val = np.zeros(z.value, np.float64)
            self.orc.lib.po_space_get(h, _p(words, u32p), _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p))
        finally:
            self.orc.lib.po_space_destroy(h)
        return words, row_ptr, col, val

    def truncate_select(self, words, coeff, q_nom, seed):
        words = _u32(words).reshape(-1, self.words)
        c, cf = _cplx_in(coeff)
        out = np.zeros_like(words)
        kept = C.c_uint64()
        self.orc._ck(self.orc.lib.po_truncate_select(self.h, _p(words, u32p), _p(cf, f64p), words.shape[0], q_nom,
                                                     C.c_uint64(seed & (2**64 - 1)), _p(out, u32p), C.byref(kept)))
        return out[: kept.value].copy()

    def remap(self, src_words, src_coeff, dst_words):
        sw = _u32(src_words).reshape(-1, self.words)
        dw = _u32(dst_words).reshape(-1, self.words)
        c, cf = _cplx_in(src_coeff)
        out = np.zeros(dw.shape[0], np.complex128)
        disc = C.c_double()
        self.orc._ck(self.orc.lib.po_remap(self.h, _p(sw, u32p), _p(cf, f64p), sw.shape[0], _p(dw, u32p), dw.shape[0],
                                           _p(out.view(np.float64), f64p), C.byref(disc)))
        return out, disc.value

    def exciton_density(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cplx_in(coeff)
        p = np.zeros(self.lattice_sites)
        self.orc._ck(self.orc.lib.po_exciton_density(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(p, f64p)))
        return p

    def dipole_amplitude(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cplx_in(coeff)
        a = np.zeros(2)
        self.orc._ck(self.orc.lib.po_dipole_amplitude(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(a, f64p)))
        return complex(a[0], a[1])

    def phonon_numbers(self, words, coeff):
        w = _u32(words).reshape(-1, self.words)
        c, cf = _cplx_in(coeff)
        p = np.zeros(self.lattice_sites)
        self.orc._ck(self.orc.lib.po_phonon_numbers(self.h, _p(w, u32p), _p(cf, f64p), w.shape[0], _p(p, f64p)))
        return p

    def run(self, **kw) -> "Run":
        return Run(self, make_cfg(self, **kw))

    def run_all(self, max_steps=100000, **kw):
        cfg, keep = make_cfg(self, **kw)
        diags = (Diag * max_steps)()
        n = C.c_uint64()
        h = C.c_void_p()
        rc = self.orc.lib.po_run_all(self.h, C.byref(cfg), diags, max_steps, C.byref(n), C.byref(h))
        err = self.orc.lib.po_last_error().decode() if rc else ""
        run = Run.__new__(Run)
        run.model, run.h, run._keep = self, h, keep
        return [diags[i].as_dict() for i in range(min(n.value, max_steps))], run, err


def make_cfg(model: Model, init="localized", site=-1, entries=None, m_init=6, m=2, q_nom=1, dt=0.05, rtol=1e-15,
             max_order=200, substeps=1, t_max=1.0, seed=0, cadence=1):
    cfg = RunCfg()
    cfg.init_kind = {"localized": 0, "optical": 1, "explicit": 2}[init]
    cfg.init_site = site
    cfg.m_init, cfg.m, cfg.q_nom = m_init, m, q_nom
    cfg.dt, cfg.rtol, cfg.max_order, cfg.substeps = dt, rtol, max_order, substeps
    cfg.t_max, cfg.seed, cfg.cadence = t_max, seed, cadence
    keep = None
    if entries:
        occ = _u32([e[0] for e in entries]).reshape(len(entries), model.layout_sites)
        amp = np.ascontiguousarray([e[1] for e in entries], dtype=np.complex128).view(np.float64)
        cfg.n_entries = len(entries)
        cfg.entry_occ = _p(occ, u32p)
        cfg.entry_amp = _p(amp, f64p)
        keep = (occ, amp)
    return cfg, keep


class Run:
    def __init__(self, model: Model, cfg_keep):
        self.model = model
        cfg, self._keep = cfg_keep
        h = C.c_void_p()
        model.orc._ck(model.orc.lib.po_run_begin(model.h, C.byref(cfg), C.byref(h)))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.model.orc.lib.po_run_destroy(self.h)
        except Exception:
            pass

    def step(self):
        d = Diag()
        self.model.orc._ck(self.model.orc.lib.po_run_step(self.h, C.byref(d)))
        return d.as_dict()

    def info(self):
        rows, nnz, t, s = C.c_uint64(), C.c_uint64(), C.c_double(), C.c_uint64()
        self.model.orc.lib.po_run_info(self.h, C.byref(rows), C.byref(nnz), C.byref(t), C.byref(s))
        return rows.value, nnz.value, t.value, s.value

    def state(self):
        rows, _, _, _ = self.info()
        words = np.zeros((rows, self.model.words), np.uint32)
        coeff = np.zeros(rows, np.complex128)
        self.model.orc.lib.po_run_state(self.h, _p(words, u32p), _p(coeff.view(np.float64), f64p))
        return words, coeff

    def csr(self):
        rows, nnz, _, _ = self.info()
        row_ptr = np.zeros(rows + 1, np.int64)
        col = np.zeros(nnz, np.int32)
        val = np.zeros(nnz, np.float64)
        self.model.orc.lib.po_run_csr(self.h, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p))
        return row_ptr, col, val

    def observe(self):
        L = self.model.lattice_sites
        s = [C.c_double() for _ in range(4)]
        amp = np.zeros(2)
        dens = np.zeros(L)
        self.model.orc._ck(self.model.orc.lib.po_run_observe(self.h, *[C.byref(x) for x in s], _p(amp, f64p), _p(dens, f64p)))
        return dict(norm=s[0].value, energy=s[1].value, rmsd=s[2].value, xbar=s[3].value, amp=complex(amp[0], amp[1]),
                    density=dens)

    def times(self):
        t = PhaseTimes()
        self.model.orc.lib.po_run_times(self.h, C.byref(t))
        return {f: getattr(t, f) for f, _ in t._fields_}


# -- free sparse kernels ---------------------------------------------------
def csr_matvec(orc: Oracle, row_ptr, col, val, x):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f64(val)
    x = np.ascontiguousarray(x, np.complex128)
    y = np.zeros_like(x)
    orc._ck(orc.lib.po_csr_matvec(len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p),
                                  _p(x.view(np.float64), f64p), _p(y.view(np.float64), f64p)))
    return y


def csr_expectation(orc: Oracle, row_ptr, col, val, x):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f64(val)
    x = np.ascontiguousarray(x, np.complex128)
    out = C.c_double()
    orc._ck(orc.lib.po_csr_expectation(len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p),
                                       _p(x.view(np.float64), f64p), C.byref(out)))
    return out.value


def expmv(orc: Oracle, row_ptr, col, val, c, dt=0.05, rtol=1e-15, max_order=200, substeps=1):
    row_ptr = np.ascontiguousarray(row_ptr, np.int64)
    col = np.ascontiguousarray(col, np.int32)
    val = _f64(val)
    c = np.array(c, dtype=np.complex128, copy=True)
    order, last = C.c_int(), C.c_double()
    orc._ck(orc.lib.po_expmv(len(row_ptr) - 1, _p(row_ptr, i64p), _p(col, i32p), _p(val, f64p),
                             _p(c.view(np.float64), f64p), dt, rtol, max_order, substeps, C.byref(order), C.byref(last)))
    return c, order.value, last.value


def state_norm(orc: Oracle, coeff):
    c = np.ascontiguousarray(coeff, np.complex128)
    out = C.c_double()
    orc.lib.po_state_norm(_p(c.view(np.float64), f64p), c.size, C.byref(out))
    return out.value


def weight_histogram(orc: Oracle, coeff, bins=0):
    """weight_histogram (observables.hpp:123-176) -> dict(support, q50, q90, q99, q9999, tail_exponent, rank, weight)."""
    c = np.ascontiguousarray(coeff, np.complex128)
    cap = c.size if bins == 0 else min(c.size, bins)
    rank, weight = np.zeros(max(cap, 1), np.uint64), np.zeros(max(cap, 1), np.float64)
    h, npts = WeightHist(), C.c_uint64()
    orc._ck(orc.lib.po_weight_histogram(_p(c.view(np.float64), f64p), c.size, bins, C.byref(h), _p(rank, u64p),
                                        _p(weight, f64p), cap, C.byref(npts)))
    k = min(npts.value, cap)
    return dict(support=h.support, q50=h.q50, q90=h.q90, q99=h.q99, q9999=h.q9999, tail_exponent=h.tail_exponent,
                rank=rank[:k].copy(), weight=weight[:k].copy())


def fnv1a64(arr: np.ndarray) -> str:
    """FNV-1a-64 over the raw little-endian bytes (the hash SURVEY App. B quotes)."""
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(arr).view(np.uint8).ravel().tolist():
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def load_reference() -> Oracle:
    return Oracle(REF_LIB)


def load_port() -> Oracle:
    return Oracle(PORT_LIB)
