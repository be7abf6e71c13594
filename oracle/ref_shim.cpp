// ref_shim.cpp -- C-ABI adapter over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle_abi.h).  This file contains no
// algorithm of its own: every po_* entry point forwards to the reference's
// inline functions in /root/reference/proj/include/paces/*.hpp, compiled where
// they lie by oracle/Makefile into oracle/_ref/libpaces_ref.so.  It exists so
// that (a) the restatement in paces_oracle.cpp and the CUDA path can be
// checked against the real reference on flat arrays, and (b) bench.py can time
// the reference's own CPU implementation (cpu_baseline.kind = "reference").
//
// The one piece of orchestration restated here is the body of run()'s loop
// (engine.hpp:333-368): po_run_step() performs step 1 exactly as
// engine.hpp:335-352 and steps >= 2 through the same five calls as
// paces::step (engine.hpp:268-291) so that phases can be timed; po_run_all()
// goes through the reference's own paces::run() and the tests assert both
// produce identical bits.

#include <chrono>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "paces/engine.hpp"

#include "oracle_abi.h"

using namespace paces;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown exception";
        return 2;
    }
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

std::shared_ptr<PackedBasisTable<Word>> make_table(const HamiltonianTermSet& ts, const uint32_t* words,
                                                   uint64_t rows) {
    auto t = std::make_shared<PackedBasisTable<Word>>(ts.layout);
    const std::size_t w = ts.layout.words_per_row;
    t->words.assign(words, words + rows * w);
    t->rows = rows;
    bool sorted = true;
    for (uint64_t i = 1; i < rows && sorted; ++i)
        sorted = row_less<Word>(t->row(i - 1), t->row(i));
    t->sorted = sorted;
    return t;
}

SparseState make_state(const HamiltonianTermSet& ts, const uint32_t* words, const double* coeff,
                       uint64_t rows) {
    SparseState s;
    s.table = make_table(ts, words, rows);
    s.coeff.resize(rows);
    for (uint64_t i = 0; i < rows; ++i) s.coeff[i] = cplx(coeff[2 * i], coeff[2 * i + 1]);
    return s;
}

CsrMatrix make_csr(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val) {
    CsrMatrix a;
    a.n = n;
    a.row_ptr.assign(row_ptr, row_ptr + n + 1);
    const std::size_t nnz = static_cast<std::size_t>(row_ptr[n]);
    a.col.assign(col, col + nnz);
    a.val.assign(val, val + nnz);
    return a;
}
}  // namespace

struct po_model {
    ModelSpec spec;
    HamiltonianTermSet ts;
};
struct po_space {
    EffectiveSpace sp;
};
struct po_run {
    const po_model* model = nullptr;
    RunConfig cfg;
    SparseState state;
    EffectiveSpace space;
    uint64_t steps_done = 0;
    po_phase_times times{};
};

extern "C" {

const char* po_last_error(void) { return g_err.c_str(); }
const char* po_impl_name(void) { return "reference"; }
void po_set_threads(int n) { set_thread_count(n); }
int po_get_threads(void) { return thread_count(); }
uint64_t po_mix_seed(uint64_t x) { return mix_seed(x); }

int po_model_create(int kind, int ndim, const uint32_t* extents, const double* eps, int n_eps,
                    const double* hop, int n_hop, const double* omega, int n_omega, const double* g,
                    int n_g, uint32_t d_pho, po_model** out) {
    return guarded([&] {
        auto m = std::make_unique<po_model>();
        m->spec.kind = kind == 0 ? ModelKind::tight_binding : ModelKind::holstein;
        m->spec.geometry = LatticeGeometry(std::vector<std::uint32_t>(extents, extents + ndim));
        m->spec.holstein.eps.assign(eps, eps + n_eps);
        m->spec.holstein.hop_j.assign(hop, hop + n_hop);
        m->spec.holstein.omega.assign(omega, omega + n_omega);
        m->spec.holstein.g.assign(g, g + n_g);
        m->spec.holstein.d_pho = d_pho;
        m->ts = build_model(m->spec);
        *out = m.release();
    });
}
void po_model_destroy(po_model* m) { delete m; }

int po_model_info(const po_model* m, uint32_t* layout_sites, uint32_t* words_per_row,
                  uint32_t* lattice_sites, uint32_t* n_terms, uint32_t* total_bits) {
    if (layout_sites) *layout_sites = static_cast<uint32_t>(m->ts.layout.site_count());
    if (words_per_row) *words_per_row = m->ts.layout.words_per_row;
    if (lattice_sites) *lattice_sites = m->ts.lattice_sites();
    if (n_terms) *n_terms = static_cast<uint32_t>(m->ts.terms.size());
    if (total_bits) *total_bits = m->ts.layout.total_bits;
    return 0;
}
int po_model_dims(const po_model* m, uint32_t* dims) {
    std::copy(m->ts.layout.dims.begin(), m->ts.layout.dims.end(), dims);
    return 0;
}

int po_pack(const po_model* m, const uint32_t* occ, uint32_t* words) {
    return guarded([&] {
        pack_state<Word>(m->ts.layout, {occ, m->ts.layout.site_count()},
                         {words, m->ts.layout.words_per_row});
    });
}
int po_unpack(const po_model* m, const uint32_t* words, uint32_t* occ) {
    return guarded([&] {
        unpack_state<Word>(m->ts.layout, {words, m->ts.layout.words_per_row},
                           {occ, m->ts.layout.site_count()});
    });
}

int po_apply_terms(const po_model* m, const uint32_t* key, uint32_t* out_keys, double* out_amps,
                   int cap, int* count) {
    return guarded([&] {
        NeighborBuffer nb;
        const std::size_t w = m->ts.layout.words_per_row;
        apply_terms(m->ts, {key, w}, nb);
        if (static_cast<int>(nb.size()) > cap) throw Error("po_apply_terms: output capacity too small");
        std::copy(nb.keys.begin(), nb.keys.end(), out_keys);
        std::copy(nb.amps.begin(), nb.amps.end(), out_amps);
        *count = static_cast<int>(nb.size());
    });
}

int po_grow(const po_model* m, const uint32_t* seeds, uint64_t rows, int order, po_space** out) {
    return guarded([&] {
        auto t = make_table(m->ts, seeds, rows);
        auto s = std::make_unique<po_space>();
        s->sp = grow_subspace(*t, m->ts, order);
        *out = s.release();
    });
}
int po_space_info(const po_space* s, uint64_t* q_true, uint64_t* nnz, uint64_t* q_nom) {
    if (q_true) *q_true = s->sp.q_true();
    if (nnz) *nnz = s->sp.hamiltonian.nnz();
    if (q_nom) *q_nom = s->sp.q_nom;
    return 0;
}
int po_space_get(const po_space* s, uint32_t* words, int64_t* row_ptr, int32_t* col, double* val) {
    const auto& h = s->sp.hamiltonian;
    if (words) std::copy(s->sp.table->words.begin(), s->sp.table->words.end(), words);
    if (row_ptr) std::copy(h.row_ptr.begin(), h.row_ptr.end(), row_ptr);
    if (col) std::copy(h.col.begin(), h.col.end(), col);
    if (val) std::copy(h.val.begin(), h.val.end(), val);
    return 0;
}
void po_space_destroy(po_space* s) { delete s; }

int po_truncate_select(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                       uint64_t q_nom, uint64_t seed, uint32_t* out_words, uint64_t* kept) {
    return guarded([&] {
        SparseState s = make_state(m->ts, words, coeff, rows);
        auto k = truncate_select(s, q_nom, seed);
        std::copy(k.words.begin(), k.words.end(), out_words);
        *kept = k.rows;
    });
}

int po_remap(const po_model* m, const uint32_t* src_words, const double* src_coeff,
             uint64_t src_rows, const uint32_t* dst_words, uint64_t dst_rows, double* out_coeff,
             double* discarded) {
    return guarded([&] {
        SparseState s = make_state(m->ts, src_words, src_coeff, src_rows);
        EffectiveSpace target;
        target.table = make_table(m->ts, dst_words, dst_rows);
        auto [o, d] = remap_state(s, target);
        for (uint64_t i = 0; i < dst_rows; ++i) {
            out_coeff[2 * i] = o.coeff[i].real();
            out_coeff[2 * i + 1] = o.coeff[i].imag();
        }
        *discarded = d;
    });
}

int po_csr_matvec(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                  const double* x, double* y) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, row_ptr, col, val);
        std::span<const cplx> xs{reinterpret_cast<const cplx*>(x), static_cast<std::size_t>(n)};
        std::span<cplx> ys{reinterpret_cast<cplx*>(y), static_cast<std::size_t>(n)};
        csr_matvec(a, xs, ys);
    });
}
int po_csr_expectation(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val,
                       const double* x, double* out) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, row_ptr, col, val);
        std::span<const cplx> xs{reinterpret_cast<const cplx*>(x), static_cast<std::size_t>(n)};
        *out = csr_expectation(a, xs);
    });
}
int po_expmv(int64_t n, const int64_t* row_ptr, const int32_t* col, const double* val, double* c,
             double dt, double rtol, int max_order, int substeps, int* order_used,
             double* last_term_norm) {
    return guarded([&] {
        CsrMatrix a = make_csr(n, row_ptr, col, val);
        std::vector<cplx> v(static_cast<std::size_t>(n));
        std::memcpy(static_cast<void*>(v.data()), c, sizeof(cplx) * v.size());
        PropagatorConfig pc;
        pc.dt = dt;
        pc.rtol = rtol;
        pc.max_order = max_order;
        pc.substeps = substeps;
        ExpmvResult r = expmv(a, v, pc);
        std::memcpy(c, static_cast<const void*>(v.data()), sizeof(cplx) * v.size());
        if (order_used) *order_used = r.order_used;
        if (last_term_norm) *last_term_norm = r.last_term_norm;
    });
}

int po_state_norm(const double* coeff, uint64_t rows, double* out) {
    SparseState s;
    s.coeff.resize(rows);
    std::memcpy(static_cast<void*>(s.coeff.data()), coeff, sizeof(cplx) * rows);
    *out = state_norm(s);
    return 0;
}
int po_exciton_density(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                       double* p) {
    return guarded([&] {
        SparseState s = make_state(m->ts, words, coeff, rows);
        auto d = exciton_density(s, m->ts);
        std::copy(d.p.begin(), d.p.end(), p);
    });
}
int po_dipole_amplitude(const po_model* m, const uint32_t* words, const double* coeff,
                        uint64_t rows, double* amp) {
    return guarded([&] {
        SparseState s = make_state(m->ts, words, coeff, rows);
        cplx a = dipole_amplitude(s, m->ts);
        amp[0] = a.real();
        amp[1] = a.imag();
    });
}
int po_phonon_numbers(const po_model* m, const uint32_t* words, const double* coeff, uint64_t rows,
                      double* n_out) {
    return guarded([&] {
        SparseState s = make_state(m->ts, words, coeff, rows);
        auto n = phonon_numbers(s, m->ts);
        std::copy(n.begin(), n.end(), n_out);
    });
}

int po_weight_histogram(const double* coeff, uint64_t rows, uint64_t bins, po_weight_hist* out,
                        uint64_t* rank, double* weight, uint64_t cap, uint64_t* npts) {
    return guarded([&] {
        SparseState s;  // weight_histogram only reads the coefficients (observables.hpp:123-129)
        s.coeff.resize(rows);
        for (uint64_t i = 0; i < rows; ++i) s.coeff[i] = cplx(coeff[2 * i], coeff[2 * i + 1]);
        const WeightHistogram h = weight_histogram(s, std::size_t(bins));
        out->support = h.support;
        out->q50 = h.q50;
        out->q90 = h.q90;
        out->q99 = h.q99;
        out->q9999 = h.q9999;
        out->tail_exponent = h.tail_exponent;
        *npts = h.rank.size();
        for (uint64_t k = 0; k < h.rank.size() && k < cap; ++k) {
            rank[k] = h.rank[k];
            weight[k] = h.weight[k];
        }
    });
}

static RunConfig to_run_config(const po_model* m, const po_run_cfg* c) {
    RunConfig cfg;
    cfg.model = m->spec;
    cfg.initial.kind = c->init_kind == 0   ? InitialStateSpec::Kind::localized
                       : c->init_kind == 1 ? InitialStateSpec::Kind::optical
                                           : InitialStateSpec::Kind::explicit_list;
    cfg.initial.site = c->init_site;
    const std::size_t ls = m->ts.layout.site_count();
    for (uint64_t e = 0; e < c->n_entries; ++e) {
        std::vector<std::uint32_t> occ(c->entry_occ + e * ls, c->entry_occ + (e + 1) * ls);
        cfg.initial.entries.emplace_back(std::move(occ), cplx(c->entry_amp[2 * e], c->entry_amp[2 * e + 1]));
    }
    cfg.m_init = c->m_init;
    cfg.m = c->m;
    cfg.q_nom = c->q_nom;
    cfg.propagator.dt = c->dt;
    cfg.propagator.rtol = c->rtol;
    cfg.propagator.max_order = c->max_order;
    cfg.propagator.substeps = c->substeps;
    cfg.t_max = c->t_max;
    cfg.seed = c->seed;
    cfg.cadence = c->cadence;
    return cfg;
}

static void fill_diag(const DiagnosticsRecord& r, po_diag* o) {
    o->step = r.step;
    o->t = r.t;
    o->norm_pre = r.norm_pre;
    o->norm_post = r.norm_post;
    o->discarded_weight = r.discarded_weight;
    o->delta_norm_expmv = r.delta_norm_expmv;
    o->energy = r.energy;
    o->q_true = r.q_true;
    o->taylor_order = r.taylor_order;
    o->pad_ = 0;
}

int po_run_begin(const po_model* m, const po_run_cfg* c, po_run** out) {
    return guarded([&] {
        auto r = std::make_unique<po_run>();
        r->model = m;
        r->cfg = to_run_config(m, c);
        auto [state, space] = initialize(r->cfg, m->ts);
        r->state = std::move(state);
        r->space = std::move(space);
        *out = r.release();
    });
}

int po_run_step(po_run* r, po_diag* out) {
    return guarded([&] {
        const std::size_t s = r->steps_done + 1;
        const RunConfig& config = r->cfg;
        const HamiltonianTermSet& terms = r->model->ts;
        DiagnosticsRecord rec;
        const double t0 = now_s();
        if (s == 1) {  // engine.hpp:335-352
            rec.step = s;
            rec.norm_pre = state_norm(r->state);
            rec.norm_post = rec.norm_pre;
            rec.q_true = r->space.q_true();
            const double ta = now_s();
            rec.energy = csr_expectation(r->space.hamiltonian, r->state.coeff);
            const double tb = now_s();
            SparseState psi = r->state;
            auto res = expmv(r->space.hamiltonian, psi.coeff, config.propagator);
            const double tc = now_s();
            rec.taylor_order = res.order_used;
            rec.delta_norm_expmv = state_norm(psi) - rec.norm_post;
            psi.t = r->state.t + config.propagator.dt;
            rec.t = psi.t;
            r->state = std::move(psi);
            r->times.expectation += tb - ta;
            r->times.expmv += tc - tb;
            r->times.spmv_nnz += std::uint64_t(res.order_used) * r->space.hamiltonian.nnz();
        } else {  // same calls, same order as paces::step, engine.hpp:268-291
            rec.step = s;
            rec.norm_pre = state_norm(r->state);
            const double ta = now_s();
            auto kept = truncate_select(r->state, config.q_nom, mix_seed(config.seed + s));
            const double tb = now_s();
            EffectiveSpace next = grow_subspace(kept, terms, config.m);
            require_memory(next.q_true() * sizeof(cplx) * 4, "state vectors");
            const double tc = now_s();
            auto [psi, discarded] = remap_state(r->state, next);
            const double td = now_s();
            rec.discarded_weight = discarded;
            rec.norm_post = state_norm(psi);
            rec.q_true = next.q_true();
            rec.energy = csr_expectation(next.hamiltonian, psi.coeff);
            const double te = now_s();
            auto res = expmv(next.hamiltonian, psi.coeff, config.propagator);
            const double tf = now_s();
            rec.taylor_order = res.order_used;
            rec.delta_norm_expmv = state_norm(psi) - rec.norm_post;
            psi.t = r->state.t + config.propagator.dt;
            rec.t = psi.t;
            r->state = std::move(psi);
            r->space = std::move(next);
            r->times.select += tb - ta;
            r->times.grow += tc - tb;
            r->times.remap += td - tc;
            r->times.expectation += te - td;
            r->times.expmv += tf - te;
            r->times.spmv_nnz += std::uint64_t(res.order_used) * r->space.hamiltonian.nnz();
        }
        r->times.total += now_s() - t0;
        r->steps_done = s;
        if (out) fill_diag(rec, out);
    });
}

int po_run_info(const po_run* r, uint64_t* rows, uint64_t* nnz, double* t, uint64_t* steps_done) {
    if (rows) *rows = r->state.table ? r->state.table->rows : 0;
    if (nnz) *nnz = r->space.hamiltonian.nnz();
    if (t) *t = r->state.t;
    if (steps_done) *steps_done = r->steps_done;
    return 0;
}
int po_run_state(const po_run* r, uint32_t* words, double* coeff) {
    if (words) std::copy(r->state.table->words.begin(), r->state.table->words.end(), words);
    if (coeff)
        std::memcpy(coeff, static_cast<const void*>(r->state.coeff.data()),
                    sizeof(cplx) * r->state.coeff.size());
    return 0;
}
int po_run_csr(const po_run* r, int64_t* row_ptr, int32_t* col, double* val) {
    const auto& h = r->space.hamiltonian;
    if (row_ptr) std::copy(h.row_ptr.begin(), h.row_ptr.end(), row_ptr);
    if (col) std::copy(h.col.begin(), h.col.end(), col);
    if (val) std::copy(h.val.begin(), h.val.end(), val);
    return 0;
}
int po_run_observe(const po_run* r, double* norm, double* energy, double* rmsd_out, double* xbar,
                   double* amp, double* density) {
    return guarded([&] {
        ObservablesRow row = detail::observe(r->state, r->space, r->model->ts);
        if (norm) *norm = row.norm;
        if (energy) *energy = row.energy;
        if (rmsd_out) *rmsd_out = row.rmsd;
        if (xbar) *xbar = row.xbar;
        if (amp) {
            amp[0] = row.amp.real();
            amp[1] = row.amp.imag();
        }
        if (density) std::copy(row.density.begin(), row.density.end(), density);
    });
}
void po_run_destroy(po_run* r) { delete r; }

int po_run_all(const po_model* m, const po_run_cfg* c, po_diag* diag, uint64_t cap, uint64_t* n_diag,
               po_run** final_out) {
    return guarded([&] {
        auto r = std::make_unique<po_run>();
        r->model = m;
        r->cfg = to_run_config(m, c);
        RunResult res = run(r->cfg, m->ts);
        const uint64_t n = std::min<uint64_t>(cap, res.diagnostics.size());
        for (uint64_t i = 0; i < n; ++i) fill_diag(res.diagnostics[i], diag + i);
        if (n_diag) *n_diag = res.diagnostics.size();
        r->state = std::move(res.final_state);
        r->space = std::move(res.final_space);
        r->steps_done = res.diagnostics.size();
        if (!res.error.empty()) {
            g_err = res.error;
            if (final_out) *final_out = r.release();
            throw Error(g_err);
        }
        if (final_out) *final_out = r.release();
    });
}

int po_run_times(const po_run* r, po_phase_times* out) {
    *out = r->times;
    return 0;
}

}  // extern "C"
