// paces_b200.hpp -- source-compatible C++ host shim over the C ABI (include/paces_b200.h).
//
// Include AFTER the reference headers (it uses their types: paces::SparseState, EffectiveSpace,
// CsrMatrix, HamiltonianTermSet, RunConfig, DiagnosticsRecord, ... from proj/include/paces/).  It
// provides, in namespace paces::b200, callables with EXACTLY the reference signatures for every function
// on the adapt-evolve-truncate path, each forwarding to libpaces_b200.so:
//
//   truncate_select   engine.hpp:107      grow_subspace    subspace.hpp:195     remap_state  subspace.hpp:281
//   csr_matvec        subspace.hpp:35     csr_expectation  subspace.hpp:46      expmv        propagator.hpp:52
//   state_norm        subspace.hpp:91     exciton_density  observables.hpp:26   dipole_amplitude  observables.hpp:99
//   phonon_numbers    observables.hpp:84  weight_histogram observables.hpp:123  initialize   engine.hpp:235
//   step              engine.hpp:268      run              engine.hpp:318 (both overloads)
//   resume            (new) continue a run from a checkpoint file written by write_checkpoint (io.hpp:77-144)
//
// Drop-in use, no call-site edit: put PACES_B200_DROP_IN; at the top of a function body (or any block).  From there on
// the unqualified names above mean the B200 versions -- they are function OBJECTS, so the block-scope using-declarations
// both hide the reference's functions and switch off argument-dependent lookup, and `run(cfg, terms)`,
// `truncate_select(state, q, seed)`, ... compile unchanged.  (tests/cpp/acceptance_b200.cpp runs the reference's
// acceptance criteria that way.)  The GPU context behind a call is found from the HamiltonianTermSet (one cached
// Device per distinct model and thread); functions whose reference signature carries no terms use the model-less
// operators or the Device of the model used last.  Every callable also accepts an explicit `Device&` first.
// Failures rethrow paces::Error with the reference's text.  run() keeps (state, space) resident in HBM across
// steps and only downloads at the observation cadence and at the end.
#pragma once

#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "paces/engine.hpp"
#include "paces/io.hpp"  // read_checkpoint (resume)
#include "paces_b200.h"

namespace paces::b200 {

/// RAII owner of one pb200_ctx bound to one HamiltonianTermSet.
class Device {
public:
    explicit Device(const HamiltonianTermSet& terms, int device = 0) {
        if (pb200_ctx_create(device, &ctx_) != PB200_OK) throw Error(pb200_last_error(nullptr));
        set_model(terms);
        words_ = terms.layout.words_per_row;
    }
    /// model-less context: the operators that need no model (csr_matvec, csr_expectation, expmv, state_norm)
    struct NoModel {};
    explicit Device(NoModel, int device = 0) {
        if (pb200_ctx_create(device, &ctx_) != PB200_OK) throw Error(pb200_last_error(nullptr));
    }
    ~Device() { pb200_ctx_destroy(ctx_); }
    std::uint32_t words_per_row() const { return words_; }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    pb200_ctx* get() const { return ctx_; }
    void check(int rc) const {
        if (rc != PB200_OK) throw Error(pb200_last_error(ctx_));
    }

private:
    /// Recovers the ModelSpec parameters from the term list (build_model is injective on them up to
    /// zero-valued parameters, which produce no term: lattice_models.hpp:160-171).
    void set_model(const HamiltonianTermSet& ts) {
        if (!ts.has_exciton_register()) throw Error("dynamics runs support exciton models (tb, holstein) only");
        const std::uint32_t n = ts.lattice_sites();
        const auto bonds = ts.geometry.bonds();
        std::vector<double> eps(n, 0.0), omega(n, 0.0), g(n, 0.0), hop(bonds.size(), 0.0);
        for (const Term& t : ts.terms) {
            switch (t.kind) {
                case TermKind::diagonal_exciton: eps[t.a] = t.amp; break;
                case TermKind::phonon_number: omega[t.a] = t.amp; break;
                case TermKind::vibronic_ladder: g[t.a] = t.amp; break;
                case TermKind::hop:
                    for (std::size_t b = 0; b < bonds.size(); ++b)
                        if (bonds[b].first == t.a && bonds[b].second == t.b) hop[b] = t.amp;
                    break;
                default: throw Error("unsupported term kind for the B200 path");
            }
        }
        std::uint32_t ext[3] = {ts.geometry.extents[0], ts.geometry.extents[1], ts.geometry.extents[2]};
        const int kind = ts.kind == ModelKind::holstein ? 1 : 0;
        check(pb200_model_set(ctx_, kind, ts.geometry.ndim, ext, eps.data(), int(n), hop.data(), int(hop.size()),
                              omega.data(), int(n), g.data(), int(n), ts.d_pho));
    }
    pb200_ctx* ctx_ = nullptr;
    std::uint32_t words_ = 0;
};

namespace detail {

/// One cached Device per distinct model and thread (key: the term list and layout, bit for bit).
inline std::string fingerprint(const HamiltonianTermSet& ts) {
    std::string k;
    auto put = [&k](const void* p, std::size_t n) { k.append(static_cast<const char*>(p), n); };
    const int kind = int(ts.kind), ndim = ts.geometry.ndim;
    put(&kind, sizeof kind);
    put(&ndim, sizeof ndim);
    put(ts.geometry.extents.data(), sizeof(ts.geometry.extents[0]) * 3);
    put(&ts.d_pho, sizeof ts.d_pho);
    for (const Term& t : ts.terms) {
        const int tk = int(t.kind);
        put(&tk, sizeof tk);
        put(&t.a, sizeof t.a);
        put(&t.b, sizeof t.b);
        put(&t.amp, sizeof t.amp);
    }
    return k;
}
inline Device*& last_device_slot() {
    thread_local Device* last = nullptr;
    return last;
}
inline Device& device_for(const HamiltonianTermSet& ts) {
    thread_local std::map<std::string, std::unique_ptr<Device>> cache;
    auto& slot = cache[fingerprint(ts)];
    if (!slot) slot = std::make_unique<Device>(ts);
    last_device_slot() = slot.get();
    return *slot;
}
/// For reference signatures that carry no HamiltonianTermSet but need the key width: the model used last.
inline Device& last_device(std::uint32_t words_per_row, const char* who) {
    Device* d = last_device_slot();
    if (!d || d->words_per_row() != words_per_row)
        throw Error(std::string(who) +
                    ": no B200 context for this key layout yet -- call a function that carries the HamiltonianTermSet "
                    "first (grow_subspace, initialize, step, run) or pass a paces::b200::Device explicitly");
    return *d;
}
inline Device& plain_device() {
    if (Device* d = last_device_slot()) return *d;
    thread_local Device bare{Device::NoModel{}};
    return bare;
}

inline const double* reim(const std::vector<cplx>& v) { return reinterpret_cast<const double*>(v.data()); }
inline double* reim(std::vector<cplx>& v) { return reinterpret_cast<double*>(v.data()); }

inline pb200_run_cfg to_cfg(const RunConfig& c, std::vector<std::uint32_t>& occ, std::vector<double>& amp) {
    pb200_run_cfg r{};
    r.init_kind = int(c.initial.kind);
    r.init_site = c.initial.site;
    r.m_init = c.m_init;
    r.m = c.m;
    r.q_nom = c.q_nom;
    r.dt = c.propagator.dt;
    r.rtol = c.propagator.rtol;
    r.max_order = c.propagator.max_order;
    r.substeps = c.propagator.substeps;
    r.t_max = c.t_max;
    r.seed = c.seed;
    r.cadence = c.cadence;
    for (const auto& [o, a] : c.initial.entries) {
        occ.insert(occ.end(), o.begin(), o.end());
        amp.push_back(a.real());
        amp.push_back(a.imag());
    }
    r.n_entries = c.initial.entries.size();
    r.entry_occ = occ.data();
    r.entry_amp = amp.data();
    return r;
}

inline DiagnosticsRecord to_record(const pb200_diag& d) {
    DiagnosticsRecord r;
    r.step = d.step;
    r.t = d.t;
    r.norm_pre = d.norm_pre;
    r.norm_post = d.norm_post;
    r.discarded_weight = d.discarded_weight;
    r.delta_norm_expmv = d.delta_norm_expmv;
    r.energy = d.energy;
    r.q_true = d.q_true;
    r.taylor_order = d.taylor_order;
    return r;
}

/// Downloads the resident (state, space) pair in the reference's types.
inline std::pair<SparseState, EffectiveSpace> download(const Device& dev, const HamiltonianTermSet& terms, int order,
                                                       std::size_t q_nom) {
    std::uint64_t rows = 0, nnz = 0, steps = 0;
    double t = 0;
    dev.check(pb200_run_info(dev.get(), &rows, &nnz, &t, &steps));
    auto table = std::make_shared<PackedBasisTable<Word>>(terms.layout);
    table->rows = rows;
    table->words.resize(rows * terms.layout.words_per_row);
    table->sorted = true;
    SparseState st;
    st.coeff.resize(rows);
    st.t = t;
    dev.check(pb200_run_state(dev.get(), table->words.data(), reim(st.coeff)));
    EffectiveSpace sp;
    sp.hamiltonian.n = std::int64_t(rows);
    sp.hamiltonian.row_ptr.resize(rows + 1);
    sp.hamiltonian.col.resize(nnz);
    sp.hamiltonian.val.resize(nnz);
    dev.check(pb200_run_csr(dev.get(), sp.hamiltonian.row_ptr.data(), sp.hamiltonian.col.data(),
                            sp.hamiltonian.val.data()));
    sp.table = table;
    sp.neighbor_order = order;
    std::uint64_t seeds = q_nom;
    dev.check(pb200_space_info(dev.get(), nullptr, nullptr, &seeds));  // EffectiveSpace::q_nom = seed count
    sp.q_nom = seeds;
    st.table = table;
    return {std::move(st), std::move(sp)};
}

}  // namespace detail

namespace impl {  // the work, with an explicit Device; the public callables below forward here

// ---- stand-alone operators (host data in, host data out) ---------------------------------------------------------

inline PackedBasisTable<Word> truncate_select(const Device& dev, const SparseState& state, std::size_t q_nom,
                                              std::uint64_t seed) {
    if (q_nom < 1) throw Error("truncate_select: q_nom must be >= 1");
    if (!state.table || !state.table->sorted) throw Error("truncate_select: state table must be sorted");
    const auto& table = *state.table;
    PackedBasisTable<Word> out(table.layout);
    out.words.resize(std::min<std::size_t>(table.rows, q_nom) * table.layout.words_per_row);
    std::uint64_t kept = 0;
    dev.check(pb200_truncate_select(dev.get(), table.words.data(), detail::reim(state.coeff), table.rows, q_nom, seed,
                                    out.words.data(), &kept));
    out.rows = kept;
    out.words.resize(kept * table.layout.words_per_row);
    out.sorted = true;
    return out;
}

inline EffectiveSpace grow_subspace(const Device& dev, const PackedBasisTable<Word>& seeds,
                                    const HamiltonianTermSet& terms, int m) {
    if (seeds.rows == 0) throw Error("grow_subspace: empty seed set");
    if (!seeds.sorted) throw Error("grow_subspace: seed keys must be sorted");
    if (m < 0) throw Error("grow_subspace: neighbor order must be >= 0");
    if (!(seeds.layout == terms.layout)) throw Error("grow_subspace: layout mismatch");
    std::uint64_t q = 0, z = 0;
    dev.check(pb200_grow(dev.get(), seeds.words.data(), seeds.rows, m, &q, &z));
    auto table = std::make_shared<PackedBasisTable<Word>>(terms.layout);
    table->rows = q;
    table->words.resize(q * terms.layout.words_per_row);
    table->sorted = true;
    EffectiveSpace sp;
    sp.hamiltonian.n = std::int64_t(q);
    sp.hamiltonian.row_ptr.resize(q + 1);
    sp.hamiltonian.col.resize(z);
    sp.hamiltonian.val.resize(z);
    dev.check(pb200_space_get(dev.get(), table->words.data(), sp.hamiltonian.row_ptr.data(),
                              sp.hamiltonian.col.data(), sp.hamiltonian.val.data()));
    sp.table = table;
    sp.neighbor_order = m;
    sp.q_nom = seeds.rows;
    return sp;
}

inline std::pair<SparseState, double> remap_state(const Device& dev, const SparseState& state,
                                                  const EffectiveSpace& target) {
    if (!state.table || !state.table->sorted) throw Error("remap: state table must be sorted");
    SparseState out;
    out.table = target.table;
    out.coeff.assign(target.table->rows, cplx(0, 0));
    out.t = state.t;
    double discarded = 0;
    dev.check(pb200_remap(dev.get(), state.table->words.data(), detail::reim(state.coeff), state.table->rows,
                          target.table->words.data(), target.table->rows, detail::reim(out.coeff), &discarded));
    return {std::move(out), discarded};
}

inline void csr_matvec(const Device& dev, const CsrMatrix& a, std::span<const cplx> x, std::span<cplx> y) {
    dev.check(pb200_csr_matvec(dev.get(), a.n, a.row_ptr.data(), a.col.data(), a.val.data(),
                               reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())));
}

inline double csr_expectation(const Device& dev, const CsrMatrix& a, std::span<const cplx> x) {
    double out = 0;
    dev.check(pb200_csr_expectation(dev.get(), a.n, a.row_ptr.data(), a.col.data(), a.val.data(),
                                    reinterpret_cast<const double*>(x.data()), &out));
    return out;
}

inline ExpmvResult expmv(const Device& dev, const CsrMatrix& h, std::vector<cplx>& c, const PropagatorConfig& cfg) {
    cfg.validate();
    if (static_cast<std::int64_t>(c.size()) != h.n) throw Error("expmv: dimension mismatch");
    ExpmvResult res;
    dev.check(pb200_expmv(dev.get(), h.n, h.row_ptr.data(), h.col.data(), h.val.data(), detail::reim(c), cfg.dt,
                          cfg.rtol, cfg.max_order, cfg.substeps, &res.order_used, &res.last_term_norm));
    return res;
}

inline double state_norm(const Device& dev, const SparseState& s) {
    double out = 0;
    dev.check(pb200_state_norm(dev.get(), detail::reim(s.coeff), s.coeff.size(), &out));
    return out;
}

inline ExcitonDensity exciton_density(const Device& dev, const SparseState& state, const HamiltonianTermSet& terms) {
    ExcitonDensity d;
    d.p.assign(terms.lattice_sites(), 0.0);
    dev.check(pb200_exciton_density(dev.get(), state.table->words.data(), detail::reim(state.coeff),
                                    state.table->rows, d.p.data()));
    return d;
}

inline cplx dipole_amplitude(const Device& dev, const SparseState& state, const HamiltonianTermSet&) {
    double a[2] = {0, 0};
    dev.check(pb200_dipole_amplitude(dev.get(), state.table->words.data(), detail::reim(state.coeff),
                                     state.table->rows, a));
    return {a[0], a[1]};
}

inline std::vector<double> phonon_numbers(const Device& dev, const SparseState& state, const HamiltonianTermSet& terms) {
    if (terms.kind != ModelKind::holstein) throw Error("phonon numbers: not a Holstein model");
    std::vector<double> n(terms.lattice_sites(), 0.0);
    dev.check(pb200_phonon_numbers(dev.get(), state.table->words.data(), detail::reim(state.coeff), state.table->rows,
                                   n.data()));
    return n;
}

/// weight_histogram (observables.hpp:123-176): the GPU sorts the weights, the serial sums are replayed on the host,
/// so every field equals the reference's.
inline WeightHistogram weight_histogram(const Device& dev, const SparseState& state, std::size_t bins = 0) {
    const std::size_t cap = (bins == 0) ? state.coeff.size() : std::min<std::size_t>(bins, state.coeff.size());
    std::vector<std::uint64_t> rank(std::max<std::size_t>(cap, 1));
    std::vector<double> weight(std::max<std::size_t>(cap, 1));
    pb200_weight_hist h{};
    std::uint64_t npts = 0;
    dev.check(pb200_weight_histogram(dev.get(), detail::reim(state.coeff), state.coeff.size(), bins, &h, rank.data(),
                                     weight.data(), cap, &npts));
    WeightHistogram out;
    out.support = h.support;
    out.q50 = h.q50;
    out.q90 = h.q90;
    out.q99 = h.q99;
    out.q9999 = h.q9999;
    out.tail_exponent = h.tail_exponent;
    const std::size_t k = std::min<std::size_t>(npts, cap);
    out.rank.assign(rank.begin(), rank.begin() + k);
    out.weight.assign(weight.begin(), weight.begin() + k);
    return out;
}

// ---- initialize / step / run -------------------------------------------------------------------------------------

inline std::pair<SparseState, EffectiveSpace> initialize(const Device& dev, const RunConfig& config,
                                                         const HamiltonianTermSet& terms) {
    config.validate();
    std::vector<std::uint32_t> occ;
    std::vector<double> amp;
    pb200_run_cfg c = detail::to_cfg(config, occ, amp);
    dev.check(pb200_run_begin(dev.get(), &c));
    std::size_t nseeds = config.initial.kind == InitialStateSpec::Kind::optical
                             ? terms.lattice_sites()
                             : (config.initial.kind == InitialStateSpec::Kind::localized ? 1 : config.initial.entries.size());
    return detail::download(dev, terms, config.m_init, nseeds);
}

/// paces::step on host data: uploads `state`, runs the device step, downloads StepOutput.
inline StepOutput step(const Device& dev, const SparseState& state, const EffectiveSpace& space,
                       const RunConfig& config, const HamiltonianTermSet& terms, std::size_t step_index) {
    (void)space;  // superseded by the regrowth, as in the reference
    if (!state.table || !state.table->sorted) throw Error("truncate_select: state table must be sorted");
    std::vector<std::uint32_t> occ;
    std::vector<double> amp;
    pb200_run_cfg c = detail::to_cfg(config, occ, amp);
    pb200_diag d{};
    std::uint64_t rows = 0, nnz = 0;
    dev.check(pb200_step(dev.get(), &c, step_index, state.table->words.data(), detail::reim(state.coeff),
                         state.table->rows, state.t, &d, &rows, &nnz));
    auto [psi, next] = detail::download(dev, terms, config.m, std::min<std::size_t>(config.q_nom, state.table->rows));
    return {std::move(psi), std::move(next), detail::to_record(d)};
}

/// paces::run with the state resident on the device between steps (engine.hpp:318-375).  `from`: continue from
/// this state (a checkpoint) instead of initialize(); the step index resumes at round(t / dt) + 1.
inline RunResult run(const Device& dev, const RunConfig& config, const HamiltonianTermSet& terms,
                     const SparseState* from = nullptr) {
    config.validate();
    RunResult result;
    std::vector<std::uint32_t> occ;
    std::vector<double> amp;
    pb200_run_cfg c = detail::to_cfg(config, occ, amp);
    std::size_t first_step = 1;
    if (from) {
        if (!from->table || !from->table->sorted) throw Error("resume: checkpoint table must be sorted");
        if (!(from->table->layout == terms.layout)) throw Error("resume: checkpoint layout does not match the model");
        const std::uint64_t done = std::uint64_t(std::llround(from->t / config.propagator.dt));
        dev.check(pb200_run_load_state(dev.get(), &c, from->table->words.data(), detail::reim(from->coeff),
                                       from->table->rows, from->t, done));
        first_step = std::size_t(done) + 1;
    } else {
        dev.check(pb200_run_begin(dev.get(), &c));
    }
    std::uint64_t rows = 0;
    dev.check(pb200_run_info(dev.get(), &rows, nullptr, nullptr, nullptr));
    if (!from && rows > config.q_nom)
        result.warnings.push_back("initial effective space (q_true=" + std::to_string(rows) + ") exceeds q_nom=" +
                                  std::to_string(config.q_nom) +
                                  "; memory is bounded by the initial growth until truncation binds");
    auto observe = [&]() {
        ObservablesRow row;
        row.density.assign(terms.lattice_sites(), 0.0);
        double a[2] = {0, 0};
        dev.check(pb200_run_observe(dev.get(), &row.norm, &row.energy, &row.rmsd, &row.xbar, a, row.density.data()));
        dev.check(pb200_run_info(dev.get(), nullptr, nullptr, &row.t, nullptr));
        row.amp = cplx(a[0], a[1]);
        return row;
    };
    auto histogram = [&]() {
        // weight_histogram (observables.hpp:123-176) of the resident state: sorted on the GPU, no state download
        std::uint64_t nrows = 0, npts = 0;
        double t_now = 0;
        dev.check(pb200_run_info(dev.get(), &nrows, nullptr, &t_now, nullptr));
        const std::size_t bins = config.histogram_bins;
        const std::size_t cap = (bins == 0) ? nrows : std::min<std::size_t>(bins, nrows);
        std::vector<std::uint64_t> rank(std::max<std::size_t>(cap, 1));
        std::vector<double> weight(std::max<std::size_t>(cap, 1));
        pb200_weight_hist h{};
        dev.check(pb200_run_weight_histogram(dev.get(), bins, &h, rank.data(), weight.data(), cap, &npts));
        WeightHistogram wh;
        wh.support = h.support;
        wh.q50 = h.q50;
        wh.q90 = h.q90;
        wh.q99 = h.q99;
        wh.q9999 = h.q9999;
        wh.tail_exponent = h.tail_exponent;
        const std::size_t k = std::min<std::size_t>(npts, cap);
        wh.rank.assign(rank.begin(), rank.begin() + k);
        wh.weight.assign(weight.begin(), weight.begin() + k);
        result.histograms.emplace_back(t_now, std::move(wh));
    };
    result.trajectory.push_back(observe());
    if (config.emit_histograms) histogram();
    const std::size_t nsteps = config.step_count();
    for (std::size_t s = first_step; s <= nsteps; ++s) {
        pb200_diag d{};
        if (pb200_run_step(dev.get(), &d) != PB200_OK) {
            result.error = "step " + std::to_string(s) + ": " + pb200_last_error(dev.get());
            break;
        }
        result.diagnostics.push_back(detail::to_record(d));
        if (s % config.cadence == 0 || s == nsteps) {
            result.trajectory.push_back(observe());
            if (config.emit_histograms) histogram();
        }
    }
    std::uint64_t steps_done = 0;
    dev.check(pb200_run_info(dev.get(), nullptr, nullptr, nullptr, &steps_done));
    auto [st, sp] = detail::download(dev, terms, steps_done > 1 ? config.m : config.m_init, config.q_nom);
    result.final_state = std::move(st);
    result.final_space = std::move(sp);
    return result;
}

}  // namespace impl

// ------------------------------------------------------------------------------------------------------------------
// The public callables: function objects, one per reference function, overloaded on (explicit Device, ...) and on the
// reference's exact signature.
// ------------------------------------------------------------------------------------------------------------------
inline constexpr struct truncate_select_fn {
    PackedBasisTable<Word> operator()(const Device& dev, const SparseState& state, std::size_t q_nom,
                                      std::uint64_t seed) const {
        return impl::truncate_select(dev, state, q_nom, seed);
    }
    PackedBasisTable<Word> operator()(const SparseState& state, std::size_t q_nom, std::uint64_t seed) const {  // engine.hpp:107
        if (q_nom < 1) throw Error("truncate_select: q_nom must be >= 1");
        if (!state.table || !state.table->sorted) throw Error("truncate_select: state table must be sorted");
        return impl::truncate_select(detail::last_device(state.table->layout.words_per_row, "truncate_select"), state,
                                     q_nom, seed);
    }
} truncate_select{};

inline constexpr struct grow_subspace_fn {
    EffectiveSpace operator()(const Device& dev, const PackedBasisTable<Word>& seeds, const HamiltonianTermSet& terms,
                              int m) const {
        return impl::grow_subspace(dev, seeds, terms, m);
    }
    EffectiveSpace operator()(const PackedBasisTable<Word>& seeds, const HamiltonianTermSet& terms, int m) const {  // subspace.hpp:195
        return impl::grow_subspace(detail::device_for(terms), seeds, terms, m);
    }
} grow_subspace{};

inline constexpr struct remap_state_fn {
    std::pair<SparseState, double> operator()(const Device& dev, const SparseState& state,
                                              const EffectiveSpace& target) const {
        return impl::remap_state(dev, state, target);
    }
    std::pair<SparseState, double> operator()(const SparseState& state, const EffectiveSpace& target) const {  // subspace.hpp:281
        if (!state.table || !state.table->sorted) throw Error("remap: state table must be sorted");
        return impl::remap_state(detail::last_device(state.table->layout.words_per_row, "remap_state"), state, target);
    }
} remap_state{};

inline constexpr struct csr_matvec_fn {
    void operator()(const Device& dev, const CsrMatrix& a, std::span<const cplx> x, std::span<cplx> y) const {
        impl::csr_matvec(dev, a, x, y);
    }
    void operator()(const CsrMatrix& a, std::span<const cplx> x, std::span<cplx> y) const {  // subspace.hpp:35
        impl::csr_matvec(detail::plain_device(), a, x, y);
    }
} csr_matvec{};

inline constexpr struct csr_expectation_fn {
    double operator()(const Device& dev, const CsrMatrix& a, std::span<const cplx> x) const {
        return impl::csr_expectation(dev, a, x);
    }
    double operator()(const CsrMatrix& a, std::span<const cplx> x) const {  // subspace.hpp:46
        return impl::csr_expectation(detail::plain_device(), a, x);
    }
} csr_expectation{};

inline constexpr struct expmv_fn {
    ExpmvResult operator()(const Device& dev, const CsrMatrix& h, std::vector<cplx>& c, const PropagatorConfig& cfg) const {
        return impl::expmv(dev, h, c, cfg);
    }
    ExpmvResult operator()(const CsrMatrix& h, std::vector<cplx>& c, const PropagatorConfig& cfg) const {  // propagator.hpp:52
        return impl::expmv(detail::plain_device(), h, c, cfg);
    }
} expmv{};

inline constexpr struct state_norm_fn {
    double operator()(const Device& dev, const SparseState& s) const { return impl::state_norm(dev, s); }
    double operator()(const SparseState& s) const { return impl::state_norm(detail::plain_device(), s); }  // subspace.hpp:91
} state_norm{};

inline constexpr struct exciton_density_fn {
    ExcitonDensity operator()(const Device& dev, const SparseState& state, const HamiltonianTermSet& terms) const {
        return impl::exciton_density(dev, state, terms);
    }
    ExcitonDensity operator()(const SparseState& state, const HamiltonianTermSet& terms) const {  // observables.hpp:26
        return impl::exciton_density(detail::device_for(terms), state, terms);
    }
} exciton_density{};

inline constexpr struct dipole_amplitude_fn {
    cplx operator()(const Device& dev, const SparseState& state, const HamiltonianTermSet& terms) const {
        return impl::dipole_amplitude(dev, state, terms);
    }
    cplx operator()(const SparseState& state, const HamiltonianTermSet& terms) const {  // observables.hpp:99
        return impl::dipole_amplitude(detail::device_for(terms), state, terms);
    }
} dipole_amplitude{};

inline constexpr struct phonon_numbers_fn {
    std::vector<double> operator()(const Device& dev, const SparseState& state, const HamiltonianTermSet& terms) const {
        return impl::phonon_numbers(dev, state, terms);
    }
    std::vector<double> operator()(const SparseState& state, const HamiltonianTermSet& terms) const {  // observables.hpp:84
        return impl::phonon_numbers(detail::device_for(terms), state, terms);
    }
} phonon_numbers{};

inline constexpr struct weight_histogram_fn {
    WeightHistogram operator()(const Device& dev, const SparseState& state, std::size_t bins = 0) const {
        return impl::weight_histogram(dev, state, bins);
    }
    WeightHistogram operator()(const SparseState& state, std::size_t bins = 0) const {  // observables.hpp:123
        return impl::weight_histogram(detail::plain_device(), state, bins);
    }
} weight_histogram{};

inline constexpr struct initialize_fn {
    std::pair<SparseState, EffectiveSpace> operator()(const Device& dev, const RunConfig& config,
                                                      const HamiltonianTermSet& terms) const {
        return impl::initialize(dev, config, terms);
    }
    std::pair<SparseState, EffectiveSpace> operator()(const RunConfig& config, const HamiltonianTermSet& terms) const {  // engine.hpp:235
        return impl::initialize(detail::device_for(terms), config, terms);
    }
} initialize{};

inline constexpr struct step_fn {
    StepOutput operator()(const Device& dev, const SparseState& state, const EffectiveSpace& space, const RunConfig& config,
                          const HamiltonianTermSet& terms, std::size_t step_index) const {
        return impl::step(dev, state, space, config, terms, step_index);
    }
    StepOutput operator()(const SparseState& state, const EffectiveSpace& space, const RunConfig& config,
                          const HamiltonianTermSet& terms, std::size_t step_index) const {  // engine.hpp:268
        return impl::step(detail::device_for(terms), state, space, config, terms, step_index);
    }
} step{};

inline constexpr struct run_fn {
    RunResult operator()(const Device& dev, const RunConfig& config, const HamiltonianTermSet& terms) const {
        return impl::run(dev, config, terms);
    }
    RunResult operator()(const RunConfig& config, const HamiltonianTermSet& terms) const {  // engine.hpp:318
        return impl::run(detail::device_for(terms), config, terms);
    }
    RunResult operator()(const RunConfig& config) const {  // engine.hpp:371-375
        config.validate();
        const HamiltonianTermSet terms = build_model(config.model);
        return impl::run(detail::device_for(terms), config, terms);
    }
} run{};

/// Continues a run from a checkpoint file (io.hpp:101-144 read side): the trajectory / diagnostics of the result start
/// at the checkpoint's time; the remaining steps are exactly those the uninterrupted run would have taken.
inline constexpr struct resume_fn {
    RunResult operator()(const Device& dev, const std::string& checkpoint_path, const RunConfig& config,
                         const HamiltonianTermSet& terms) const {
        const SparseState from = read_checkpoint(checkpoint_path);
        return impl::run(dev, config, terms, &from);
    }
    RunResult operator()(const std::string& checkpoint_path, const RunConfig& config, const HamiltonianTermSet& terms) const {
        const SparseState from = read_checkpoint(checkpoint_path);
        return impl::run(detail::device_for(terms), config, terms, &from);
    }
} resume{};

/// One line at the top of a block: the unqualified hot-path names mean the B200 versions from here on (see header).
#define PACES_B200_DROP_IN                                                                                          \
    using paces::b200::truncate_select; using paces::b200::grow_subspace; using paces::b200::remap_state;         \
    using paces::b200::csr_matvec; using paces::b200::csr_expectation; using paces::b200::expmv;                   \
    using paces::b200::state_norm; using paces::b200::exciton_density; using paces::b200::dipole_amplitude;       \
    using paces::b200::phonon_numbers; using paces::b200::weight_histogram; using paces::b200::initialize;        \
    using paces::b200::step; using paces::b200::run; using paces::b200::resume

}  // namespace paces::b200
