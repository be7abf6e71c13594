// paces_b200.hpp -- source-compatible C++ host shim over the C ABI (include/paces_b200.h).
//
// Include AFTER the reference headers (it uses their types: paces::SparseState, EffectiveSpace,
// CsrMatrix, HamiltonianTermSet, RunConfig, DiagnosticsRecord, ... from proj/include/paces/).  It
// provides, in namespace paces::b200, functions with EXACTLY the reference signatures for every function
// on the adapt-evolve-truncate path, each forwarding to libpaces_b200.so:
//
//   truncate_select   engine.hpp:107      grow_subspace    subspace.hpp:195     remap_state  subspace.hpp:281
//   csr_matvec        subspace.hpp:35     csr_expectation  subspace.hpp:46      expmv        propagator.hpp:52
//   state_norm        subspace.hpp:91     exciton_density  observables.hpp:26   dipole_amplitude  observables.hpp:99
//   phonon_numbers    observables.hpp:84  initialize       engine.hpp:235       step         engine.hpp:268
//   run               engine.hpp:318
//
// A maintainer switches a call site by replacing `paces::step(...)` with `paces::b200::step(...)` (or with a
// using-declaration); failures rethrow paces::Error with the reference's text.  run() keeps (state, space)
// resident in HBM across steps and only downloads at the observation cadence and at the end.
#pragma once

#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "paces_b200.h"

namespace paces::b200 {

/// RAII owner of one pb200_ctx bound to one HamiltonianTermSet.
class Device {
public:
    explicit Device(const HamiltonianTermSet& terms, int device = 0) {
        if (pb200_ctx_create(device, &ctx_) != PB200_OK) throw Error(pb200_last_error(nullptr));
        set_model(terms);
    }
    ~Device() { pb200_ctx_destroy(ctx_); }
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
};

namespace detail {

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

/// paces::run with the state resident on the device between steps (engine.hpp:318-375).
inline RunResult run(const RunConfig& config, const HamiltonianTermSet& terms, int device = 0) {
    config.validate();
    RunResult result;
    Device dev(terms, device);
    std::vector<std::uint32_t> occ;
    std::vector<double> amp;
    pb200_run_cfg c = detail::to_cfg(config, occ, amp);
    dev.check(pb200_run_begin(dev.get(), &c));
    std::uint64_t rows = 0;
    dev.check(pb200_run_info(dev.get(), &rows, nullptr, nullptr, nullptr));
    if (rows > config.q_nom)
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
        std::uint64_t rows = 0, npts = 0;
        double t_now = 0;
        dev.check(pb200_run_info(dev.get(), &rows, nullptr, &t_now, nullptr));
        const std::size_t bins = config.histogram_bins;
        const std::size_t cap = (bins == 0) ? rows : std::min<std::size_t>(bins, rows);
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
    for (std::size_t s = 1; s <= nsteps; ++s) {
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
    std::size_t q_nom_last = config.q_nom;
    auto [st, sp] = detail::download(dev, terms, result.diagnostics.size() > 1 ? config.m : config.m_init, q_nom_last);
    result.final_state = std::move(st);
    result.final_space = std::move(sp);
    return result;
}

}  // namespace paces::b200
