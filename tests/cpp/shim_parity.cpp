// shim_parity.cpp -- drop-in proof: the reference's own paces::run()/step() and the free functions on the
// path, side by side with paces::b200::* (include/paces_b200.hpp over libpaces_b200.so), on the same inputs.
// Built in the build container against the UNMODIFIED reference headers (oracle/Makefile target `shim`) into
// oracle/_ref/shim_parity; executed on the GPU box by tests/test_gpu_shim.py.  Exit code 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "paces/engine.hpp"
#include "paces/spectra.hpp"

#include "paces_b200.hpp"

using namespace paces;

static int g_fail = 0;
#define CHECK(cond, ...)                                   \
    do {                                                   \
        if (!(cond)) {                                     \
            ++g_fail;                                      \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                      \
            std::printf("\n");                             \
        }                                                  \
    } while (0)

static bool close(double a, double b, double rtol = 1e-10, double atol = 0) {
    return std::fabs(a - b) <= atol + rtol * std::max(std::fabs(a), std::fabs(b));
}
template <class T>
static bool same_bits(const std::vector<T>& a, const std::vector<T>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}

static RunConfig holstein(std::vector<std::uint32_t> ext, std::uint32_t d, double g, double j, std::size_t q_nom,
                          double t_max, InitialStateSpec::Kind kind) {
    RunConfig c;
    c.model.kind = ModelKind::holstein;
    c.model.geometry = LatticeGeometry(ext);
    c.model.holstein.eps = {0.0};
    c.model.holstein.hop_j = {j};
    c.model.holstein.omega = {1.0};
    c.model.holstein.g = {g};
    c.model.holstein.d_pho = d;
    c.initial.kind = kind;
    c.m_init = 4;
    c.m = 2;
    c.q_nom = q_nom;
    c.t_max = t_max;
    c.seed = 7;
    return c;
}

static void compare_runs(const char* name, const RunConfig& cfg) {
    const HamiltonianTermSet terms = build_model(cfg.model);
    RunResult a = run(cfg, terms);
    RunResult b = b200::run(cfg, terms);
    CHECK(a.error == b.error, "%s: error '%s' vs '%s'", name, a.error.c_str(), b.error.c_str());
    CHECK(a.diagnostics.size() == b.diagnostics.size(), "%s: diagnostics count", name);
    CHECK(a.trajectory.size() == b.trajectory.size(), "%s: trajectory count", name);
    CHECK(a.warnings == b.warnings, "%s: warnings", name);
    for (std::size_t i = 0; i < std::min(a.diagnostics.size(), b.diagnostics.size()); ++i) {
        const auto &x = a.diagnostics[i], &y = b.diagnostics[i];
        CHECK(x.step == y.step && x.q_true == y.q_true && x.taylor_order == y.taylor_order, "%s: diag %zu ints", name, i);
        CHECK(close(x.t, y.t, 1e-14) && close(x.norm_pre, y.norm_pre) && close(x.norm_post, y.norm_post) &&
                  close(x.energy, y.energy, 1e-10, 1e-12) && close(x.discarded_weight, y.discarded_weight, 1e-9, 1e-30) &&
                  std::fabs(x.delta_norm_expmv - y.delta_norm_expmv) <= 1e-12,
              "%s: diag %zu values", name, i);
    }
    for (std::size_t i = 0; i < std::min(a.trajectory.size(), b.trajectory.size()); ++i) {
        const auto &x = a.trajectory[i], &y = b.trajectory[i];
        CHECK(close(x.t, y.t, 1e-14) && close(x.norm, y.norm) && close(x.energy, y.energy, 1e-10, 1e-12) &&
                  close(x.rmsd, y.rmsd, 1e-10, 1e-12) && close(x.xbar, y.xbar, 1e-10, 1e-12) &&
                  std::abs(x.amp - y.amp) <= 1e-12,
              "%s: trajectory row %zu", name, i);
        CHECK(x.density.size() == y.density.size(), "%s: density size", name);
        for (std::size_t k = 0; k < std::min(x.density.size(), y.density.size()); ++k)
            CHECK(close(x.density[k], y.density[k], 1e-10, 1e-18), "%s: density %zu/%zu", name, i, k);
    }
    CHECK(a.histograms.size() == b.histograms.size(), "%s: histogram count", name);
    for (std::size_t i = 0; i < std::min(a.histograms.size(), b.histograms.size()); ++i) {
        const auto &x = a.histograms[i].second, &y = b.histograms[i].second;
        CHECK(close(a.histograms[i].first, b.histograms[i].first, 1e-14) && x.support == y.support && x.q50 == y.q50 &&
                  x.q90 == y.q90 && x.q99 == y.q99 && x.q9999 == y.q9999 &&
                  close(x.tail_exponent, y.tail_exponent, 1e-10, 1e-12) &&  // device log + tree sums, not the host loop
                 
                  x.rank == y.rank && x.weight == y.weight,
              "%s: weight histogram %zu", name, i);
    }
    CHECK(same_bits(a.final_state.table->words, b.final_state.table->words), "%s: final table", name);
    CHECK(same_bits(a.final_state.coeff, b.final_state.coeff), "%s: final coefficients not bit-identical", name);
    CHECK(a.final_state.t == b.final_state.t, "%s: final t", name);
    CHECK(same_bits(a.final_space.hamiltonian.row_ptr, b.final_space.hamiltonian.row_ptr) &&
              same_bits(a.final_space.hamiltonian.col, b.final_space.hamiltonian.col) &&
              same_bits(a.final_space.hamiltonian.val, b.final_space.hamiltonian.val),
          "%s: final CSR", name);
    std::printf("%-28s steps=%zu q_true=%zu fails so far=%d\n", name, a.diagnostics.size(), a.final_space.q_true(), g_fail);
}

static void compare_functions() {
    RunConfig cfg = holstein({3, 2}, 6, 0.71, 0.55, 150, 1.0, InitialStateSpec::Kind::optical);
    cfg.model.holstein.eps = {0.1, -0.2, 0.05, 0.3, -0.1, 0.2};
    const HamiltonianTermSet terms = build_model(cfg.model);
    b200::Device dev(terms);
    auto [state, space] = initialize(cfg, terms);
    auto [gstate, gspace] = b200::initialize(dev, cfg, terms);
    CHECK(same_bits(state.table->words, gstate.table->words) && same_bits(state.coeff, gstate.coeff), "initialize");
    CHECK(same_bits(space.hamiltonian.val, gspace.hamiltonian.val) && same_bits(space.hamiltonian.col, gspace.hamiltonian.col),
          "initialize CSR");
    // drive the five calls by hand, as acceptance_main.cpp:321-347 does
    std::vector<cplx> c = state.coeff;
    expmv(space.hamiltonian, c, cfg.propagator);
    std::vector<cplx> cg = state.coeff;
    auto r2 = b200::expmv(dev, space.hamiltonian, cg, cfg.propagator);
    CHECK(same_bits(c, cg) && r2.order_used >= 3, "expmv");
    state.coeff = c;
    for (std::size_t s = 2; s <= 6; ++s) {
        StepOutput o = step(state, space, cfg, terms, s);
        StepOutput g = b200::step(dev, state, space, cfg, terms, s);
        CHECK(same_bits(o.state.table->words, g.state.table->words), "step %zu table", s);
        CHECK(same_bits(o.state.coeff, g.state.coeff), "step %zu coeff", s);
        CHECK(same_bits(o.space.hamiltonian.val, g.space.hamiltonian.val), "step %zu H values", s);
        CHECK(o.record.q_true == g.record.q_true && o.record.taylor_order == g.record.taylor_order, "step %zu record", s);
        CHECK(o.space.q_nom == g.space.q_nom, "step %zu q_nom %zu vs %zu", s, o.space.q_nom, g.space.q_nom);
        state = std::move(o.state);
        space = std::move(o.space);
    }
    auto kept = truncate_select(state, 40, 99), gkept = b200::truncate_select(dev, state, 40, 99);
    CHECK(same_bits(kept.words, gkept.words) && kept.rows == gkept.rows, "truncate_select");
    EffectiveSpace sp = grow_subspace(kept, terms, 2), gsp = b200::grow_subspace(dev, kept, terms, 2);
    CHECK(same_bits(sp.table->words, gsp.table->words) && same_bits(sp.hamiltonian.row_ptr, gsp.hamiltonian.row_ptr) &&
              same_bits(sp.hamiltonian.col, gsp.hamiltonian.col) && same_bits(sp.hamiltonian.val, gsp.hamiltonian.val),
          "grow_subspace");
    auto [psi, disc] = remap_state(state, sp);
    auto [gpsi, gdisc] = b200::remap_state(dev, state, gsp);
    CHECK(same_bits(psi.coeff, gpsi.coeff) && close(disc, gdisc, 1e-9, 1e-30), "remap_state");
    std::vector<cplx> y(psi.coeff.size()), gy(psi.coeff.size());
    csr_matvec(sp.hamiltonian, psi.coeff, y);
    b200::csr_matvec(dev, sp.hamiltonian, psi.coeff, gy);
    CHECK(same_bits(y, gy), "csr_matvec");
    CHECK(close(csr_expectation(sp.hamiltonian, psi.coeff), b200::csr_expectation(dev, sp.hamiltonian, psi.coeff), 1e-10, 1e-12),
          "csr_expectation");
    CHECK(close(state_norm(psi), b200::state_norm(dev, psi)), "state_norm");
    auto d = exciton_density(psi, terms), gd = b200::exciton_density(dev, psi, terms);
    for (std::size_t k = 0; k < d.p.size(); ++k) CHECK(close(d.p[k], gd.p[k], 1e-10, 1e-18), "density %zu", k);
    CHECK(std::abs(dipole_amplitude(psi, terms) - b200::dipole_amplitude(dev, psi, terms)) <= 1e-12, "dipole");
    auto pn = phonon_numbers(psi, terms), gpn = b200::phonon_numbers(dev, psi, terms);
    for (std::size_t k = 0; k < pn.size(); ++k) CHECK(close(pn[k], gpn[k], 1e-10, 1e-18), "phonon numbers %zu", k);
    {  // weight_histogram (observables.hpp:123-176; test_observables.cpp:170-220): counts and curve exact, slope 1e-10
        const WeightHistogram wh = weight_histogram(psi, 16), gwh = b200::weight_histogram(dev, psi, 16);
        CHECK(wh.support == gwh.support && wh.q50 == gwh.q50 && wh.q90 == gwh.q90 && wh.q99 == gwh.q99 &&
                  wh.q9999 == gwh.q9999 && close(wh.tail_exponent, gwh.tail_exponent, 1e-10, 1e-12) && wh.rank == gwh.rank &&
                  wh.weight == gwh.weight,
              "weight_histogram");
    }
    // error text parity (test_propagator.cpp:157-169, test_subspace.cpp preconditions)
    PropagatorConfig bad = cfg.propagator;
    bad.dt = 50.0;
    bad.max_order = 10;
    std::string m1, m2;
    try { auto cc = psi.coeff; expmv(sp.hamiltonian, cc, bad); } catch (const Error& e) { m1 = e.what(); }
    try { auto cc = psi.coeff; b200::expmv(dev, sp.hamiltonian, cc, bad); } catch (const Error& e) { m2 = e.what(); }
    CHECK(!m1.empty() && m1 == m2, "expmv divergence message '%s' vs '%s'", m1.c_str(), m2.c_str());
    std::printf("functions                    fails so far=%d\n", g_fail);
}

// BASELINE config 3 end to end at a size the CPU finishes quickly: 2D aggregate, optical start, the autocorrelation
// <mu(t) mu(0)> (ObservablesRow.amp) of the GPU trajectory goes through the reference's own damp_signal + transform
// (spectra.hpp:42-88, as tools/paces.cpp:106-109 does) and must give the reference's absorption spectrum.
static void compare_spectrum() {
    RunConfig cfg = holstein({4, 4}, 6, 0.71, -0.55, 1500, 6.0, InitialStateSpec::Kind::optical);
    cfg.m_init = 4;
    const HamiltonianTermSet terms = build_model(cfg.model);
    const RunResult a = run(cfg, terms), b = b200::run(cfg, terms);
    CHECK(a.error.empty() && b.error.empty() && a.trajectory.size() == b.trajectory.size(), "spectrum: runs");
    SpectrumConfig sc;
    sc.tau = 1.0 / 0.0577;
    sc.pad_factor = 4;
    sc.omega_min = -5.0;
    sc.omega_max = 5.0;
    std::vector<SignalSample> sa, sb;
    for (const auto& r : a.trajectory) sa.push_back({r.t, r.amp});
    for (const auto& r : b.trajectory) sb.push_back({r.t, r.amp});
    damp_signal(sa, sc.tau);
    damp_signal(sb, sc.tau);
    const auto pa = transform(sa, sc), pb = transform(sb, sc);
    CHECK(pa.size() == pb.size() && pa.size() > 10, "spectrum: bins");
    double amax = 0, dmax = 0;
    for (std::size_t k = 0; k < std::min(pa.size(), pb.size()); ++k) {
        amax = std::max(amax, std::fabs(pa[k].a));
        dmax = std::max(dmax, std::fabs(pa[k].a - pb[k].a));
        CHECK(pa[k].omega == pb[k].omega, "spectrum: grid %zu", k);
    }
    CHECK(dmax <= 1e-10 * amax, "spectrum: max |dA| = %.3e of peak %.3e", dmax, amax);
    std::printf("absorption spectrum (cfg 3)  bins=%zu peak=%.6f max|dA|=%.2e fails so far=%d\n", pa.size(), amax, dmax,
                g_fail);
}

int main() {
    try {
        compare_functions();
        compare_spectrum();
        compare_runs("holstein 1D L=4 d=8 (cfg 1)", [] {
            RunConfig c = holstein({4}, 8, 1.0, 1.0, 2000, 2.0, InitialStateSpec::Kind::localized);
            c.m_init = 6;
            return c;
        }());
        compare_runs("holstein 1D L=5 d=6 ties", [] {
            RunConfig c = holstein({5}, 6, 1.0, 1.0, 300, 3.0, InitialStateSpec::Kind::localized);
            c.m_init = 6;
            return c;
        }());
        compare_runs("holstein 2D 3x3 optical", holstein({3, 3}, 5, 0.71, -0.55, 500, 1.5, InitialStateSpec::Kind::optical));
        compare_runs("holstein 3D 2x2x2 d=16", holstein({2, 2, 2}, 16, 0.71, 0.55, 600, 1.5, InitialStateSpec::Kind::localized));
        compare_runs("cadence 3 + substeps 2", [] {
            RunConfig c = holstein({4}, 4, 1.3, 0.8, 60, 1.0, InitialStateSpec::Kind::localized);
            c.cadence = 3;
            c.emit_histograms = true;  // RunResult.histograms from the resident state (engine.hpp:329-330, 365-366)
            c.histogram_bins = 32;
            c.propagator.substeps = 2;
            c.propagator.dt = 0.1;
            c.m_init = 3;
            return c;
        }());
        compare_runs("diverging dt keeps last state", [] {
            RunConfig c = holstein({4}, 8, 4.0, 1.0, 200, 40.0, InitialStateSpec::Kind::localized);
            c.propagator.dt = 20.0;
            c.propagator.max_order = 12;
            return c;
        }());
    } catch (const std::exception& e) {
        std::printf("EXCEPTION: %s\n", e.what());
        return 2;
    }
    std::printf(g_fail ? "shim parity: %d FAILED\n" : "shim parity: all checks passed (%d failures)\n", g_fail);
    return g_fail ? 1 : 0;
}
