// acceptance_b200.cpp -- the reference's acceptance criteria and engine tests that live on the hot path, run THROUGH
// the drop-in shim (include/paces_b200.hpp over libpaces_b200.so) on the GPU.  Every block below starts with
// PACES_B200_DROP_IN, after which the unqualified reference calls (run, initialize, truncate_select, grow_subspace,
// remap_state, expmv, state_norm, ...) are the B200 versions -- the loops are written the way the reference's own
// tests write them (proj/tests/acceptance_main.cpp, proj/tests/test_engine.cpp; cited per block).  The reference's
// CPU functions stay reachable as paces::<name> and serve as the comparison where a criterion needs one.
// Eigen and GoogleTest are not in this image: the dense oracle of criterion 3 is the closed-form spectrum of the open
// tight-binding chain, and checks are plain CHECK lines.  Built by `make -C oracle accept` where the reference
// headers exist; runs on the GPU box from oracle/_ref/.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "paces/config.hpp"
#include "paces/engine.hpp"
#include "paces/io.hpp"

#include "paces_b200.hpp"

using namespace paces;
namespace fs = std::filesystem;

static int g_fail = 0;
#define CHECK(cond, ...)                                    \
    do {                                                    \
        if (!(cond)) {                                      \
            ++g_fail;                                       \
            std::printf("FAIL %s:%d: ", __FILE__, __LINE__); \
            std::printf(__VA_ARGS__);                       \
            std::printf("\n");                              \
        }                                                   \
    } while (0)

static double seconds_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

static ModelSpec holstein_model(std::vector<std::uint32_t> extents, double eps, double j, double g, std::uint32_t d_pho,
                                double omega = 1.0) {
    ModelSpec s;
    s.kind = ModelKind::holstein;
    s.geometry = LatticeGeometry(std::move(extents));
    s.holstein = {{eps}, {j}, {omega}, {g}, d_pho};
    return s;
}

static std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

// ---- criterion 3 (acceptance_main.cpp:139-176): tight-binding chain L = 101, RMSD against exact propagation -------
static void criterion3() {
    PACES_B200_DROP_IN;
    const auto t0 = std::chrono::steady_clock::now();
    RunConfig cfg;
    cfg.model.kind = ModelKind::tight_binding;
    cfg.model.geometry = LatticeGeometry({101});
    cfg.model.holstein.eps = {0.0};
    cfg.model.holstein.hop_j = {1.0};
    cfg.initial.kind = InitialStateSpec::Kind::localized;  // centre site 50
    cfg.m_init = 10;
    cfg.m = 2;
    cfg.q_nom = 101;
    cfg.propagator.dt = 0.05;
    cfg.t_max = 10.0;
    cfg.cadence = 20;
    auto ts = build_model(cfg.model);
    auto result = run(cfg, ts);
    CHECK(result.error.empty(), "criterion 3: run aborted: %s", result.error.c_str());
    // exact propagation of the open chain: eigenpairs sqrt(2/(L+1)) sin(pi k (j+1) / (L+1)), E_k = 2 J cos(pi k / (L+1))
    const int L = 101;
    const double pi = std::acos(-1.0);
    double max_err = 0;
    for (const auto& row : result.trajectory) {
        ExcitonDensity d;
        d.p.assign(L, 0.0);
        for (int j = 0; j < L; ++j) {
            cplx a(0, 0);
            for (int k = 1; k <= L; ++k) {
                const double vk0 = std::sin(pi * k * 51.0 / (L + 1)), vkj = std::sin(pi * k * (j + 1.0) / (L + 1));
                const double e = 2.0 * std::cos(pi * k / (L + 1));
                a += (2.0 / (L + 1)) * vk0 * vkj * std::exp(cplx(0, -e * row.t));
            }
            d.p[j] = std::norm(a);
        }
        max_err = std::max(max_err, std::abs(row.rmsd - rmsd(d, cfg.model.geometry)));
    }
    const double secs = seconds_since(t0);
    std::printf("criterion 3   max RMSD error = %.3e (<= 1e-8), %zu rows, %.2f s (need < 30)\n", max_err,
                result.trajectory.size(), secs);
    CHECK(max_err <= 1e-8 && secs < 30.0, "criterion 3");
}

// ---- criterion 6 (acceptance_main.cpp:300-377): q_nom sweep, manual step loop, q_true = kappa^(m) q_nom exactly ---
static void criterion6() {
    PACES_B200_DROP_IN;
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<std::size_t> sweep{2000, 4000, 8000, 16000, 32000};
    std::vector<double> final_loss;
    std::size_t law_checks = 0, law_failures = 0;
    bool q_bound_ok = true;
    for (std::size_t q_nom : sweep) {
        RunConfig cfg;
        cfg.model = holstein_model({7}, 0.0, 1.0, 4.0, 8);
        cfg.initial.kind = InitialStateSpec::Kind::localized;
        cfg.m_init = 6;
        cfg.m = 2;
        cfg.q_nom = q_nom;
        cfg.propagator.dt = 0.05;
        cfg.t_max = 5.0;
        cfg.seed = 11;
        auto terms = build_model(cfg.model);
        auto [state, space] = initialize(cfg, terms);
        {
            SparseState first = state;
            expmv(space.hamiltonian, first.coeff, cfg.propagator);
            first.t = cfg.propagator.dt;
            state = std::move(first);
        }
        const std::size_t nsteps = cfg.step_count();
        for (std::size_t s = 2; s <= nsteps; ++s) {
            auto kept = truncate_select(state, cfg.q_nom, mix_seed(cfg.seed + s));
            const bool truncating = kept.rows < state.coeff.size();
            auto next = grow_subspace(kept, terms, cfg.m);
            if (truncating) {
                if (next.q_true() < cfg.q_nom) q_bound_ok = false;
                ++law_checks;  // the law in exact integer form, against the reference's CPU image count
                if (next.q_true() != neighbor_image_size(kept, terms, cfg.m)) ++law_failures;
            }
            auto [psi, discarded] = remap_state(state, next);
            (void)discarded;
            expmv(next.hamiltonian, psi.coeff, cfg.propagator);
            psi.t = state.t + cfg.propagator.dt;
            state = std::move(psi);
            space = std::move(next);
        }
        final_loss.push_back(1.0 - state_norm(state));
    }
    bool monotone = true;
    for (std::size_t i = 1; i < final_loss.size(); ++i)
        if (final_loss[i] > final_loss[i - 1]) monotone = false;
    const double secs = seconds_since(t0);
    std::printf("criterion 6   final norm loss");
    for (double l : final_loss) std::printf(" %.3e", l);
    std::printf(" (non-increasing: %s), q_true = kappa^(m) q_nom held at %zu/%zu truncating steps, %.1f s (need < 300)\n",
                monotone ? "yes" : "NO", law_checks - law_failures, law_checks, secs);
    CHECK(monotone && q_bound_ok && law_failures == 0 && law_checks > 0 && secs < 300.0, "criterion 6");
}

// ---- criterion 10 (acceptance_main.cpp:463-523): determinism; here also: the GPU's CSVs against the reference's ---
static void criterion10() {
    auto dir = fs::temp_directory_path() / "paces_b200_acceptance_c10";
    fs::remove_all(dir);
    fs::create_directories(dir);
    RunConfig cfg;
    cfg.model = holstein_model({3}, 0.0, 1.0, 1.5, 4);
    cfg.initial.kind = InitialStateSpec::Kind::localized;
    cfg.m_init = 4;
    cfg.m = 2;
    cfg.q_nom = 60;
    cfg.propagator.dt = 0.05;
    cfg.t_max = 2.0;
    cfg.seed = 77;
    std::vector<std::string> files;
    RunResult gpu;
    {
        PACES_B200_DROP_IN;
        for (int rep = 0; rep < 2; ++rep) {
            auto result = run(cfg);
            CHECK(result.error.empty(), "criterion 10: run aborted: %s", result.error.c_str());
            const std::string obs = (dir / ("obs" + std::to_string(rep) + ".csv")).string();
            const std::string diag = (dir / ("diag" + std::to_string(rep) + ".csv")).string();
            write_observables_csv(obs, "acceptance determinism", result.trajectory, 3);
            write_diagnostics_csv(diag, "acceptance determinism", result.diagnostics);
            files.push_back(obs);
            files.push_back(diag);
            gpu = std::move(result);
        }
    }
    const bool bytes_equal = slurp(files[0]) == slurp(files[2]) && slurp(files[1]) == slurp(files[3]);
    // the reference on the CPU: same trajectory to 1e-12 (its own thread-count criterion), same diagnostics integers
    set_thread_count(1);
    const RunResult cpu = paces::run(cfg);
    double max_diff = 0;
    CHECK(cpu.trajectory.size() == gpu.trajectory.size(), "criterion 10: trajectory length");
    for (std::size_t i = 0; i < std::min(cpu.trajectory.size(), gpu.trajectory.size()); ++i) {
        max_diff = std::max(max_diff, std::abs(cpu.trajectory[i].norm - gpu.trajectory[i].norm));
        max_diff = std::max(max_diff, std::abs(cpu.trajectory[i].energy - gpu.trajectory[i].energy));
        for (std::size_t j = 0; j < cpu.trajectory[i].density.size(); ++j)
            max_diff = std::max(max_diff, std::abs(cpu.trajectory[i].density[j] - gpu.trajectory[i].density[j]));
    }
    bool ints_equal = cpu.diagnostics.size() == gpu.diagnostics.size();
    for (std::size_t i = 0; ints_equal && i < cpu.diagnostics.size(); ++i)
        ints_equal = cpu.diagnostics[i].q_true == gpu.diagnostics[i].q_true &&
                     cpu.diagnostics[i].taylor_order == gpu.diagnostics[i].taylor_order;
    fs::remove_all(dir);
    std::printf("criterion 10  GPU CSVs byte-identical across runs: %s; GPU vs reference observable drift = %.3e (<= 1e-12); "
                "q_true / Taylor order per step equal: %s\n",
                bytes_equal ? "yes" : "NO", max_diff, ints_equal ? "yes" : "NO");
    CHECK(bytes_equal && max_diff <= 1e-12 && ints_equal, "criterion 10");
}

// ---- test_engine.cpp:126-160: tie break unbiased over 10^4 seeds, and identical to the reference's draw ------------
static SparseState state_with_weights(const HamiltonianTermSet& ts,
                                      const std::vector<std::pair<std::vector<std::uint32_t>, double>>& entries) {
    auto table = std::make_shared<PackedBasisTable<Word>>(ts.layout);
    std::vector<std::pair<std::vector<Word>, double>> rows;
    for (const auto& [occ, amp] : entries) rows.push_back({pack_state<Word>(ts.layout, occ), amp});
    std::sort(rows.begin(), rows.end());
    SparseState st;
    for (const auto& [key, amp] : rows) {
        table->words.insert(table->words.end(), key.begin(), key.end());
        st.coeff.push_back(cplx(amp, 0));
    }
    table->rows = rows.size();
    table->sorted = true;
    st.table = table;
    return st;
}

static void tie_break_statistics() {
    PACES_B200_DROP_IN;
    auto ts = build_model(holstein_model({4}, 0.0, 1.0, 0.5, 2));
    auto psi = state_with_weights(
        ts, {{{0, 0, 0, 0, 0}, 0.5}, {{1, 0, 0, 0, 0}, 0.5}, {{2, 0, 0, 0, 0}, 0.5}, {{3, 0, 0, 0, 0}, 0.5}});
    (void)grow_subspace(*psi.table, ts, 0);  // binds the model's context for the terms-less signature below
    std::map<std::uint32_t, int> counts;
    const int trials = 10000;
    int differ = 0;
    for (int seed = 0; seed < trials; ++seed) {
        auto kept = truncate_select(psi, 2, static_cast<std::uint64_t>(seed));
        CHECK(kept.rows == 2u, "tie break: kept rows");
        for (std::size_t i = 0; i < kept.rows; ++i) counts[get_site<Word>(ts.layout, kept.row(i), 0)]++;
        if (seed % 50 == 0 && kept.words != paces::truncate_select(psi, 2, static_cast<std::uint64_t>(seed)).words) ++differ;
    }
    double worst = 0;
    for (auto [site, count] : counts) worst = std::max(worst, std::abs(double(count) / trials - 0.5));
    std::printf("tie break     max |frequency - 0.5| over %d seeds = %.4f (<= 0.02); draws differing from the reference: %d\n",
                trials, worst, differ);
    CHECK(counts.size() == 4 && worst <= 0.02 && differ == 0, "tie break statistics");
}

// ---- test_engine.cpp:394-422 + resume: checkpoint bytes, round trip, continuation --------------------------------
static void checkpoint_and_resume() {
    RunConfig cfg;
    cfg.model = holstein_model({3}, 0.3, 0.8, 0.9, 3);
    cfg.initial.kind = InitialStateSpec::Kind::optical;
    cfg.m_init = 3;
    cfg.m = 2;
    cfg.q_nom = 30;
    cfg.propagator.dt = 0.05;
    cfg.t_max = 1.0;
    const auto terms = build_model(cfg.model);
    const auto dir = fs::temp_directory_path();
    const std::string p_gpu = (dir / "paces_b200_ckpt_gpu.bin").string(), p_cpu = (dir / "paces_b200_ckpt_cpu.bin").string();
    RunResult whole, half, rest;
    {
        PACES_B200_DROP_IN;
        whole = run(cfg, terms);
        RunConfig first = cfg;
        first.t_max = 0.5;
        half = run(first, terms);
        CHECK(whole.error.empty() && half.error.empty(), "checkpoint: runs aborted");
        write_checkpoint(p_gpu, half.final_state);
        rest = resume(p_gpu, cfg, terms);
        CHECK(rest.error.empty(), "resume aborted: %s", rest.error.c_str());
    }
    RunConfig first = cfg;
    first.t_max = 0.5;
    const RunResult cpu_half = paces::run(first, terms);
    write_checkpoint(p_cpu, cpu_half.final_state);
    const std::string bytes_gpu = slurp(p_gpu), bytes_cpu = slurp(p_cpu);
    CHECK(bytes_gpu.size() > 6 && bytes_gpu.compare(0, 6, std::string("PACES\x01", 6)) == 0, "checkpoint magic");
    CHECK(bytes_gpu == bytes_cpu, "a GPU run's checkpoint is not byte-identical to the reference's (%zu vs %zu bytes)",
          bytes_gpu.size(), bytes_cpu.size());
    const SparseState loaded = read_checkpoint(p_gpu);
    CHECK(loaded.t == half.final_state.t && loaded.coeff == half.final_state.coeff &&
              loaded.table->words == half.final_state.table->words && loaded.table->sorted,
          "checkpoint round trip");
    CHECK(rest.final_state.t == whole.final_state.t && rest.final_state.coeff == whole.final_state.coeff &&
              rest.final_state.table->words == whole.final_state.table->words,
          "resumed run does not end in the uninterrupted run's state");
    CHECK(rest.diagnostics.size() + half.diagnostics.size() == whole.diagnostics.size(), "resume: step count");
    bool same_tail = true;
    for (std::size_t i = 0; i < rest.diagnostics.size() && same_tail; ++i) {
        const auto &a = rest.diagnostics[i], &b = whole.diagnostics[half.diagnostics.size() + i];
        same_tail = a.step == b.step && a.q_true == b.q_true && a.taylor_order == b.taylor_order && a.energy == b.energy &&
                    a.norm_post == b.norm_post;
    }
    CHECK(same_tail, "resume: diagnostics of the remaining steps differ");
    std::printf("checkpoint    %zu bytes, byte-identical to the reference's: %s; resumed %zu steps to the same bits: %s\n",
                bytes_gpu.size(), bytes_gpu == bytes_cpu ? "yes" : "NO", rest.diagnostics.size(),
                rest.final_state.coeff == whole.final_state.coeff ? "yes" : "NO");
    fs::remove(p_gpu);
    fs::remove(p_cpu);
}

int main() {
    criterion3();
    criterion6();
    criterion10();
    tie_break_statistics();
    checkpoint_and_resume();
    if (g_fail) {
        std::printf("acceptance (B200 shim): %d FAILED\n", g_fail);
        return 1;
    }
    std::printf("acceptance (B200 shim): all passed\n");
    return 0;
}
