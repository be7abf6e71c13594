// paces_b200 -- command-line front-end of the B200 path: the reference's `paces dynamics` and
// `paces spectrum` sub-commands (proj/tools/paces.cpp:84-130) with the timestep loop on the GPU.  Configuration files,
// CSV / checkpoint formats and the spectrum transform are the reference's own (config.hpp, io.hpp, spectra.hpp are
// used as they are); only run() is the drop-in from include/paces_b200.hpp.  CLI11 is not in this image, so the few
// options are parsed by hand: --config FILE (required), --out DIR, --seed N, --threads N, --deterministic,
// --resume CHECKPOINT (continue a dynamics run from a checkpoint.bin), --cpu (run the reference's CPU path instead:
// the A/B switch used by tests/test_gpu_cli.py).
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <iostream>
#include <string>

#include "paces/config.hpp"
#include "paces/engine.hpp"
#include "paces/io.hpp"
#include "paces/spectra.hpp"

#include "paces_b200.hpp"

namespace fs = std::filesystem;
using namespace paces;

namespace {

struct Options {
    std::string command, config_path, out_dir = ".", resume_path;
    std::uint64_t seed = 0;
    bool seed_set = false, deterministic = false, cpu = false;
    int threads = 0;
};

[[noreturn]] void usage(const char* why) {
    std::cerr << "paces_b200: " << why
              << "\nusage: paces_b200 dynamics|spectrum --config FILE [--out DIR] [--seed N] [--threads N] [--deterministic]"
                 " [--resume CHECKPOINT] [--cpu]\n";
    std::exit(2);
}

Options parse(int argc, char** argv) {
    Options o;
    if (argc < 2) usage("missing sub-command");
    o.command = argv[1];
    if (o.command != "dynamics" && o.command != "spectrum") usage("unknown sub-command");
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto value = [&]() -> std::string {
            if (i + 1 >= argc) usage(("option " + a + " needs a value").c_str());
            return argv[++i];
        };
        if (a == "--config") o.config_path = value();
        else if (a == "--out") o.out_dir = value();
        else if (a == "--seed") { o.seed = std::stoull(value()); o.seed_set = true; }
        else if (a == "--threads") o.threads = std::stoi(value());
        else if (a == "--resume") o.resume_path = value();
        else if (a == "--deterministic") o.deterministic = true;
        else if (a == "--cpu") o.cpu = true;
        else usage(("unknown option " + a).c_str());
    }
    if (o.config_path.empty()) usage("--config is required");
    return o;
}

std::string out_path(const Options& o, const std::string& name) {
    fs::create_directories(o.out_dir);
    return (fs::path(o.out_dir) / name).string();
}

RunResult run_configured(const Options& o, const LoadedConfig& cfg) {
    if (o.cpu) {
        if (!o.resume_path.empty()) usage("--resume needs the B200 path");
        return paces::run(cfg.run);
    }
    const HamiltonianTermSet terms = build_model(cfg.run.model);
    if (!o.resume_path.empty()) return b200::resume(o.resume_path, cfg.run, terms);
    return b200::run(cfg.run, terms);
}

/// The files `paces dynamics` leaves behind (paces.cpp:61-82): observables, diagnostics, checkpoint, histograms.
int write_outputs(const Options& o, const LoadedConfig& cfg, const RunResult& result) {
    const std::string prov = "paces " + o.command + " " + cfg.provenance;
    write_observables_csv(out_path(o, "observables.csv"), prov, result.trajectory, cfg.run.model.geometry.sites());
    write_diagnostics_csv(out_path(o, "diagnostics.csv"), prov, result.diagnostics);
    write_checkpoint(out_path(o, "checkpoint.bin"), result.final_state);
    for (std::size_t i = 0; i < result.histograms.size(); ++i) {
        char name[48];
        std::snprintf(name, sizeof(name), "histogram_%04zu.csv", i);
        write_histogram_csv(out_path(o, name), prov, result.histograms[i].first, result.histograms[i].second);
    }
    for (const auto& w : result.warnings) std::cerr << "warning: " << w << "\n";
    if (!result.error.empty()) {
        std::cerr << "error: run aborted at " << result.error << "\nlast good state written to checkpoint.bin (t="
                  << result.final_state.t << ")\n";
        return 1;
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Options o = parse(argc, argv);
        if (o.deterministic)
            set_thread_count(1);
        else if (o.threads > 0)
            set_thread_count(o.threads);
        const LoadedConfig cfg = load_run_config(parse_config_file(o.config_path), o.seed, o.seed_set);
        if (o.command == "dynamics") {
            const RunResult result = run_configured(o, cfg);
            const int rc = write_outputs(o, cfg, result);
            if (rc == 0)
                std::cout << "dynamics: " << result.diagnostics.size() << " steps, final norm "
                          << state_norm(result.final_state) << ", outputs in " << o.out_dir << "\n";
            return rc;
        }
        // spectrum (paces.cpp:110-130): autocorrelation from a dynamics run (or a previous observables.csv), damped and
        // transformed by the reference's spectra.hpp
        std::vector<SignalSample> signal;
        if (!cfg.spectrum.input.empty()) {
            signal = read_observables_signal(cfg.spectrum.input);
        } else {
            if (cfg.run.initial.kind != InitialStateSpec::Kind::optical)
                std::cerr << "note: spectrum runs usually start from initial = optical\n";
            const RunResult result = run_configured(o, cfg);
            const int rc = write_outputs(o, cfg, result);
            if (rc != 0) return rc;
            for (const auto& row : result.trajectory) signal.push_back({row.t, row.amp});
        }
        damp_signal(signal, cfg.spectrum.spectrum.tau);
        const auto spec = transform(signal, cfg.spectrum.spectrum);
        write_spectrum_csv(out_path(o, "spectrum.csv"), "paces spectrum " + cfg.provenance, spec);
        std::cout << "spectrum: " << spec.size() << " frequency bins written to " << out_path(o, "spectrum.csv") << "\n";
        return 0;
    } catch (const Error& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
