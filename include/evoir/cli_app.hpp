// Run driver and report rendering (reference: include/evoir/cli_app.hpp:10-68
// of arxiv/paper_2004_08140). Only the parts that define the trajectory
// artefacts are provided: seed derivation, tolerance mode, log.csv and
// report.json rendering, and cmd_run / cmd_replay.
#pragma once

#include "evoir/engine.hpp"

#include <cstdint>
#include <optional>
#include <string>

namespace evoir::cli {

inline constexpr int kExitOk = 0;
inline constexpr int kExitUsage = 1;
inline constexpr int kExitInitFailure = 2;

struct RunOptions {
    std::string bench;
    std::string kernel_path;
    std::string tests_dir;
    std::string heldout_dir;
    std::string mode = "default";
    std::optional<double> tolerance;
    int pop = 256;
    std::optional<int> generations;
    std::optional<double> wallclock_seconds;
    double cross_rate = 0.80;
    double mutate_rate = 0.30;
    int init_dist = 3;
    uint64_t seed = 0;
    int jobs = 1;
    int train_tests = 3;
    int heldout_tests = 3;
    std::string out_dir = "evoir-out";
};

struct ReplayOptions {
    std::string bench;
    std::string kernel_path;
    std::string tests_dir;
    std::string patch_path;
    std::string mode = "default";
    std::optional<double> tolerance;
    uint64_t seed = 0;
    int train_tests = 3;
};

int cmd_run(const RunOptions& opt);
int cmd_replay(const ReplayOptions& opt);

double effective_tolerance(const std::string& mode, std::optional<double> tolerance);
uint64_t train_seed(uint64_t master);
uint64_t heldout_seed(uint64_t master);

// Artefacts of a finished run, byte-compatible with the reference CLI.
std::string render_log_csv(const SearchResult& r);
std::string render_report(const RunOptions& opt, const std::string& source, double tolerance,
                          const SearchResult& r);

// Runs a registry benchmark like `evoir run` and returns the artefacts
// instead of writing them (used by the C ABI and parity tests).
struct RunArtifacts {
    std::string log_csv;
    std::string report_json;
    std::string best_ir;
    std::string best_patch;
    EngineCounters counters;
    double seconds = 0.0;
};
RunArtifacts run_benchmark(const RunOptions& opt);

} // namespace evoir::cli
