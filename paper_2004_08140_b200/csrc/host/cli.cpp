// Run driver: seeds, tolerance mode and the log.csv / report.json artefacts.
// Formats follow src/cli_app.cpp of arxiv/paper_2004_08140 (log 91-101 with
// %.10g, report 103-178, tolerance modes 182-191, seed derivation 193-201,
// cmd_run 203-253, cmd_replay 255-294) so trajectories compare byte for byte.
#include "evoir/cli_app.hpp"

#include "evoir/corpus.hpp"

#include <json.hpp>

#include <chrono>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>

namespace evoir::cli {

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

std::string g10(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.10g", v);
    return b;
}

std::string slurp(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in)
        throw std::runtime_error("cannot open '" + path + "'");
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

void spill(const fs::path& p, const std::string& text) {
    std::ofstream out(p, std::ios::binary);
    if (!out)
        throw std::runtime_error("cannot write '" + p.string() + "'");
    out << text;
}

std::vector<TestCase> tests_from_dir(const std::string& dir) {
    std::vector<fs::path> files;
    for (const auto& e : fs::directory_iterator(dir))
        if (e.is_regular_file() && e.path().extension() == ".json")
            files.push_back(e.path());
    std::sort(files.begin(), files.end());
    std::vector<TestCase> out;
    for (const auto& f : files)
        out.push_back(testcase_from_json(slurp(f.string())));
    return out;
}

struct Problem {
    Kernel kernel;
    std::vector<TestCase> tests, heldout;
    std::string source;
};

Problem resolve(const std::string& bench, const std::string& kernel_path,
                const std::string& tests_dir, const std::string& heldout_dir, uint64_t seed,
                int n_train, int n_heldout) {
    Problem p;
    if (!bench.empty() && !kernel_path.empty())
        throw std::runtime_error("give either a benchmark name or a kernel path, not both");
    if (!bench.empty()) {
        const Benchmark b = load_benchmark(bench);
        p.kernel = b.kernel;
        p.tests = generate_tests(b, n_train, train_seed(seed));
        if (n_heldout > 0)
            p.heldout = generate_tests(b, n_heldout, heldout_seed(seed));
        p.source = bench;
        return p;
    }
    if (kernel_path.empty())
        throw std::runtime_error("a benchmark (--bench) or kernel file (--kernel) is required");
    p.kernel = parse_kernel(slurp(kernel_path));
    if (tests_dir.empty())
        throw std::runtime_error("--tests <dir> is required with --kernel");
    p.tests = tests_from_dir(tests_dir);
    if (!heldout_dir.empty())
        p.heldout = tests_from_dir(heldout_dir);
    p.source = kernel_path;
    return p;
}

json fit_json(const FitnessVector& f) { return json{{"cost", f.cost}, {"error", f.error}}; }

SearchConfig search_config(const RunOptions& o, double tol) {
    SearchConfig c;
    c.pop_size = o.pop;
    c.cross_rate = o.cross_rate;
    c.mutate_rate = o.mutate_rate;
    c.init_dist = o.init_dist;
    c.tolerance = tol;
    c.master_seed = o.seed;
    c.jobs = o.jobs;
    c.budget = o.wallclock_seconds ? Budget::for_wallclock(*o.wallclock_seconds)
                                   : Budget::for_generations(o.generations.value_or(30));
    return c;
}

} // namespace

double effective_tolerance(const std::string& mode, std::optional<double> tolerance) {
    if (mode == "default") {
        if (tolerance && *tolerance != 0.0)
            std::cerr << "note: mode 'default' enforces exact outputs; tolerance forced to 0\n";
        return 0.0;
    }
    if (mode == "mo")
        return tolerance.value_or(0.01);
    throw std::runtime_error("unknown mode '" + mode + "' (expected 'default' or 'mo')");
}

uint64_t train_seed(uint64_t master) {
    uint64_t x = master ^ 0x7261696e5f736574ULL; // "rain_set"
    return Rng::splitmix64(x);
}

uint64_t heldout_seed(uint64_t master) {
    uint64_t x = master ^ 0x68656c645f6f7574ULL; // "held_out"
    return Rng::splitmix64(x);
}

std::string render_log_csv(const SearchResult& r) {
    std::ostringstream o;
    o << "gen,best_cost_err0,best_cost_tol,min_error,front0_size,mut_attempts,mut_accepts,"
         "cx_attempts,cx_accepts\n";
    for (const GenerationLog& g : r.log)
        o << g.gen << "," << g10(g.best_cost_err0) << "," << g10(g.best_cost_tol) << ","
          << g10(g.min_error) << "," << g.front0_size << "," << g.mut_attempts << ","
          << g.mut_accepts << "," << g.cx_attempts << "," << g.cx_accepts << "\n";
    return o.str();
}

std::string render_report(const RunOptions& opt, const std::string& source, double tolerance,
                          const SearchResult& r) {
    json rep;
    rep["source"] = source;
    rep["config"] = {{"mode", opt.mode},
                     {"tolerance", tolerance},
                     {"pop", opt.pop},
                     {"generations", r.generations_run},
                     {"cross_rate", opt.cross_rate},
                     {"mutate_rate", opt.mutate_rate},
                     {"init_dist", opt.init_dist},
                     {"seed", opt.seed},
                     {"jobs", opt.jobs},
                     {"train_tests", opt.train_tests},
                     {"heldout_tests", opt.heldout_tests}};
    rep["baseline"] = fit_json(r.baseline);
    json arch = json::array();
    for (const ArchiveEntry& e : r.archive) {
        json x;
        x["fitness"] = fit_json(*e.ind.fitness);
        x["edits"] = e.ind.patch.size();
        x["patch"] = json::parse(patch_to_json(e.ind.patch));
        x["overfit"] = e.overfit;
        if (e.heldout_error >= 0.0)
            x["heldout_error"] = e.heldout_error;
        arch.push_back(std::move(x));
    }
    rep["archive"] = std::move(arch);
    rep["best_index"] = r.best_index;
    if (r.best_index >= 0) {
        const ArchiveEntry& b = r.archive[static_cast<size_t>(r.best_index)];
        rep["best"] = {{"fitness", fit_json(*b.ind.fitness)},
                       {"edits", b.ind.patch.size()},
                       {"gain_over_baseline", (r.baseline.cost - b.ind.fitness->cost) / r.baseline.cost}};
    }
    json ops = json::object();
    for (int k = 0; k < kOperatorCount; ++k) {
        const double rate = r.stats.attempts[k] > 0 ? static_cast<double>(r.stats.accepts[k]) /
                                                          static_cast<double>(r.stats.attempts[k])
                                                    : 0.0;
        ops[operator_kind_name(static_cast<OperatorKind>(k))] = {
            {"attempts", r.stats.attempts[k]}, {"accepts", r.stats.accepts[k]}, {"rate", rate}};
    }
    const double cx_rate = r.stats.cx_attempts > 0 ? static_cast<double>(r.stats.cx_accepts) /
                                                         static_cast<double>(r.stats.cx_attempts)
                                                   : 0.0;
    const double mut_rate = r.stats.total_attempts() > 0
                                ? static_cast<double>(r.stats.total_accepts()) /
                                      static_cast<double>(r.stats.total_attempts())
                                : 0.0;
    rep["acceptance"] = {
        {"mutation", ops},
        {"mutation_overall", mut_rate},
        {"crossover",
         {{"attempts", r.stats.cx_attempts}, {"accepts", r.stats.cx_accepts}, {"rate", cx_rate}}},
        {"typical_range_note",
         "single-mutation acceptance typically lands in 0.05-0.30 and crossover acceptance "
         "reaches 0.80 in comparable genetic-improvement systems; recorded here for manual "
         "comparison, not asserted"},
    };
    return rep.dump(2) + "\n";
}

RunArtifacts run_benchmark(const RunOptions& opt) {
    const double tol = effective_tolerance(opt.mode, opt.tolerance);
    const Problem p = resolve(opt.bench, opt.kernel_path, opt.tests_dir, opt.heldout_dir, opt.seed,
                              opt.train_tests, opt.heldout_tests);
    const auto t0 = std::chrono::steady_clock::now();
    Engine engine(p.kernel, search_config(opt, tol), p.tests);
    const SearchResult r = engine.run(p.heldout);
    RunArtifacts a;
    a.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    a.counters = engine.counters();
    a.log_csv = render_log_csv(r);
    a.report_json = render_report(opt, p.source, tol, r);
    if (r.best_index >= 0) {
        const ArchiveEntry& b = r.archive[static_cast<size_t>(r.best_index)];
        a.best_ir = print_kernel(b.ind.kernel);
        a.best_patch = patch_to_json(b.ind.patch);
    }
    return a;
}

int cmd_run(const RunOptions& opt) {
    try {
        RunArtifacts a;
        try {
            a = run_benchmark(opt);
        } catch (const InitFailure& e) {
            std::cerr << "initialization failed: " << e.what() << "\n";
            return kExitInitFailure;
        }
        fs::create_directories(opt.out_dir);
        spill(fs::path(opt.out_dir) / "log.csv", a.log_csv);
        spill(fs::path(opt.out_dir) / "report.json", a.report_json);
        if (!a.best_ir.empty()) {
            spill(fs::path(opt.out_dir) / "best.ir", a.best_ir);
            spill(fs::path(opt.out_dir) / "best.patch.json", a.best_patch);
        }
        return kExitOk;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    }
}

int cmd_replay(const ReplayOptions& opt) {
    try {
        const double tol = effective_tolerance(opt.mode, opt.tolerance);
        const Problem p = resolve(opt.bench, opt.kernel_path, opt.tests_dir, "", opt.seed,
                                  opt.train_tests, 0);
        const Patch patch = patch_from_json(slurp(opt.patch_path));
        const PatchResult ap = apply_patch(p.kernel, patch);
        if (ap.applied.size() != patch.size()) {
            std::cout << "warning: " << patch.size() - ap.applied.size()
                      << " edit(s) were inapplicable and dropped:\n";
            for (const Edit& e : patch)
                if (std::find(ap.applied.begin(), ap.applied.end(), e) == ap.applied.end())
                    std::cout << "  dropped: " << edit_key(e) << "\n";
        }
        const auto errs = validate(ap.kernel);
        std::cout << "validate: " << (errs.empty() ? "ok" : "FAILED") << "\n";
        for (const auto& e : errs)
            std::cout << "  [" << e.rule << "] uid " << e.uid << ": " << e.detail << "\n";
        const EvalOutcome o =
            evaluate_fitness(ap.kernel, p.tests, ExecConfig::for_kernel(p.kernel), tol);
        if (o.accepted)
            std::cout << "fitness: cost " << g10(o.fitness.cost) << ", error " << g10(o.fitness.error)
                      << "\n";
        else
            std::cout << "rejected: test " << o.failing_test << ": " << o.reason << "\n";
        std::cout << print_kernel(ap.kernel);
        return kExitOk;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    }
}

} // namespace evoir::cli
