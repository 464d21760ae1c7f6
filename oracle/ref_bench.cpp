// CPU baseline driver. TEST/BENCH INFRASTRUCTURE ONLY.
//
// Times the reference's own fitness evaluation (evaluate_fitness,
// src/vm.cpp:558-579, the evaluation half of Engine::sanity_check,
// src/engine.cpp:91-95) over a workload of variants, on the host cores, with a
// plain std::thread pool (the reference's parallel_for shape,
// src/engine.cpp:28-62). Validation (is_valid) runs before the timed region,
// as the device arm's timed region holds evaluation only. Used by bench.py for
// the `cpu_baseline` field and for `--impl reference`.
//
//   ref_bench <bench> <variants.txt> <n_tests> <test_seed> <threads> <max_seconds>
//             [budget=1000000] [tolerance=0] [start=0]
//
// start: first variant of the sample (the timed loop walks the variants from
// there, wrapping around, until max_seconds).
//
// <bench> is a registry name, or file:<prefix> for an authored kernel
// (<prefix>.ir + <prefix>.gen.json, via the reference's parse_kernel,
// generator_spec_from_json and generate_tests_for). REF_BENCH_NOCOUNT=1 skips
// the untimed dynamic-IR counting pass (ir = -1).
//
// variants.txt: one patch per line as compact JSON (patch_to_json format).
// Prints one JSON object: variants, executions (tests actually run, i.e. up to
// and including the first failing one), ir (reference dynamic instruction
// count of those executions), seconds, threads.

#include "evoir/corpus.hpp"
#include "evoir/engine.hpp"

#include <atomic>
#include <cstdlib>
#include <sstream>
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <thread>

using namespace evoir;

int main(int argc, char** argv) {
    if (argc < 7) {
        std::cerr << "usage: ref_bench <bench> <variants.txt> <n_tests> <test_seed> <threads> "
                     "<max_seconds> [budget] [tolerance]\n";
        return 1;
    }
    const std::string name = argv[1];
    Kernel kernel;
    GeneratorSpec gen;
    bool registry = name.rfind("file:", 0) != 0;
    Benchmark b;
    if (registry) {
        b = load_benchmark(name);
        kernel = b.kernel;
    } else {
        auto slurp = [](const std::string& path) {
            std::ifstream f(path);
            std::stringstream ss;
            ss << f.rdbuf();
            return ss.str();
        };
        const std::string prefix = name.substr(5);
        kernel = parse_kernel(slurp(prefix + ".ir"));
        gen = generator_spec_from_json(slurp(prefix + ".gen.json"));
    }
    std::ifstream in(argv[2]);
    int n_tests = std::stoi(argv[3]);
    uint64_t seed = std::stoull(argv[4]);
    int threads = std::stoi(argv[5]);
    double max_seconds = std::stod(argv[6]);
    int64_t budget = argc > 7 ? std::stoll(argv[7]) : 1000000;
    double tol = argc > 8 ? std::stod(argv[8]) : 0.0;
    const size_t start = argc > 9 ? std::stoull(argv[9]) : 0;

    std::vector<Kernel> variants;
    std::string line;
    while (std::getline(in, line)) {
        if (line.empty())
            continue;
        variants.push_back(apply_patch(kernel, patch_from_json(line)).kernel);
    }
    // untimed: validation, and the sample order (from `start`, wrapping)
    std::vector<char> valid(variants.size(), 0);
    for (size_t i = 0; i < variants.size(); ++i)
        valid[i] = is_valid(variants[i]);
    std::vector<size_t> order(variants.size());
    for (size_t i = 0; i < order.size(); ++i)
        order[i] = (start + i) % order.size();
    auto tests = registry ? generate_tests(b, n_tests, seed)
                          : generate_tests_for(kernel, gen, n_tests, seed);
    ExecConfig cfg = ExecConfig::for_kernel(kernel);
    cfg.instruction_budget = budget;
    ExecConfig unit = cfg;
    {
        CostTable& t = unit.cost_table;
        t.arith = t.cmp = t.select_op = t.phi = t.constant = t.br = t.intrinsic = t.getindex = 1;
        t.load_shared = t.store_shared = t.load_global = t.store_global = t.sync = t.ret = 1;
    }

    std::atomic<size_t> next{0};
    std::atomic<bool> stop{false};
    std::vector<char> done(variants.size(), 0);
    std::vector<int> ran(variants.size(), 0); // tests evaluate_fitness ran
    const int n_suite = static_cast<int>(tests.size());
    auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    std::vector<std::thread> pool;
    for (int w = 0; w < threads; ++w)
        pool.emplace_back([&] {
            for (;;) {
                const size_t k = next.fetch_add(1);
                if (k >= variants.size() || stop.load())
                    return;
                const size_t i = order[k];
                if (valid[i]) {
                    const EvalOutcome o = evaluate_fitness(variants[i], tests, cfg, tol);
                    ran[i] = o.accepted ? n_suite : o.failing_test + 1;
                }
                done[i] = 1;
                if (elapsed() > max_seconds)
                    stop.store(true);
            }
        });
    for (auto& t : pool)
        t.join();
    double secs = elapsed();

    // Counting pass (untimed): executions and dynamic IR of the same work.
    int64_t execs = 0, ir = 0, processed = 0;
    const bool count = !std::getenv("REF_BENCH_NOCOUNT");
    if (!count)
        ir = -1;
    for (size_t i = 0; i < variants.size(); ++i) {
        if (!done[i])
            continue;
        ++processed;
        if (!count) {
            execs += ran[i];
            continue;
        }
        if (!valid[i])
            continue;
        for (const auto& t : tests) {
            ExecResult r = execute(variants[i], t, unit);
            ++execs;
            ir += r.cost;
            if (r.status != ExecStatus::Completed)
                break;
            if (compute_error(r.outputs, t.oracle) > tol)
                break;
        }
    }
    std::printf("{\"variants\": %lld, \"executions\": %lld, \"ir\": %lld, \"seconds\": %.6f, "
                "\"threads\": %d}\n",
                static_cast<long long>(processed), static_cast<long long>(execs),
                static_cast<long long>(ir), secs, threads);
    return 0;
}
