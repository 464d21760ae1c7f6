// Golden-vector generator. TEST INFRASTRUCTURE ONLY.
//
// Links the reference library compiled in place from /root/reference/proj/src
// (see oracle/Makefile) and writes JSON-lines fixtures that pin the product's
// behaviour to the reference's own outputs. Nothing in the product links or
// calls this; tests/golden/ holds its committed output and
// oracle/gen_golden.sh is the recipe.
//
// Subcommands (all write to stdout):
//   corpus                     printed kernels, generated tests (train/held-out seeds of
//                              configs 1-2) with oracles, per-test cost and dynamic IR
//   mutants <n> [budget]       seeded random-walk mutants per corpus kernel: edit, apply,
//                              validate rules, per-test execute records, EvalOutcome
//   vmcases                    hand-written kernels that exercise every trap class
//   nsga <n>                   random fitness sets -> rank_population / select_best /
//                              tournament_select
//   nsga_bin <in.bin> <keep> <out.bin> [reps]
//                              one large fitness set (n, then n costs, then n errors,
//                              native doubles) -> rank_population + select_best; writes
//                              n_fronts, front[n], crowding[n], fronts flattened, and
//                              select_best[keep] to out.bin; prints the wall seconds of
//                              rank_population + select_best (best of reps) as JSON
//   run <bench> <seed> <pop> <gens> <mode> <train> <heldout> <outdir>
//                              reference CLI run (log.csv, report.json)
//   authored <kernel.ir> <gen.json> <n_tests> <seed> <patches.txt> <budget> <tol>
//                              an authored kernel (configs 3-4): generate_tests_for,
//                              then per patch (line 0 = original) per-test execute
//                              records and the EvalOutcome

#include "evoir/cli_app.hpp"
#include "evoir/corpus.hpp"
#include "evoir/engine.hpp"

#include <json.hpp>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>

using namespace evoir;
using nlohmann::json;

namespace {

uint64_t fnv1a(const void* data, size_t n, uint64_t h = 1469598103934665603ULL) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 1099511628211ULL;
    }
    return h;
}

std::string hex64(uint64_t v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%016llx", static_cast<unsigned long long>(v));
    return buf;
}

std::string hexd(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return hex64(u);
}

// Output-map digest: names in map order, element kind, raw 32-bit words with
// every NaN canonicalised to 0x7fc00000 (x86 and sm_100 differ only in NaN
// payloads).
std::string buffers_hash(const BufferMap& m) {
    uint64_t h = 1469598103934665603ULL;
    for (const auto& [name, b] : m) {
        h = fnv1a(name.data(), name.size(), h);
        uint8_t k = static_cast<uint8_t>(b.elem);
        h = fnv1a(&k, 1, h);
        if (b.elem == TypeKind::I32) {
            h = fnv1a(b.i.data(), b.i.size() * 4, h);
        } else {
            for (float f : b.f) {
                uint32_t w;
                std::memcpy(&w, &f, 4);
                if (std::isnan(f))
                    w = 0x7fc00000u;
                h = fnv1a(&w, 4, h);
            }
        }
    }
    return hex64(h);
}

json buffer_words(const Buffer& b) {
    json j;
    j["elem"] = b.elem == TypeKind::I32 ? "i32" : "f32";
    std::string hex;
    char buf[16];
    size_t n = b.size();
    for (size_t i = 0; i < n; ++i) {
        uint32_t w;
        if (b.elem == TypeKind::I32)
            std::memcpy(&w, &b.i[i], 4);
        else
            std::memcpy(&w, &b.f[i], 4);
        std::snprintf(buf, sizeof buf, "%08x", w);
        hex += buf;
    }
    j["hex"] = hex;
    return j;
}

json test_json(const TestCase& t) {
    json j;
    for (const auto& [n, b] : t.inputs)
        j["inputs"][n] = buffer_words(b);
    for (const auto& [n, b] : t.oracle)
        j["oracle"][n] = buffer_words(b);
    for (const auto& [n, s] : t.scalars) {
        json sj;
        sj["kind"] = static_cast<int>(s.kind);
        sj["i"] = s.i;
        sj["f"] = s.f;
        sj["b"] = s.b;
        j["scalars"][n] = sj;
    }
    return j;
}

ExecConfig unit_config(ExecConfig c) {
    CostTable& t = c.cost_table;
    t.arith = t.cmp = t.select_op = t.phi = t.constant = t.br = t.intrinsic = t.getindex = 1;
    t.load_shared = t.store_shared = t.load_global = t.store_global = t.sync = t.ret = 1;
    return c;
}

const char* status_name(ExecStatus s) {
    switch (s) {
    case ExecStatus::Completed: return "completed";
    case ExecStatus::Trap: return "trap";
    case ExecStatus::BudgetExceeded: return "budget";
    }
    return "?";
}

json exec_json(const Kernel& k, const TestCase& t, const ExecConfig& cfg) {
    ExecResult r = execute(k, t, cfg);
    ExecResult u = execute(k, t, unit_config(cfg));
    json j;
    j["status"] = status_name(r.status);
    j["reason"] = r.trap_reason;
    j["cost"] = r.cost;
    j["ir"] = u.cost; // unit table: cost == dynamic instruction count
    if (r.status == ExecStatus::Completed) {
        j["out"] = buffers_hash(r.outputs);
        j["err"] = hexd(compute_error(r.outputs, t.oracle));
    }
    return j;
}

json outcome_json(const EvalOutcome& o) {
    json j;
    j["accepted"] = o.accepted;
    j["failing_test"] = o.failing_test;
    j["reason"] = o.reason;
    j["cost"] = hexd(o.fitness.cost);
    j["error"] = hexd(o.fitness.error);
    return j;
}

std::string kernel_hash(const Kernel& k) {
    std::string s = print_kernel(k);
    return hex64(fnv1a(s.data(), s.size()));
}

// ---------------------------------------------------------------------------

int cmd_corpus() {
    for (const auto& name : benchmark_names()) {
        Benchmark b = load_benchmark(name);
        json j;
        j["kind"] = "kernel";
        j["name"] = name;
        j["ir"] = print_kernel(b.kernel);
        j["improved"] = print_kernel(b.improved);
        j["reach_patch"] = json::parse(patch_to_json(b.reach_patch));
        std::cout << j.dump() << "\n";

        ExecConfig cfg = ExecConfig::for_kernel(b.kernel);
        struct Suite {
            const char* label;
            int count;
            uint64_t seed;
        };
        const Suite suites[] = {
            {"train3_seed1", 3, cli::train_seed(1)},
            {"heldout3_seed1", 3, cli::heldout_seed(1)},
            {"train16_seed1", 16, cli::train_seed(1)},
        };
        for (const auto& s : suites) {
            auto tests = generate_tests(b, s.count, s.seed);
            for (size_t ti = 0; ti < tests.size(); ++ti) {
                json t;
                t["kind"] = "test";
                t["name"] = name;
                t["suite"] = s.label;
                t["seed"] = s.seed;
                t["index"] = ti;
                t["test"] = test_json(tests[ti]);
                t["orig"] = exec_json(b.kernel, tests[ti], cfg);
                t["improved"] = exec_json(b.improved, tests[ti], cfg);
                std::cout << t.dump() << "\n";
            }
        }
    }
    return 0;
}

// Seeded random walk over each corpus kernel. Parents are drawn from the
// variants accepted so far (tolerance 0.01), so the walk reaches multi-edit
// programs, not just single mutations of the original.
int cmd_mutants(int n, int64_t budget) {
    int kidx = 0;
    for (const auto& name : benchmark_names()) {
        Benchmark b = load_benchmark(name);
        auto tests = generate_tests(b, 3, 4242);
        ExecConfig cfg = ExecConfig::for_kernel(b.kernel);
        cfg.instruction_budget = budget;

        struct Parent {
            Kernel k;
            Patch p;
        };
        std::vector<Parent> parents{{b.kernel, {}}};
        Rng pick(0xBEEF + static_cast<uint64_t>(kidx));
        for (int i = 0; i < n; ++i) {
            const Parent& par = parents[pick.index(parents.size())];
            Rng rng = Rng::stream(0x5EED, static_cast<uint64_t>(kidx), static_cast<uint64_t>(i), 77);
            DomTree dom = DomTree::build(par.k);
            MutationContext ctx(par.k, dom, rng);
            MutationResult m = random_mutation(ctx);
            json j;
            j["kind"] = "mutant";
            j["name"] = name;
            j["i"] = i;
            j["parent_patch"] = json::parse(patch_to_json(par.p));
            j["probe"] = hex64(rng.next_u64()); // pins the number of draws consumed
            if (!m) {
                j["edit"] = nullptr;
                std::cout << j.dump() << "\n";
                continue;
            }
            j["edit"] = json::parse(patch_to_json(Patch{*m}))[0];
            j["op_kind"] = operator_kind_name(operator_kind(*m));
            ApplyResult ar = apply_edit(par.k, *m);
            j["applied"] = ar.applied;
            if (!ar.applied) {
                std::cout << j.dump() << "\n";
                continue;
            }
            j["kernel_hash"] = kernel_hash(ar.kernel);
            auto errs = validate(ar.kernel);
            json rules = json::array();
            for (const auto& e : errs)
                rules.push_back(e.rule + "@" + std::to_string(e.uid));
            j["rules"] = rules;
            // Execute valid variants, and a slice of invalid ones too: the
            // interpreter is a public entry point and must agree on them.
            bool run = errs.empty() || (i % 3 == 0);
            if (run) {
                json per = json::array();
                for (const auto& t : tests)
                    per.push_back(exec_json(ar.kernel, t, cfg));
                j["tests"] = per;
                j["outcome0"] = outcome_json(evaluate_fitness(ar.kernel, tests, cfg, 0.0));
                j["outcome01"] = outcome_json(evaluate_fitness(ar.kernel, tests, cfg, 0.01));
                if (errs.empty() && evaluate_fitness(ar.kernel, tests, cfg, 0.01).accepted &&
                    par.p.size() < 6) {
                    Patch p = par.p;
                    p.push_back(*m);
                    parents.push_back({ar.kernel, p});
                }
            }
            std::cout << j.dump() << "\n";
        }
        ++kidx;
    }
    return 0;
}

// Kernels that reach every interpreter trap class, with their inputs.
int cmd_vmcases() {
    struct Case {
        const char* label;
        const char* ir;
        std::vector<std::pair<std::string, Buffer>> inputs;
        std::vector<std::pair<std::string, Scalar>> scalars;
        int64_t budget;
    };
    auto f32 = [](std::vector<float> v) { return Buffer::of_f32(std::move(v)); };
    auto i32 = [](std::vector<int32_t> v) { return Buffer::of_i32(std::move(v)); };
    std::vector<Case> cases = {
        {"missing_buffer", "kernel k(a: ptr<global> f32, b: ptr<global> f32) threads=2 {\nentry:\n  ret\n}\n",
         {{"a", f32({1})}}, {}, 1000000},
        {"buffer_type", "kernel k(a: ptr<global> i32) threads=2 {\nentry:\n  ret\n}\n",
         {{"a", f32({1})}}, {}, 1000000},
        {"missing_scalar", "kernel k(a: ptr<global> f32, n: i32) threads=2 {\nentry:\n  ret\n}\n",
         {{"a", f32({1})}}, {}, 1000000},
        {"scalar_type", "kernel k(a: ptr<global> f32, n: i32) threads=2 {\nentry:\n  ret\n}\n",
         {{"a", f32({1})}}, {{"n", Scalar::of_f32(1.0f)}}, 1000000},
        {"scalars_ok", "kernel k(a: ptr<global> f32, n: i32, x: f32, c: bool) threads=3 {\nentry:\n  %0 = tid i32\n  %1 = mul i32 %0, n\n  %2 = select f32 c, x, 2.5\n  %3 = icmp.lt i32 %1, 4\n  br %3, w, done\nw:\n  store a[%1], %2\n  br done\ndone:\n  ret\n}\n",
         {{"a", f32({0, 0, 0, 0})}}, {{"n", Scalar::of_i32(2)}, {"x", Scalar::of_f32(7.25f)}, {"c", Scalar::of_bool(true)}}, 1000000},
        {"divergence", "kernel f(out: ptr<global> f32) threads=4 shared=4 {\nentry:\n  %0 = tid i32\n  %1 = icmp.lt i32 %0, 2\n  br %1, guarded, done\nguarded:\n  sync\n  br done\ndone:\n  %2 = const f32 1.0\n  store out[%0], %2\n  ret\n}\n",
         {{"out", f32({0, 0, 0, 0})}}, {}, 1000000},
        {"divergence_two_syncs", "kernel f(out: ptr<global> f32) threads=4 {\nentry:\n  %0 = tid i32\n  %1 = icmp.lt i32 %0, 2\n  br %1, a, b\na:\n  sync\n  br done\nb:\n  sync\n  br done\ndone:\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"undef_value", "kernel f(out: ptr<global> f32) threads=2 {\nentry:\n  %0 = tid i32\n  %1 = icmp.eq i32 %0, 1\n  br %1, a, b\na:\n  %2 = const f32 3.0\n  br b\nb:\n  store out[%0], %2\n  ret\n}\n",
         {{"out", f32({0, 0})}}, {}, 1000000},
        {"undef_never_defined", "kernel f(out: ptr<global> f32) threads=2 {\nentry:\n  store out[0], %9\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"operand_type", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  %0 = const f32 1.0\n  %1 = add i32 %0, 1\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"not_pointer", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  %0 = const i32 1\n  %1 = load i32 %0[0]\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"shared_oob_load", "kernel f(out: ptr<global> f32, s: ptr<shared> f32) threads=1 shared=2 {\nentry:\n  %0 = load f32 s[2]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"shared_oob_store", "kernel f(out: ptr<global> f32, s: ptr<shared> f32) threads=1 shared=2 {\nentry:\n  store s[-1], 1.0\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"shared_uninit", "kernel f(out: ptr<global> f32, s: ptr<shared> f32) threads=2 shared=2 {\nentry:\n  %0 = tid i32\n  store s[%0], 1.0\n  %1 = load f32 s[1]\n  store out[%0], %1\n  ret\n}\n",
         {{"out", f32({0, 0})}}, {}, 1000000},
        {"shared_type", "kernel f(out: ptr<global> f32, s: ptr<shared> f32) threads=1 shared=2 {\nentry:\n  store s[0], 3\n  %0 = load f32 s[0]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"global_oob_load", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = load f32 out[1]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"global_oob_store", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  store out[9], 1.0\n  ret\n}\n",
         {{"out", f32({0, 0})}}, {}, 1000000},
        {"global_load_type", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = load i32 out[0]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"store_bool", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  store out[0], true\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"global_store_type", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  store out[0], 5\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"phi_no_incoming", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  br b\nc:\n  br b\nb:\n  %0 = phi i32 [1, c]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"fell_off", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = tid i32\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"unknown_block", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  br nowhere\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"phi_outside_entry", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = phi i32 [1, entry]\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"sdiv_zero", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  %0 = const i32 4\n  %1 = const i32 0\n  %2 = sdiv i32 %0, %1\n  store out[0], %2\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"sdiv_overflow", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  %0 = const i32 -2147483648\n  %1 = sdiv i32 %0, -1\n  store out[0], %1\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"sdiv_trunc", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  %1 = sdiv i32 -7, 2\n  %2 = mul i32 %1, 2147483647\n  %3 = add i32 %2, 2147483647\n  %4 = sub i32 %3, -5\n  store out[0], %4\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"select_type", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = select f32 true, 1, 2.0\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"store_nonscalar", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  store out[0], out\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"getindex_space", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  %0 = getindex ptr<shared> out, 1\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 1000000},
        {"getindex_ok", "kernel f(out: ptr<global> f32, s: ptr<shared> f32) threads=2 shared=4 {\nentry:\n  %0 = tid i32\n  %1 = getindex ptr<global> out, 1\n  %2 = getindex ptr<shared> s, %0\n  store %2[1], 2.0\n  %3 = load f32 s[1]\n  store %1[%0], %3\n  ret\n}\n",
         {{"out", f32({0, 0, 0})}}, {}, 1000000},
        {"budget", "kernel f(out: ptr<global> f32) threads=1 {\nentry:\n  br spin\nspin:\n  br spin\n}\n",
         {{"out", f32({0})}}, {}, 10000},
        {"budget_second_thread", "kernel f(out: ptr<global> f32) threads=3 {\nentry:\n  %0 = tid i32\n  %1 = icmp.eq i32 %0, 1\n  br %1, spin, done\nspin:\n  %2 = phi i32 [0, entry], [%3, spin]\n  %3 = add i32 %2, 1\n  br spin\ndone:\n  ret\n}\n",
         {{"out", f32({0})}}, {}, 5000},
        {"float_semantics", "kernel f(out: ptr<global> f32, b: ptr<global> i32) threads=1 {\nentry:\n  %0 = fdiv f32 1.0, 0.0\n  %1 = fdiv f32 0.0, 0.0\n  %2 = fcmp.ne f32 %1, %1\n  %3 = fcmp.eq f32 %1, %1\n  %4 = fcmp.lt f32 %1, 1.0\n  %5 = select i32 %2, 1, 0\n  %6 = select i32 %3, 10, 0\n  %7 = select i32 %4, 100, 0\n  %8 = add i32 %5, %6\n  %9 = add i32 %8, %7\n  store b[0], %9\n  store out[0], %0\n  %10 = fmul f32 1.0e-30, 1.0e-10\n  store out[1], %10\n  %11 = fsub f32 %0, %0\n  store out[2], %11\n  %12 = fdiv f32 1.0, 3.0\n  store out[3], %12\n  ret\n}\n",
         {{"out", f32({0, 0, 0, 0})}, {"b", i32({0})}}, {}, 1000000},
        {"phi_parallel_copy", "kernel f(out: ptr<global> i32) threads=1 {\nentry:\n  br loop\nloop:\n  %0 = phi i32 [1, entry], [%1, loop]\n  %1 = phi i32 [2, entry], [%0, loop]\n  %2 = phi i32 [0, entry], [%3, loop]\n  %3 = add i32 %2, 1\n  %4 = icmp.lt i32 %3, 5\n  br %4, loop, done\ndone:\n  %5 = mul i32 %0, 10\n  %6 = add i32 %5, %1\n  store out[0], %6\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
        {"waw_same_phase", "kernel f(out: ptr<global> i32, s: ptr<shared> i32) threads=4 shared=2 {\nentry:\n  %0 = tid i32\n  store s[0], %0\n  %1 = load i32 s[0]\n  store out[%0], %1\n  sync\n  %2 = load i32 s[0]\n  %3 = add i32 %0, 4\n  store out[%3], %2\n  ret\n}\n",
         {{"out", i32({0, 0, 0, 0, 0, 0, 0, 0})}}, {}, 1000000},
        {"raw_cross_thread", "kernel f(out: ptr<global> i32, s: ptr<shared> i32) threads=4 shared=4 {\nentry:\n  %0 = tid i32\n  %1 = add i32 %0, 1\n  store s[%1], %0\n  %2 = load i32 s[%0]\n  store out[%0], %2\n  ret\n}\n",
         {{"out", i32({0, 0, 0, 0})}}, {}, 1000000},
        {"global_cross_thread", "kernel f(out: ptr<global> i32) threads=4 {\nentry:\n  %0 = tid i32\n  %1 = add i32 %0, 1\n  %2 = load i32 out[%0]\n  %3 = add i32 %2, 10\n  store out[%1], %3\n  ret\n}\n",
         {{"out", i32({1, 0, 0, 0, 0})}}, {}, 1000000},
        {"multi_phase_values", "kernel f(out: ptr<global> i32, s: ptr<shared> i32) threads=3 shared=3 {\nentry:\n  %0 = tid i32\n  %1 = mul i32 %0, 7\n  store s[%0], %1\n  sync\n  %2 = add i32 %0, 1\n  %3 = icmp.eq i32 %2, 3\n  %4 = select i32 %3, 0, %2\n  %5 = load i32 s[%4]\n  sync\n  %6 = add i32 %5, %1\n  store out[%0], %6\n  ret\n}\n",
         {{"out", i32({0, 0, 0})}}, {}, 1000000},
        {"nthreads", "kernel f(out: ptr<global> i32) threads=5 {\nentry:\n  %0 = tid i32\n  %1 = nthreads i32\n  %2 = mul i32 %1, 100\n  %3 = add i32 %2, %0\n  store out[%0], %3\n  ret\n}\n",
         {{"out", i32({0, 0, 0, 0, 0})}}, {}, 1000000},
        {"ret_vs_sync", "kernel f(out: ptr<global> i32) threads=2 {\nentry:\n  %0 = tid i32\n  %1 = icmp.eq i32 %0, 0\n  br %1, a, b\na:\n  ret\nb:\n  sync\n  ret\n}\n",
         {{"out", i32({0})}}, {}, 1000000},
    };
    for (const auto& c : cases) {
        Kernel k = parse_kernel(c.ir);
        TestCase t;
        for (const auto& [n, b] : c.inputs)
            t.inputs[n] = b;
        for (const auto& [n, s] : c.scalars)
            t.scalars[n] = s;
        ExecConfig cfg = ExecConfig::for_kernel(k);
        cfg.instruction_budget = c.budget;
        ExecResult r = execute(k, t, cfg);
        // Oracle: the case's own outputs when it completes (error 0 path),
        // the inputs otherwise.
        t.oracle = r.status == ExecStatus::Completed ? r.outputs : t.inputs;
        json j;
        j["kind"] = "vmcase";
        j["label"] = c.label;
        j["ir"] = print_kernel(k);
        j["valid"] = validate(k).empty();
        j["budget"] = c.budget;
        j["test"] = test_json(t);
        j["exec"] = exec_json(k, t, cfg);
        if (r.status == ExecStatus::Completed) {
            json outs;
            for (const auto& [n, b] : r.outputs)
                outs[n] = buffer_words(b);
            j["outputs"] = outs;
        }
        j["outcome"] = outcome_json(evaluate_fitness(k, {t}, cfg, 0.0));
        std::cout << j.dump() << "\n";
    }
    return 0;
}

int cmd_nsga(int n) {
    Rng rng(20040814);
    for (int c = 0; c < n; ++c) {
        size_t size = 1 + rng.index(c < n / 2 ? 24 : 400);
        int levels = 1 + static_cast<int>(rng.index(12));
        std::vector<FitnessVector> fits(size);
        for (auto& f : fits) {
            f.cost = 1000.0 + static_cast<double>(rng.index(static_cast<size_t>(levels) * 7)) * 8.0;
            f.error = rng.chance(0.4) ? 0.0 : static_cast<double>(rng.index(static_cast<size_t>(levels))) / 97.0;
            if (rng.chance(0.05))
                f.cost += rng.uniform();
        }
        ParetoRank r = rank_population(fits);
        json j;
        j["kind"] = "nsga";
        json fj = json::array();
        for (const auto& f : fits)
            fj.push_back({hexd(f.cost), hexd(f.error)});
        j["fits"] = fj;
        j["fronts"] = r.fronts;
        json cj = json::array();
        for (double d : r.crowding)
            cj.push_back(hexd(d));
        j["crowding"] = cj;
        size_t keep = size / 4 == 0 ? size : size / 4 + rng.index(size - size / 4 + 1);
        j["keep"] = keep;
        j["select_best"] = select_best(r, keep);
        uint64_t tseed = rng.next_u64();
        Rng trng(tseed);
        j["tseed"] = hex64(tseed);
        j["tournament"] = tournament_select(r, size, size, trng);
        std::cout << j.dump() << "\n";
    }
    return 0;
}

int cmd_run(int argc, char** argv) {
    if (argc < 10) {
        std::cerr << "usage: run <bench> <seed> <pop> <gens> <mode> <train> <heldout> <outdir>\n";
        return 1;
    }
    cli::RunOptions opt;
    opt.bench = argv[2];
    opt.seed = std::stoull(argv[3]);
    opt.pop = std::stoi(argv[4]);
    opt.generations = std::stoi(argv[5]);
    opt.mode = argv[6];
    opt.train_tests = std::stoi(argv[7]);
    opt.heldout_tests = std::stoi(argv[8]);
    opt.out_dir = argv[9];
    if (argc > 10)
        opt.jobs = std::stoi(argv[10]);
    return cli::cmd_run(opt);
}

std::string slurp(const std::string& path) {
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

int cmd_authored(int argc, char** argv) {
    if (argc < 9) {
        std::cerr << "usage: ref_dump authored <ir> <gen.json> <n_tests> <seed> <patches> <budget> <tol>\n";
        return 1;
    }
    const Kernel k = parse_kernel(slurp(argv[2]));
    const GeneratorSpec gen = generator_spec_from_json(slurp(argv[3]));
    const int n_tests = std::stoi(argv[4]);
    const uint64_t seed = std::stoull(argv[5]);
    const double tol = std::stod(argv[8]);
    auto tests = generate_tests_for(k, gen, n_tests, seed);
    ExecConfig cfg = ExecConfig::for_kernel(k);
    cfg.instruction_budget = std::stoll(argv[7]);
    std::ifstream in(argv[6]);
    std::string line;
    int i = 0;
    while (std::getline(in, line)) {
        if (line.empty())
            continue;
        json j;
        j["kind"] = "authored";
        j["i"] = i++;
        j["patch"] = json::parse(line);
        const Kernel v = apply_patch(k, patch_from_json(line)).kernel;
        j["valid"] = is_valid(v);
        json per = json::array();
        for (const auto& t : tests)
            per.push_back(exec_json(v, t, cfg));
        j["tests"] = per;
        const EvalOutcome o = evaluate_fitness(v, tests, cfg, tol);
        j["outcome"] = {{"accepted", o.accepted}, {"failing_test", o.failing_test},
                        {"reason", o.reason}, {"cost", hexd(o.fitness.cost)},
                        {"error", hexd(o.fitness.error)}};
        std::cout << j.dump() << "\n";
    }
    return 0;
}

int cmd_nsga_bin(int argc, char** argv) {
    if (argc < 5) {
        std::cerr << "usage: nsga_bin <in.bin> <keep> <out.bin> [reps]\n";
        return 1;
    }
    std::ifstream in(argv[2], std::ios::binary);
    int64_t n = 0;
    in.read(reinterpret_cast<char*>(&n), 8);
    std::vector<double> c(static_cast<size_t>(n)), e(static_cast<size_t>(n));
    in.read(reinterpret_cast<char*>(c.data()), n * 8);
    in.read(reinterpret_cast<char*>(e.data()), n * 8);
    std::vector<FitnessVector> fits(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i)
        fits[static_cast<size_t>(i)] = FitnessVector{c[static_cast<size_t>(i)], e[static_cast<size_t>(i)]};
    const size_t keep = std::stoull(argv[3]);
    const int reps = argc > 5 ? std::stoi(argv[5]) : 1;
    double best_s = 1e300, rank_s = 1e300;
    ParetoRank r;
    std::vector<int> sel;
    for (int k = 0; k < reps; ++k) {
        auto t0 = std::chrono::steady_clock::now();
        r = rank_population(fits);
        auto t1 = std::chrono::steady_clock::now();
        sel = select_best(r, keep);
        auto t2 = std::chrono::steady_clock::now();
        best_s = std::min(best_s, std::chrono::duration<double>(t2 - t0).count());
        rank_s = std::min(rank_s, std::chrono::duration<double>(t1 - t0).count());
    }
    std::ofstream out(argv[4], std::ios::binary);
    const int32_t F = static_cast<int32_t>(r.fronts.size());
    out.write(reinterpret_cast<const char*>(&F), 4);
    out.write(reinterpret_cast<const char*>(r.front.data()), n * 4);
    out.write(reinterpret_cast<const char*>(r.crowding.data()), n * 8);
    for (const auto& f : r.fronts)
        out.write(reinterpret_cast<const char*>(f.data()), static_cast<std::streamsize>(f.size() * 4));
    out.write(reinterpret_cast<const char*>(sel.data()), static_cast<std::streamsize>(sel.size() * 4));
    std::printf("{\"n\": %lld, \"fronts\": %d, \"rank_select_s\": %.6f, \"rank_s\": %.6f}\n",
                static_cast<long long>(n), F, best_s, rank_s);
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: ref_dump corpus|mutants|vmcases|nsga|run ...\n";
        return 1;
    }
    std::string cmd = argv[1];
    if (cmd == "corpus")
        return cmd_corpus();
    if (cmd == "mutants")
        return cmd_mutants(argc > 2 ? std::stoi(argv[2]) : 200,
                           argc > 3 ? std::stoll(argv[3]) : 1000000);
    if (cmd == "vmcases")
        return cmd_vmcases();
    if (cmd == "nsga")
        return cmd_nsga(argc > 2 ? std::stoi(argv[2]) : 200);
    if (cmd == "run")
        return cmd_run(argc, argv);
    if (cmd == "nsga_bin")
        return cmd_nsga_bin(argc, argv);
    if (cmd == "authored")
        return cmd_authored(argc, argv);
    std::cerr << "unknown subcommand\n";
    return 1;
}
