// Host-side cost of candidate production (CPU only, no device): per-stage
// timing of the work one search generation does per attempt -- dominator
// tree + mutation context per parent, random_mutation, apply_edit, validate,
// crossover apply_patch, device encoding.
//
//   g++ -std=c++20 -O2 -Iinclude -Ipaper_2004_08140_b200/csrc -I$JSON_DIR \
//       scripts/native/host_cost.cpp paper_2004_08140_b200/libgevo_b200.so -o /tmp/host_cost
//   /tmp/host_cost nw-sync [max walk depth, default 6]
#include "evoir/corpus.hpp"
#include "evoir/operators.hpp"
#include "host/encode.hpp"

#include <chrono>
#include <cstdio>
#include <cstdlib>

using namespace evoir;
using Clock = std::chrono::steady_clock;

static double us(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double, std::micro>(b - a).count();
}

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "nw-sync";
    const int max_depth = argc > 2 ? std::max(1, std::atoi(argv[2])) : 6;
    const Benchmark bm = load_benchmark(name);
    const Kernel& orig = bm.kernel;
    // parents: accepted-by-validate random walks of up to 6 edits
    std::vector<Kernel> parents;
    std::vector<Patch> patches;
    Rng walk(7);
    while (parents.size() < 256) {
        Kernel k = orig;
        Patch p;
        const int depth = 1 + static_cast<int>(walk.index(static_cast<size_t>(max_depth)));
        for (int d = 0; d < depth; ++d) {
            const DomTree dom = DomTree::build(k);
            MutationContext ctx(k, dom, walk);
            auto m = random_mutation(ctx);
            if (!m)
                continue;
            ApplyResult ap = apply_edit(k, *m);
            if (ap.applied && is_valid(ap.kernel)) {
                k = std::move(ap.kernel);
                p.push_back(*m);
            }
        }
        parents.push_back(std::move(k));
        patches.push_back(std::move(p));
    }
    const int per = 24;
    double t_ctx = 0, t_mut = 0, t_apply = 0, t_valid = 0, t_cx = 0, t_cxvalid = 0;
    double t_kind[kOperatorCount] = {};
    size_t n_kind[kOperatorCount] = {};
    size_t n_mut = 0, n_apply = 0, n_cx = 0;
    std::vector<Kernel> cands;
    Rng rng(11);
    for (size_t i = 0; i < parents.size(); ++i) {
        auto t0 = Clock::now();
        const DomTree dom = DomTree::build(parents[i]);
        MutationContext ctx(parents[i], dom, rng);
        auto t1 = Clock::now();
        t_ctx += us(t0, t1);
        for (int a = 0; a < per; ++a) {
            auto u0 = Clock::now();
            auto m = random_mutation(ctx);
            auto u1 = Clock::now();
            t_mut += us(u0, u1);
            ++n_mut;
            if (!m)
                continue;
            t_kind[static_cast<size_t>(operator_kind(*m))] += us(u0, u1);
            ++n_kind[static_cast<size_t>(operator_kind(*m))];
            ApplyResult ap = apply_edit(parents[i], *m);
            auto u2 = Clock::now();
            t_apply += us(u1, u2);
            if (!ap.applied)
                continue;
            ++n_apply;
            const bool ok = is_valid(ap.kernel);
            t_valid += us(u2, Clock::now());
            if (ok && cands.size() < 4096)
                cands.push_back(std::move(ap.kernel));
        }
        // crossover with the next parent
        const size_t j = (i + 1) % parents.size();
        for (int a = 0; a < 8; ++a) {
            auto u0 = Clock::now();
            auto [pa, pb] = crossover_messy(patches[i], patches[j], rng);
            PatchResult ra = apply_patch(orig, pa), rb = apply_patch(orig, pb);
            auto u1 = Clock::now();
            t_cx += us(u0, u1);
            (void)is_valid(ra.kernel);
            (void)is_valid(rb.kernel);
            t_cxvalid += us(u1, Clock::now());
            n_cx += 2;
        }
    }
    // device encoding of the candidates (host side only)
    const std::vector<TestCase> tests = generate_inputs_for(bm.gen, 16, 1); // (no oracles: host only)
    const b200::SuiteImage suite = b200::build_suite(orig.params, tests);
    auto e0 = Clock::now();
    b200::BatchImage batch(suite);
    for (const Kernel& k : cands)
        batch.add(k);
    batch.blob();
    const double t_enc = us(e0, Clock::now());
    std::printf("{\"bench\": \"%s\", \"parents\": %zu, \"ctx_us_per_parent\": %.2f, "
                "\"mutation_us\": %.2f, \"apply_edit_us\": %.2f, \"validate_us\": %.2f, "
                "\"cx_apply_patch_us_per_child\": %.2f, \"cx_validate_us_per_child\": %.2f, "
                "\"encode_us_per_variant\": %.2f, \"candidates\": %zu, \"mutation_us_by_kind\": {",
                name.c_str(), parents.size(), t_ctx / parents.size(), t_mut / n_mut,
                t_apply / n_mut, t_valid / std::max<size_t>(n_apply, 1), t_cx / n_cx,
                t_cxvalid / n_cx, t_enc / std::max<size_t>(cands.size(), 1), cands.size());
    for (size_t o = 0; o < kOperatorCount; ++o)
        std::printf("%s\"%s\": %.2f", o ? ", " : "", operator_kind_name(static_cast<OperatorKind>(o)),
                    t_kind[o] / std::max<size_t>(n_kind[o], 1));
    std::printf("}}\n");
    return 0;
}
