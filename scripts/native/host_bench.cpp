// Host candidate-production microbenchmark (no GPU): per-call cost of the
// pieces the search engine runs for every attempt -- random_mutation,
// apply_edit, apply_patch (crossover children are re-applied from the
// original), is_valid, Kernel copy -- plus two equivalence checks: in-place
// apply_patch == the apply_edit fold, and the verdict-only is_valid ==
// validate().empty() on unfiltered (mostly invalid) children. Build:
//   g++ -O2 -std=c++20 -Iinclude scripts/native/host_bench.cpp \
//       -Lpaper_2004_08140_b200 -lgevo_b200 -Wl,-rpath,$PWD/paper_2004_08140_b200 -o /tmp/host_bench
#include "evoir/corpus.hpp"
#include "evoir/genome.hpp"
#include "evoir/operators.hpp"
#include "evoir/ir.hpp"

#include <chrono>
#include <cstdio>
#include <string>
#include <vector>

using namespace evoir;
using clk = std::chrono::steady_clock;

static double us(clk::time_point a, size_t n) {
    return std::chrono::duration<double, std::micro>(clk::now() - a).count() / static_cast<double>(n);
}

int main(int argc, char** argv) {
    const std::string name = argc > 1 ? argv[1] : "bfs-load";
    const int depth = argc > 2 ? std::atoi(argv[2]) : 8;
    Benchmark b = load_benchmark(name);
    Rng rng(42);
    // grow patches by random valid walks
    std::vector<Patch> patches;
    std::vector<Kernel> kernels;
    for (int i = 0; i < 400; ++i) {
        Kernel k = b.kernel;
        Patch p;
        for (int d = 0; d < depth; ++d) {
            DomTree dom = DomTree::build(k);
            MutationContext ctx(k, dom, rng);
            MutationResult m = random_mutation(ctx);
            if (!m)
                continue;
            ApplyResult ap = apply_edit(k, *m);
            if (!ap.applied || !is_valid(ap.kernel))
                continue;
            k = std::move(ap.kernel);
            p.push_back(*m);
        }
        patches.push_back(p);
        kernels.push_back(k);
    }
    size_t edits = 0;
    for (auto& p : patches)
        edits += p.size();
    std::printf("%s: %zu patches, mean %.1f edits, %zu instructions in the last\n", name.c_str(),
                patches.size(), double(edits) / patches.size(), kernels.back().instruction_count());
    // in-place apply_patch == left fold of apply_edit (also on crossover
    // children, whose edits often no longer apply)
    size_t mism = 0, dropped = 0, checked = 0;
    for (size_t i = 0; i + 1 < patches.size(); ++i) {
        auto [ca, cb] = crossover_messy(patches[i], patches[i + 1], rng);
        for (const Patch* pp : {&patches[i], &ca, &cb}) {
            Kernel fold = b.kernel;
            Patch applied;
            for (const Edit& e : *pp) {
                ApplyResult s = apply_edit(fold, e);
                if (!s.applied)
                    continue;
                fold = std::move(s.kernel);
                applied.push_back(e);
            }
            PatchResult r = apply_patch(b.kernel, *pp);
            dropped += pp->size() - r.applied.size();
            ++checked;
            if (!(r.kernel == fold) || !(r.applied == applied))
                ++mism;
        }
    }
    std::printf("apply_patch vs apply_edit fold: %zu patches, %zu dropped edits, %zu mismatches\n",
                checked, dropped, mism);
    if (mism)
        return 1;
    // verdict-only is_valid == validate().empty() on unfiltered children:
    // random mutations of every walk kernel and the crossover children (most
    // of them invalid, across every rule)
    size_t vchecked = 0, vmism = 0, vinvalid = 0;
    auto vcheck = [&](const Kernel& k) {
        const bool full = validate(k).empty();
        ++vchecked;
        vinvalid += !full;
        if (is_valid(k) != full)
            ++vmism;
    };
    for (size_t i = 0; i < kernels.size(); ++i) {
        const DomTree dom = DomTree::build(kernels[i]);
        MutationContext ctx(kernels[i], dom, rng);
        for (int j = 0; j < 12; ++j) {
            MutationResult m = random_mutation(ctx);
            if (!m)
                continue;
            ApplyResult ap = apply_edit(kernels[i], *m);
            if (ap.applied)
                vcheck(ap.kernel);
        }
        if (i + 1 < patches.size()) {
            auto [ca, cb] = crossover_messy(patches[i], patches[i + 1], rng);
            vcheck(apply_patch(b.kernel, ca).kernel);
            vcheck(apply_patch(b.kernel, cb).kernel);
        }
    }
    std::printf("is_valid vs validate: %zu kernels (%zu invalid), %zu validity mismatches\n", vchecked,
                vinvalid, vmism);
    if (vmism)
        return 1;
    auto t = clk::now();
    for (auto& p : patches)
        (void)apply_patch(b.kernel, p);
    std::printf("apply_patch        %8.2f us\n", us(t, patches.size()));
    t = clk::now();
    size_t ok = 0;
    for (auto& k : kernels)
        ok += is_valid(k);
    std::printf("is_valid           %8.2f us (%zu valid)\n", us(t, kernels.size()), ok);
    t = clk::now();
    for (auto& k : kernels)
        (void)DomTree::build(k);
    std::printf("DomTree::build     %8.2f us\n", us(t, kernels.size()));
    t = clk::now();
    std::vector<Kernel> copies;
    copies.reserve(kernels.size());
    for (auto& k : kernels)
        copies.push_back(k);
    std::printf("Kernel copy        %8.2f us\n", us(t, kernels.size()));
    t = clk::now();
    size_t n = 0;
    for (size_t i = 0; i + 1 < patches.size(); i += 2, ++n)
        (void)crossover_messy(patches[i], patches[i + 1], rng);
    std::printf("crossover_messy    %8.2f us\n", us(t, n));
    t = clk::now();
    n = 0;
    for (auto& k : kernels) {
        DomTree dom = DomTree::build(k);
        MutationContext ctx(k, dom, rng);
        for (int j = 0; j < 8; ++j, ++n) {
            MutationResult m = random_mutation(ctx);
            if (m)
                (void)apply_edit(k, *m);
        }
    }
    std::printf("mutation+apply_edit %7.2f us\n", us(t, n));
    return 0;
}
