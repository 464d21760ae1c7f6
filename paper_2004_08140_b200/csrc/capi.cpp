// C ABI (include/gevo_b200.h) over the C++ host and the device runtime.
#include "../../include/gevo_b200.h"

#include "evoir/cli_app.hpp"
#include "evoir/corpus.hpp"
#include "evoir/operators.hpp"
#include "host/runtime.hpp"

#include <json.hpp>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

using namespace evoir;

struct gevo_suite {
    Kernel kernel;
    std::unique_ptr<b200::Device> own_device; // non-default ordinals
    std::unique_ptr<b200::DeviceSuite> suite;
};

struct gevo_batch {
    gevo_suite* suite;
    std::unique_ptr<b200::BatchImage> image;
    std::shared_ptr<b200::ResidentBatch> resident;
};

namespace {

thread_local std::string g_error;

char* dup(const std::string& s) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    return p;
}

template <typename Fn>
int guard(Fn&& fn) {
    try {
        fn();
        return GEVO_SUCCESS;
    } catch (const DeviceUnavailable& e) {
        g_error = e.what();
        return GEVO_E_NODEVICE;
    } catch (const InitFailure& e) {
        g_error = e.what();
        return GEVO_E_INIT;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return GEVO_E_INVALID;
    } catch (const ParseError& e) {
        g_error = e.what();
        return GEVO_E_INVALID;
    } catch (const std::exception& e) {
        g_error = e.what();
        const std::string w = e.what();
        return w.find("CUDA") != std::string::npos ? GEVO_E_CUDA : GEVO_E_INVALID;
    }
}

b200::Device& device_for(int ordinal, std::unique_ptr<b200::Device>& own) {
    b200::Device& def = b200::Device::default_device();
    if (ordinal < 0 || ordinal == def.ordinal())
        return def;
    own = std::make_unique<b200::Device>(ordinal);
    return *own;
}

ExecConfig exec_from(const gevo_exec_config* c) {
    ExecConfig e;
    e.thread_count = c->threads;
    e.shared_words = c->shared_words;
    e.instruction_budget = c->instruction_budget;
    int64_t* f[14] = {&e.cost_table.arith,       &e.cost_table.cmp,          &e.cost_table.select_op,
                      &e.cost_table.phi,         &e.cost_table.constant,     &e.cost_table.br,
                      &e.cost_table.intrinsic,   &e.cost_table.getindex,     &e.cost_table.load_shared,
                      &e.cost_table.store_shared, &e.cost_table.load_global, &e.cost_table.store_global,
                      &e.cost_table.sync,        &e.cost_table.ret};
    for (int i = 0; i < 14; ++i)
        *f[i] = c->cost_table[i];
    return e;
}

std::string hex_double(double d) {
    uint64_t u;
    std::memcpy(&u, &d, 8);
    char b[24];
    std::snprintf(b, sizeof b, "%016llx", static_cast<unsigned long long>(u));
    return b;
}

nlohmann::json buffers_hex(const BufferMap& m) {
    nlohmann::json j = nlohmann::json::object();
    for (const auto& [name, buf] : m) {
        std::string h;
        char w[12];
        for (size_t e = 0; e < buf.size(); ++e) {
            uint32_t x;
            if (buf.elem == TypeKind::I32)
                std::memcpy(&x, &buf.i[e], 4);
            else
                std::memcpy(&x, &buf.f[e], 4);
            std::snprintf(w, sizeof w, "%08x", x);
            h += w;
        }
        j[name] = {{"type", buf.elem == TypeKind::I32 ? "i32" : "f32"}, {"hex", h}};
    }
    return j;
}

void fill_stats(gevo_eval_stats* s, float ms, uint64_t h2d, uint64_t d2h, int launches) {
    if (!s)
        return;
    s->device_ms = ms;
    s->h2d_bytes = h2d;
    s->d2h_bytes = d2h;
    s->launches = launches;
    s->pad = 0;
}

} // namespace

extern "C" {

int gevo_abi_version(void) { return GEVO_ABI_VERSION; }

int gevo_device_count(void) {
    int n = 0;
    if (guard([&] { (void)b200::Device::default_device(); }) != GEVO_SUCCESS)
        return 0;
    n = 1;
    return n;
}

int gevo_set_stream(void* stream) {
    return guard([&] { b200::Device::default_device().set_stream(stream); });
}

int gevo_spin_counters(uint64_t* out2, int reset) {
    return guard([&] { b200::spin_counters(b200::Device::default_device(), out2, reset != 0); });
}

int gevo_set_collective(int rank, int world, gevo_allgather_fn fn, void* ctx) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world || (world > 1 && !fn))
            throw std::invalid_argument("gevo_set_collective: bad rank / world / callback");
        b200::Collective c;
        c.rank = rank;
        c.world = world;
        c.allgather = fn;
        c.ctx = ctx;
        b200::set_collective(c);
    });
}

int gevo_nccl_unique_id(void* out128) {
    return guard([&] { b200::nccl_unique_id(out128); });
}

int gevo_set_nccl(int rank, int world, const void* id128) {
    return guard([&] { b200::set_nccl(rank, world, id128); });
}

int gevo_work_counters(uint64_t* out2, int reset) {
    return guard([&] { b200::work_counters(b200::Device::default_device(), out2, reset != 0); });
}

int gevo_tp_counters(uint64_t* out2, int reset) {
    return guard([&] { b200::tp_counters(b200::Device::default_device(), out2, reset != 0); });
}

const char* gevo_last_error(void) { return g_error.c_str(); }

void gevo_free(void* p) { std::free(p); }

int gevo_suite_from_benchmark(const char* bench, int n_tests, uint64_t seed, int device,
                              gevo_suite** out) {
    return guard([&] {
        auto s = std::make_unique<gevo_suite>();
        b200::Device& dev = device_for(device, s->own_device);
        const Benchmark b = load_benchmark(bench);
        s->kernel = b.kernel;
        const std::vector<TestCase> tests = generate_tests(b, n_tests, seed);
        s->suite = std::make_unique<b200::DeviceSuite>(dev, b200::build_suite(b.kernel.params, tests));
        *out = s.release();
    });
}

int gevo_suite_from_json(const char* kernel_ir, const char* const* tests_json, int n_tests,
                         int device, gevo_suite** out) {
    return guard([&] {
        auto s = std::make_unique<gevo_suite>();
        b200::Device& dev = device_for(device, s->own_device);
        s->kernel = parse_kernel(kernel_ir);
        std::vector<TestCase> tests;
        for (int i = 0; i < n_tests; ++i)
            tests.push_back(testcase_from_json(tests_json[i]));
        s->suite = std::make_unique<b200::DeviceSuite>(dev, b200::build_suite(s->kernel.params, tests));
        *out = s.release();
    });
}

void gevo_suite_free(gevo_suite* s) { delete s; }

int gevo_suite_n_tests(const gevo_suite* s) { return s ? s->suite->image().n_tests : 0; }

int gevo_suite_exec_config(const gevo_suite* s, gevo_exec_config* out) {
    return guard([&] {
        const b200::ExecImage e = b200::exec_image(ExecConfig::for_kernel(s->kernel));
        out->threads = e.threads;
        out->shared_words = e.shared_words;
        out->instruction_budget = e.budget;
        for (int i = 0; i < 14; ++i)
            out->cost_table[i] = e.cost[static_cast<size_t>(i)];
    });
}

int gevo_suite_kernel_ir(const gevo_suite* s, char** ir) {
    return guard([&] { *ir = dup(print_kernel(s->kernel)); });
}

int gevo_batch_create(gevo_suite* s, gevo_batch** out) {
    return guard([&] {
        auto b = std::make_unique<gevo_batch>();
        b->suite = s;
        b->image = std::make_unique<b200::BatchImage>(s->suite->image());
        *out = b.release();
    });
}

// The resident copy of a batch is dropped before its host image changes; an
// evaluation still in flight (gevo_eval_resident_async without _wait) reads
// that image, so changing the batch then is a usage error.
static void drop_resident(gevo_batch* b) {
    if (b->resident && b200::resident_pending(*b->resident))
        throw std::logic_error("batch has an evaluation in flight: call gevo_eval_resident_wait first");
    b->resident.reset();
}

int gevo_batch_add_ir(gevo_batch* b, const char* kernel_ir) {
    return guard([&] {
        drop_resident(b); // first: it holds a host registration of the blob
        b->image->add(parse_kernel(kernel_ir));
    });
}

int gevo_batch_add_patch(gevo_batch* b, const char* patch_json) {
    return guard([&] {
        drop_resident(b); // first: it holds a host registration of the blob
        b->image->add(apply_patch(b->suite->kernel, patch_from_json(patch_json)).kernel);
    });
}

int gevo_batch_size(const gevo_batch* b) { return b ? static_cast<int>(b->image->size()) : 0; }

int gevo_batch_blob(gevo_batch* b, const void** data, size_t* bytes) {
    return guard([&] {
        const auto& blob = b->image->blob();
        *data = blob.data();
        *bytes = blob.size();
    });
}

void gevo_batch_free(gevo_batch* b) { delete b; }

int gevo_eval(gevo_batch* b, const gevo_exec_config* cfg, double tolerance, uint32_t flags,
              gevo_variant_record* out_variants, gevo_test_record* out_tests,
              gevo_eval_stats* stats) {
    return guard([&] {
        if (b->suite->suite->image().n_tests == 0)
            throw std::invalid_argument("suite has no test cases");
        b200::EvalOptions opt;
        opt.tolerance = tolerance;
        opt.early_exit = (flags & GEVO_EVAL_EARLY_EXIT) != 0;
        opt.sequential = (flags & GEVO_EVAL_SEQUENTIAL) != 0;
        opt.want_tests = out_tests && (flags & GEVO_EVAL_TESTS);
        const b200::EvalResult r =
            b200::evaluate(*b->suite->suite, *b->image, b200::exec_image(exec_from(cfg)), opt);
        if (out_variants && !r.variants.empty())
            std::memcpy(out_variants, r.variants.data(), r.variants.size() * sizeof(gevo_variant_record));
        if (opt.want_tests && !r.tests.empty())
            std::memcpy(out_tests, r.tests.data(), r.tests.size() * sizeof(gevo_test_record));
        fill_stats(stats, r.kernel_ms, r.h2d_bytes, r.d2h_bytes, r.launches);
    });
}

int gevo_eval_resident_async(gevo_batch* b, const gevo_exec_config* cfg, double tolerance,
                             uint32_t flags) {
    return guard([&] {
        const bool upload = (flags & GEVO_EVAL_UPLOAD) != 0;
        if (!b->resident)
            b->resident = b200::make_resident(*b->suite->suite, *b->image);
        b200::EvalOptions opt;
        opt.tolerance = tolerance;
        opt.early_exit = (flags & GEVO_EVAL_EARLY_EXIT) != 0;
        opt.sequential = (flags & GEVO_EVAL_SEQUENTIAL) != 0;
        b200::evaluate_resident_async(*b->resident, b200::exec_image(exec_from(cfg)), opt,
                                      upload ? &b->image->blob() : nullptr);
    });
}

int gevo_eval_resident_wait(gevo_batch* b, gevo_variant_record* out_variants, gevo_eval_stats* stats) {
    return guard([&] {
        if (!b->resident)
            throw std::invalid_argument("batch is not resident");
        std::vector<gevo_variant_record> recs;
        int launches = 0;
        const float ms = b200::wait_resident(*b->resident, out_variants ? &recs : nullptr, &launches);
        if (out_variants && !recs.empty())
            std::memcpy(out_variants, recs.data(), recs.size() * sizeof(gevo_variant_record));
        fill_stats(stats, ms, b200::resident_h2d(*b->resident),
                   recs.size() * sizeof(gevo_variant_record), launches);
    });
}

int gevo_batch_make_resident(gevo_batch* b) {
    return guard([&] {
        drop_resident(b);
        b->resident = b200::make_resident(*b->suite->suite, *b->image);
    });
}

int gevo_eval_resident(gevo_batch* b, const gevo_exec_config* cfg, double tolerance,
                       uint32_t flags, gevo_variant_record* out_variants, gevo_eval_stats* stats) {
    return guard([&] {
        if (!b->resident)
            b->resident = b200::make_resident(*b->suite->suite, *b->image);
        b200::EvalOptions opt;
        opt.tolerance = tolerance;
        opt.early_exit = (flags & GEVO_EVAL_EARLY_EXIT) != 0;
        opt.sequential = (flags & GEVO_EVAL_SEQUENTIAL) != 0;
        std::vector<gevo_variant_record> recs;
        float interp = 0.0f;
        int launches = 0;
        const float ms = b200::evaluate_resident(*b->resident, b200::exec_image(exec_from(cfg)), opt,
                                                 &interp, out_variants ? &recs : nullptr, &launches);
        if (out_variants && !recs.empty())
            std::memcpy(out_variants, recs.data(), recs.size() * sizeof(gevo_variant_record));
        fill_stats(stats, ms, 0, out_variants ? recs.size() * sizeof(gevo_variant_record) : 0,
                   launches);
    });
}

int gevo_reason(const gevo_batch* b, int variant, uint32_t code, int32_t aux, double fail_error,
                char** text) {
    return guard([&] {
        if (code == GEVO_FAIL_TOLERANCE)
            *text = dup("error " + std::to_string(fail_error) + " exceeds tolerance");
        else
            *text = dup(b->image->reason(static_cast<size_t>(variant), static_cast<uint8_t>(code), aux));
    });
}

int gevo_rank(const double* cost, const double* error, int32_t n, int device, int32_t* front_out,
              double* crowding_out, int32_t* members_out, int32_t* offsets_out,
              int32_t* n_fronts_out) {
    return guard([&] {
        std::unique_ptr<b200::Device> own;
        b200::Device& dev = device_for(device, own);
        std::vector<FitnessVector> fits(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i)
            fits[static_cast<size_t>(i)] = FitnessVector{cost[i], error[i]};
        const ParetoRank r = b200::rank_on_device(dev, fits, false);
        int32_t pos = 0;
        for (size_t f = 0; f < r.fronts.size(); ++f) {
            if (offsets_out)
                offsets_out[f] = pos;
            for (int m : r.fronts[f]) {
                if (members_out)
                    members_out[pos] = m;
                ++pos;
            }
        }
        if (offsets_out)
            offsets_out[r.fronts.size()] = pos;
        for (int32_t i = 0; i < n; ++i) {
            if (front_out)
                front_out[i] = r.front[static_cast<size_t>(i)];
            if (crowding_out)
                crowding_out[i] = r.crowding[static_cast<size_t>(i)];
        }
        if (n_fronts_out)
            *n_fronts_out = static_cast<int32_t>(r.fronts.size());
    });
}

int gevo_crowding(const double* cost, const double* error, int32_t n, int device,
                  double* crowding_out) {
    return guard([&] {
        std::unique_ptr<b200::Device> own;
        b200::Device& dev = device_for(device, own);
        std::vector<FitnessVector> fits(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i)
            fits[static_cast<size_t>(i)] = FitnessVector{cost[i], error[i]};
        const ParetoRank r = b200::rank_on_device(dev, fits, true);
        for (int32_t i = 0; i < n; ++i)
            crowding_out[i] = r.crowding[static_cast<size_t>(i)];
    });
}

int gevo_nsga_select(const double* cost, const double* error, int32_t n, int device,
                     int32_t keep, int32_t* best_out, uint64_t tournament_seed, int32_t k,
                     int32_t* tournament_out) {
    return guard([&] {
        std::unique_ptr<b200::Device> own;
        b200::Device& dev = device_for(device, own);
        std::vector<FitnessVector> fits(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i)
            fits[static_cast<size_t>(i)] = FitnessVector{cost[i], error[i]};
        ParetoRank r;
        const std::vector<int> best =
            b200::select_on_device(dev, fits, static_cast<size_t>(std::max(keep, 0)), &r);
        if (best_out)
            std::copy(best.begin(), best.end(), best_out);
        if (tournament_out) {
            Rng rng(tournament_seed);
            const std::vector<int> t =
                tournament_select(r, static_cast<size_t>(n), static_cast<size_t>(k), rng);
            std::copy(t.begin(), t.end(), tournament_out);
        }
    });
}

int gevo_debug_cta_clock(uint64_t* out, size_t words, size_t* copied) {
    return guard([&] {
        const size_t n = b200::debug_cta_clock(b200::Device::default_device(), out, words);
        if (copied)
            *copied = n;
    });
}

int gevo_select_best(const double* cost, const double* error, int32_t n, int device, int32_t keep,
                     int32_t* best_out, float* device_ms) {
    return guard([&] {
        if (n < 0 || keep < 0 || keep > n)
            throw std::invalid_argument("gevo_select_best: need 0 <= keep <= n");
        std::unique_ptr<b200::Device> own;
        b200::Device& dev = device_for(device, own);
        std::vector<FitnessVector> fits(static_cast<size_t>(n));
        for (int32_t i = 0; i < n; ++i)
            fits[static_cast<size_t>(i)] = FitnessVector{cost[i], error[i]};
        float ms = 0.0f;
        const std::vector<int> best = b200::select_on_device(dev, fits, static_cast<size_t>(keep), nullptr, &ms);
        if (best_out)
            std::copy(best.begin(), best.end(), best_out);
        if (device_ms)
            *device_ms = ms;
    });
}

int gevo_eval_outputs_json(gevo_batch* b, const gevo_exec_config* cfg, char** outputs_json) {
    return guard([&] {
        b200::EvalOptions opt;
        opt.want_tests = true;
        opt.want_outputs = true;
        const b200::EvalResult r =
            b200::evaluate(*b->suite->suite, *b->image, b200::exec_image(exec_from(cfg)), opt);
        nlohmann::json all = nlohmann::json::array();
        const int T = b->suite->suite->image().n_tests;
        for (size_t v = 0; v < r.variants.size(); ++v) {
            nlohmann::json per = nlohmann::json::array();
            for (int t = 0; t < T; ++t) {
                const size_t gi = v * static_cast<size_t>(T) + static_cast<size_t>(t);
                if (r.tests[gi].status != GEVO_STATUS_COMPLETED) {
                    per.push_back(nullptr);
                    continue;
                }
                per.push_back(buffers_hex(r.outputs[v][static_cast<size_t>(t)]));
            }
            all.push_back(std::move(per));
        }
        *outputs_json = dup(all.dump());
    });
}

int gevo_execute(const char* kernel_ir, const char* test_json, const gevo_exec_config* cfg,
                 char** result_json) {
    return guard([&] {
        const ExecResult r = execute(parse_kernel(kernel_ir), testcase_from_json(test_json),
                                     exec_from(cfg));
        nlohmann::json j;
        j["status"] = r.status == ExecStatus::Completed ? "completed"
                      : r.status == ExecStatus::Trap   ? "trap"
                                                       : "budget";
        j["reason"] = r.trap_reason;
        j["cost"] = r.cost;
        j["outputs"] = buffers_hex(r.outputs);
        *result_json = dup(j.dump());
    });
}

int gevo_evaluate_fitness(const char* kernel_ir, const char* const* tests_json, int n_tests,
                          const gevo_exec_config* cfg, double tolerance, char** outcome_json) {
    return guard([&] {
        std::vector<TestCase> tests;
        for (int i = 0; i < n_tests; ++i)
            tests.push_back(testcase_from_json(tests_json[i]));
        const EvalOutcome o = evaluate_fitness(parse_kernel(kernel_ir), tests, exec_from(cfg), tolerance);
        nlohmann::json j;
        j["accepted"] = o.accepted;
        j["failing_test"] = o.failing_test;
        j["reason"] = o.reason;
        j["cost"] = hex_double(o.fitness.cost);
        j["error"] = hex_double(o.fitness.error);
        *outcome_json = dup(j.dump());
    });
}

int gevo_kernel_canonical(const char* kernel_ir, char** printed) {
    return guard([&] { *printed = dup(print_kernel(parse_kernel(kernel_ir))); });
}

int gevo_kernel_validate(const char* kernel_ir, char** rules_json) {
    return guard([&] {
        nlohmann::json a = nlohmann::json::array();
        for (const auto& e : validate(parse_kernel(kernel_ir)))
            a.push_back(e.rule + "@" + std::to_string(e.uid));
        *rules_json = dup(a.dump());
    });
}

int gevo_kernel_is_valid(const char* kernel_ir, int32_t* valid) {
    return guard([&] { *valid = is_valid(parse_kernel(kernel_ir)) ? 1 : 0; });
}

int gevo_apply_patch(const char* kernel_ir, const char* patch_json, char** printed,
                     int32_t* n_applied) {
    return guard([&] {
        const PatchResult r = apply_patch(parse_kernel(kernel_ir), patch_from_json(patch_json));
        *printed = dup(print_kernel(r.kernel));
        if (n_applied)
            *n_applied = static_cast<int32_t>(r.applied.size());
    });
}

int gevo_random_mutation(const char* kernel_ir, uint64_t master, uint64_t a, uint64_t b,
                         uint64_t c, char** edit_json, uint64_t* probe) {
    return guard([&] {
        const Kernel k = parse_kernel(kernel_ir);
        Rng rng = Rng::stream(master, a, b, c);
        const DomTree dom = DomTree::build(k);
        MutationContext ctx(k, dom, rng);
        const MutationResult m = random_mutation(ctx);
        *edit_json = dup(m ? edit_key(*m) : std::string("null"));
        if (probe)
            *probe = rng.next_u64();
    });
}

int gevo_benchmark_inputs(const char* bench, int count, uint64_t seed, char** tests_json) {
    return guard([&] {
        const Benchmark b = load_benchmark(bench);
        nlohmann::json a = nlohmann::json::array();
        for (const TestCase& t : generate_inputs_for(b.gen, count, seed))
            a.push_back(nlohmann::json::parse(testcase_to_json(t)));
        *tests_json = dup(a.dump());
    });
}

int gevo_benchmark_names(char** names_json) {
    return guard([&] { *names_json = dup(nlohmann::json(benchmark_names()).dump()); });
}

int gevo_benchmark_ir(const char* bench, char** ir) {
    return guard([&] { *ir = dup(print_kernel(load_benchmark(bench).kernel)); });
}

namespace {
std::string sample_candidates_of(const Kernel& kernel, int n, uint64_t seed, int max_depth) {
    if (n < 0 || max_depth < 1)
        throw std::invalid_argument("gevo_sample_candidates: n >= 0 and max_depth >= 1");
    struct Parent {
        Kernel k;
        Patch p;
    };
    std::vector<Parent> parents{{kernel, {}}};
    Rng pick(seed ^ 0xCA7D1DA7E5ULL);
    std::string out;
    int made = 0;
    for (uint64_t i = 0; made < n; ++i) {
        if (i > static_cast<uint64_t>(n) * 200 + 1000)
            throw std::invalid_argument("gevo_sample_candidates: kernel yields no valid mutants");
        const Parent& par = parents[pick.index(parents.size())];
        Rng rng = Rng::stream(seed, 0xC4, i, 1);
        const DomTree dom = DomTree::build(par.k);
        MutationContext ctx(par.k, dom, rng);
        const MutationResult m = random_mutation(ctx);
        if (!m)
            continue;
        ApplyResult ar = apply_edit(par.k, *m);
        if (!ar.applied || !is_valid(ar.kernel))
            continue;
        Patch p = par.p;
        p.push_back(*m);
        out += nlohmann::json::parse(patch_to_json(p)).dump();
        out += '\n';
        ++made;
        if (static_cast<int>(p.size()) < max_depth)
            parents.push_back({std::move(ar.kernel), std::move(p)});
    }
    return out;
}
} // namespace

int gevo_sample_candidates(const char* bench, int n, uint64_t seed, int max_depth,
                           char** patches) {
    return guard([&] {
        *patches = dup(sample_candidates_of(load_benchmark(bench).kernel, n, seed, max_depth));
    });
}

int gevo_sample_candidates_ir(const char* kernel_ir, int n, uint64_t seed, int max_depth,
                              char** patches) {
    return guard([&] {
        *patches = dup(sample_candidates_of(parse_kernel(kernel_ir), n, seed, max_depth));
    });
}

int gevo_suite_from_spec(const char* kernel_ir, const char* gen_json, int n_tests, uint64_t seed,
                         int device, gevo_suite** out) {
    return guard([&] {
        auto s = std::make_unique<gevo_suite>();
        b200::Device& dev = device_for(device, s->own_device);
        s->kernel = parse_kernel(kernel_ir);
        const std::vector<TestCase> tests =
            generate_tests_for(s->kernel, generator_spec_from_json(gen_json), n_tests, seed);
        s->suite = std::make_unique<b200::DeviceSuite>(dev, b200::build_suite(s->kernel.params, tests));
        *out = s.release();
    });
}

int gevo_spec_inputs(const char* gen_json, int count, uint64_t seed, char** tests_json) {
    return guard([&] {
        nlohmann::json a = nlohmann::json::array();
        for (const TestCase& t : generate_inputs_for(generator_spec_from_json(gen_json), count, seed))
            a.push_back(nlohmann::json::parse(testcase_to_json(t)));
        *tests_json = dup(a.dump());
    });
}

uint64_t gevo_train_seed(uint64_t master) { return cli::train_seed(master); }
uint64_t gevo_heldout_seed(uint64_t master) { return cli::heldout_seed(master); }

int gevo_run_search(const char* bench, uint64_t seed, int pop, int generations, const char* mode,
                    double tolerance, int train_tests, int heldout_tests, int jobs, char** log_csv,
                    char** report_json, gevo_run_stats* stats) {
    return guard([&] {
        cli::RunOptions o;
        o.bench = bench;
        o.seed = seed;
        o.pop = pop;
        o.generations = generations;
        o.mode = mode ? mode : "default";
        if (tolerance >= 0.0)
            o.tolerance = tolerance;
        o.train_tests = train_tests;
        o.heldout_tests = heldout_tests;
        o.jobs = jobs;
        const cli::RunArtifacts a = cli::run_benchmark(o);
        if (log_csv)
            *log_csv = dup(a.log_csv);
        if (report_json)
            *report_json = dup(a.report_json);
        if (stats) {
            stats->candidates = a.counters.candidates;
            stats->executions = a.counters.executions;
            stats->dynamic_ir = a.counters.dynamic_ir;
            stats->launches = a.counters.launches;
            stats->batches = a.counters.batches;
            stats->device_ms = a.counters.device_ms;
            stats->host_gen_ms = a.counters.host_gen_ms;
            stats->seconds = a.seconds;
        }
    });
}

} // extern "C"
