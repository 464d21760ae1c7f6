// Speculative, batched GEVO search engine.
//
// Observable behaviour (population, archive, log rows, operator statistics,
// RNG stream usage) is that of src/engine.cpp of arxiv/paper_2004_08140:
// stream purposes (19-26), baseline (66-89), sanity_check (91-95), retry loops
// (97-151), initialisation (153-193), generation step (195-273), archive
// (275-292), logging (306-332), run + held-out pass + best pick (334-389).
//
// What changes is the schedule. A retry loop's k-th attempt draws from the
// stream left by attempt k-1 and from the (fixed) parent only, so the host
// draws a wave of attempts per slot ahead of time, recording the stream state
// after each; all candidates of all slots go to the device as one batch; the
// first accepted attempt wins and the slot's stream is rewound to the state
// recorded after it. Statistics count only the attempts the sequential loop
// would have made.
#include "evoir/engine.hpp"

#include "runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <exception>
#include <functional>
#include <limits>
#include <mutex>
#include <thread>

#include <unistd.h>

namespace evoir {

namespace {

enum StreamPurpose : uint64_t {
    kStreamInit = 1,
    kStreamTournament = 2,
    kStreamGateCross = 3,
    kStreamGateMutate = 4,
    kStreamCross = 5,
    kStreamMutate = 6,
};

// Persistent host worker pool. A search issues a few hundred parallel
// sections (draw/apply/validate waves, encoding) about a millisecond apart;
// spawning threads for each would cost ~10^4 thread creations per run, and a
// condition-variable wake per section costs tens of microseconds. Workers
// spin on a section word for a while before they sleep, and claim seats in
// it with one CAS: [epoch:32][pending:16][seats:16] -- seats still open in
// this section, helpers inside it. The caller revokes unclaimed seats once
// every index is taken and waits only for helpers already inside.
class HostPool {
public:
    static HostPool& get() {
        static HostPool p;
        return p;
    }
    // fn(i) for i in [0, n) on the caller plus up to jobs - 1 workers; the
    // first exception is rethrown after every participant stopped.
    void run(size_t n, int jobs, const std::function<void(size_t)>& fn) {
        std::unique_lock<std::mutex> section(section_mu_); // one section at a time
        const uint64_t helpers = std::min<size_t>(
            {static_cast<size_t>(std::max(jobs - 1, 0)), workers_.size(), n - 1, 0xFFFF});
        fn_ = &fn;
        n_ = n;
        next_.store(0);
        stop_.store(false);
        err_ = nullptr;
        const uint64_t e = ++epoch_ & 0xFFFFFFFFu;
        word_.store((e << 32) | helpers); // publish the section
        if (sleepers_.load() > 0) {
            std::lock_guard<std::mutex> g(mu_);
            cv_.notify_all();
        }
        work();
        // revoke the seats nobody took, then wait for the helpers inside
        uint64_t w = word_.load();
        while ((w & 0xFFFF) && !word_.compare_exchange_weak(w, w & ~uint64_t(0xFFFF))) {
        }
        for (int spin = 0; ((word_.load() >> 16) & 0xFFFF) != 0; ++spin)
            if (spin > 1000)
                std::this_thread::yield();
        if (err_)
            std::rethrow_exception(err_);
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            quit_.store(true);
        }
        cv_.notify_all();
        for (auto& t : workers_)
            t.join();
    }
    static bool on_worker() { return worker_flag(); }
    // a forked child inherits the pool object but not its threads
    bool usable() const { return ::getpid() == pid_; }

private:
    static constexpr int kSpin = 1 << 16; // ~1 ms of pause loops before sleeping
    static bool& worker_flag() {
        static thread_local bool f = false;
        return f;
    }
    HostPool() : pid_(::getpid()) {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        for (unsigned w = 0; w + 1 < hw; ++w)
            workers_.emplace_back([this] { loop(); });
    }
    void work() {
        for (;;) {
            const size_t i = next_.fetch_add(1);
            if (i >= n_ || stop_.load())
                return;
            try {
                (*fn_)(i);
            } catch (...) {
                std::lock_guard<std::mutex> g(err_mu_);
                if (!err_)
                    err_ = std::current_exception();
                stop_.store(true);
                return;
            }
        }
    }
    static bool open(uint64_t w, uint64_t seen) { return (w >> 32) != seen && (w & 0xFFFF) != 0; }
    static void relax() {
#if defined(__x86_64__)
        __builtin_ia32_pause();
#endif
    }
    void loop() {
        worker_flag() = true;
        uint64_t seen = 0;
        for (;;) {
            uint64_t w = word_.load();
            for (int spin = 0; !open(w, seen); w = word_.load()) {
                if (quit_.load())
                    return;
                if (++spin < kSpin) {
                    relax();
                    continue;
                }
                std::unique_lock<std::mutex> g(mu_);
                sleepers_.fetch_add(1);
                cv_.wait(g, [&] { return quit_.load() || open(word_.load(), seen); });
                sleepers_.fetch_sub(1);
                spin = 0;
            }
            // claim a seat: seats - 1, pending + 1 (fails if the section moved on)
            if (!word_.compare_exchange_weak(w, w - 1 + (uint64_t(1) << 16)))
                continue;
            seen = w >> 32;
            work();
            word_.fetch_sub(uint64_t(1) << 16);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex section_mu_, mu_, err_mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> word_{0};
    std::atomic<int> sleepers_{0};
    std::atomic<bool> quit_{false};
    uint64_t epoch_ = 0;
    const std::function<void(size_t)>* fn_ = nullptr;
    size_t n_ = 0;
    std::atomic<size_t> next_{0};
    std::atomic<bool> stop_{false};
    std::exception_ptr err_;
    pid_t pid_;
};

// Work-sharing loop over [0, n) on up to `jobs` host threads; the first
// exception is rethrown after all workers stop.
void host_parallel(size_t n, int jobs, const std::function<void(size_t)>& fn) {
    if (jobs <= 1 || n <= 1 || HostPool::on_worker() || !HostPool::get().usable()) {
        for (size_t i = 0; i < n; ++i)
            fn(i);
        return;
    }
    HostPool::get().run(n, jobs, fn);
}

b200::Collective& collective_slot() {
    static b200::Collective c;
    return c;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// GEVO_TRACE=1: wall-time split of a search on stderr (diagnostic)
struct Trace {
    double verdicts_ms = 0, eval_ms = 0;
    double select_ms = 0, cx_ms = 0, mut_ms = 0, rank_ms = 0, archive_ms = 0;
    double cx_gen_ms = 0, cx_resolve_ms = 0, mut_gen_ms = 0, mut_resolve_ms = 0;
    static Trace& get() {
        static Trace t;
        return t;
    }
    static bool on() {
        static const bool v = std::getenv("GEVO_TRACE") != nullptr;
        return v;
    }
};

// Wave schedule: attempts drawn per slot per round before the next device batch.
int wave_size(int used, int retries) {
    const int want = used == 0 ? 6 : (used < 16 ? 12 : 24);
    return std::max(0, std::min(want, retries - used));
}

// Device verdicts for a list of kernels (no validation; evaluate_fitness).
// With a multi-rank collective, rank r evaluates the contiguous shard
// [begin_r, end_r) of the batch and the records are all-gathered.
std::vector<EvalOutcome> device_verdicts(b200::DeviceSuite& suite, const b200::ExecImage& ex,
                                         const std::vector<const Kernel*>& ks, double tol,
                                         bool with_reasons, EngineCounters& ctr, int jobs = 1,
                                         const std::vector<double>* weight = nullptr) {
    std::vector<EvalOutcome> out(ks.size());
    if (ks.empty())
        return out;
    struct Timer {
        std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
        ~Timer() { Trace::get().verdicts_ms += ms_since(t0); }
    } timer;
    if (suite.image().n_tests == 0) {
        for (auto& o : out)
            o = EvalOutcome::rejected(-1, "no test cases");
        return out;
    }
    // Sharding: with an NCCL communicator in the library (one process per
    // GPU) the records are all-gathered on the device inside the evaluation;
    // otherwise through the caller's collective callback (host buffers).
    const b200::Collective& col = b200::collective();
    const int nw = b200::nccl_world();
    const bool via_nccl = nw >= 1 && !with_reasons;
    const bool shard = via_nccl || (col.world > 1 && col.allgather && !with_reasons);
    const size_t n = ks.size();
    const size_t W = !shard ? 1 : via_nccl ? static_cast<size_t>(nw) : static_cast<size_t>(col.world);
    const size_t R = !shard ? 0 : via_nccl ? static_cast<size_t>(b200::nccl_rank()) : static_cast<size_t>(col.rank);
    // contiguous shards (gathered records concatenate back into batch order),
    // cut at equal shares of the predicted cost when weights are given -- a
    // budget spinner costs ~10^3 ordinary variants -- else at
    // equal counts; every rank computes the same cuts
    std::vector<size_t> cut(W + 1, n);
    cut[0] = 0;
    if (weight && weight->size() == n && W > 1) {
        double total = 0;
        for (double w : *weight)
            total += std::max(w, 1.0);
        double acc = 0;
        size_t r = 1;
        for (size_t v = 0; v < n && r < W; ++v) {
            acc += std::max((*weight)[v], 1.0);
            while (r < W && acc >= total * static_cast<double>(r) / static_cast<double>(W))
                cut[r++] = v + 1;
        }
    } else {
        for (size_t r = 1; r < W; ++r) {
            const size_t q = n / W, m = n % W;
            cut[r] = r * q + std::min(r, m);
        }
    }
    auto span = [&](size_t r) { return std::make_pair(cut[r], cut[r + 1]); };
    const auto [lo, hi] = span(R);
    // encode in parallel parts (the device bytecode of ~10^5 candidates per
    // search is otherwise a serial host term), joined in candidate order
    const auto t_enc = std::chrono::steady_clock::now();
    b200::BatchImage batch(suite.image());
    constexpr size_t kPart = 16; // (a wave holds a few hundred candidates: enough parts for every worker)
    const size_t parts = (hi - lo + kPart - 1) / kPart;
    if (jobs > 1 && parts > 1) {
        std::vector<std::unique_ptr<b200::BatchImage>> part(parts);
        const size_t rec_hint = (ks[lo]->instruction_count() + ks[lo]->blocks.size()) * kPart * 5 / 4;
        host_parallel(parts, jobs, [&](size_t p) {
            part[p] = std::make_unique<b200::BatchImage>(suite.image());
            part[p]->reserve(kPart, rec_hint);
            for (size_t v = lo + p * kPart; v < std::min(hi, lo + (p + 1) * kPart); ++v)
                part[p]->add(*ks[v]);
        });
        batch.reserve(hi - lo, rec_hint * parts);
        for (auto& p : part)
            batch.append(std::move(*p));
    } else {
        for (size_t v = lo; v < hi; ++v)
            batch.add(*ks[v]);
    }
    batch.header(); // lay out here, so the encode time below covers it
    ctr.host_gen_ms += ms_since(t_enc);
    b200::EvalOptions opt;
    opt.tolerance = tol;
    opt.early_exit = true;
    size_t m = 0; // largest shard: the exchange pads every shard to it
    for (size_t q = 0; q < W; ++q)
        m = std::max(m, cut[q + 1] - cut[q]);
    b200::EvalResult r;
    const auto t_ev = std::chrono::steady_clock::now();
    if (via_nccl) {
        opt.gather_count = std::max<size_t>(m, 1);
        r = b200::evaluate(suite, batch, ex, opt); // (an empty shard still joins the all-gather)
    } else if (hi > lo) {
        r = b200::evaluate(suite, batch, ex, opt);
    }
    Trace::get().eval_ms += ms_since(t_ev);
    std::vector<gevo_variant_record> recs;
    if (via_nccl) {
        const size_t mm = std::max<size_t>(m, 1);
        recs.reserve(n);
        for (size_t q = 0; q < W; ++q) {
            const auto [b, e] = span(q);
            recs.insert(recs.end(), r.variants.begin() + q * mm, r.variants.begin() + q * mm + (e - b));
        }
    } else if (shard) {
        std::vector<gevo_variant_record> send(m), recv(m * W);
        std::copy(r.variants.begin(), r.variants.end(), send.begin());
        col.allgather(col.ctx, send.data(), m * sizeof(gevo_variant_record), recv.data());
        recs.reserve(n);
        for (size_t q = 0; q < W; ++q) {
            const auto [b, e] = span(q);
            recs.insert(recs.end(), recv.begin() + q * m, recv.begin() + q * m + (e - b));
        }
    } else {
        recs = std::move(r.variants);
    }
    ctr.candidates += static_cast<int64_t>(ks.size());
    ctr.launches += r.launches;
    ctr.batches += 1;
    ctr.device_ms += r.kernel_ms;
    for (size_t v = 0; v < ks.size(); ++v) {
        const gevo_variant_record& x = recs[v];
        ctr.executions += x.execs_ref;
        ctr.dynamic_ir += x.ir_ref;
        if (x.accepted) {
            out[v] = EvalOutcome::ok(FitnessVector{x.cost_mean, x.error_max});
        } else if (!with_reasons) {
            out[v] = EvalOutcome::rejected(x.failing_test, std::string());
        } else if (x.code == GEVO_FAIL_TOLERANCE) {
            out[v] = EvalOutcome::rejected(x.failing_test, "error " + std::to_string(x.fail_error) +
                                                               " exceeds tolerance");
        } else {
            out[v] = EvalOutcome::rejected(x.failing_test, batch.reason(v, x.code, x.aux));
        }
    }
    return out;
}

} // namespace

namespace b200 {
void set_collective(const Collective& c) { collective_slot() = c; }
const Collective& collective() { return collective_slot(); }
} // namespace b200

// ---------------------------------------------------------------------------
// Speculation state
// ---------------------------------------------------------------------------

struct Engine::MutJob {
    const Individual* parent = nullptr;
    Rng* rng = nullptr;
    OperatorStats* stats = nullptr;
    Individual result;
    bool done = false;
    int used = 0;
    std::unique_ptr<DomTree> dom;
    std::unique_ptr<MutationContext> ctx;
    struct Attempt {
        uint64_t rng_after[4];
        int kind = -1; // -1: NoCandidate
        Edit edit;
        Kernel kernel;
        bool candidate = false; // applied and valid: goes to the device
        int verdict = -1;       // index into the wave's verdicts
    };
    std::vector<Attempt> wave;
};

struct Engine::CxJob {
    const Individual* a = nullptr;
    const Individual* b = nullptr;
    Rng* rng = nullptr;
    OperatorStats* stats = nullptr;
    Individual ra, rb;
    bool done = false;
    int used = 0;
    struct Attempt {
        uint64_t rng_after[4];
        PatchResult pa, pb;
        int va = -1, vb = -1; // verdict indices, -1: failed validation
    };
    std::vector<Attempt> wave;
};

Engine::Engine(Kernel original, SearchConfig cfg, std::vector<TestCase> tests)
    : original_(std::move(original)), cfg_(std::move(cfg)), tests_(std::move(tests)) {
    cfg_.check();
    if (tests_.empty())
        throw InitFailure("no test cases");
    if (!is_valid(original_))
        throw InitFailure("original kernel fails validation");
    exec_ = ExecConfig::for_kernel(original_);
    exec_.instruction_budget = cfg_.instruction_budget;
    exec_.cost_table = cfg_.cost_table;
    suite_ = std::make_shared<b200::DeviceSuite>(b200::Device::default_device(),
                                                 b200::build_suite(original_.params, tests_));
    exec_img_ = std::make_unique<b200::ExecImage>(b200::exec_image(exec_));

    const EvalOutcome base =
        device_verdicts(*suite_, *exec_img_, {&original_}, 0.0, true, counters_).at(0);
    if (!base.accepted)
        throw InitFailure("original kernel fails its own oracle: " + base.reason);
    baseline_ = base.fitness;
    Individual origin;
    origin.kernel = original_;
    origin.fitness = baseline_;
    archive_add(origin);
}

Engine::~Engine() = default;

EvalOutcome Engine::sanity_check(const Kernel& k) const {
    return sanity_check_batch({&k}, true).at(0);
}

std::vector<EvalOutcome> Engine::sanity_check_batch(const std::vector<const Kernel*>& ks,
                                                    bool with_reasons) const {
    std::vector<EvalOutcome> out(ks.size());
    std::vector<char> ok(ks.size(), 0);
    host_parallel(ks.size(), cfg_.jobs, [&](size_t i) { ok[i] = is_valid(*ks[i]) ? 1 : 0; });
    std::vector<const Kernel*> dev;
    std::vector<size_t> where;
    for (size_t i = 0; i < ks.size(); ++i) {
        if (!ok[i]) {
            out[i] = EvalOutcome::rejected(-1, "validation failed");
            continue;
        }
        dev.push_back(ks[i]);
        where.push_back(i);
    }
    const auto v = device_verdicts(*suite_, *exec_img_, dev, cfg_.tolerance, with_reasons, counters_, cfg_.jobs);
    for (size_t j = 0; j < where.size(); ++j)
        out[where[j]] = v[j];
    return out;
}

void Engine::run_mutations(std::vector<MutJob>& jobs) const {
    const int retries = cfg_.mutation_retries;
    for (MutJob& j : jobs) {
        if (retries <= 0) {
            ++j.stats->mut_exhausted;
            j.result = *j.parent;
            j.done = true;
        }
    }
    for (;;) {
        std::vector<MutJob*> active;
        for (MutJob& j : jobs)
            if (!j.done)
                active.push_back(&j);
        if (active.empty())
            return;
        const auto t0 = std::chrono::steady_clock::now();
        // 1. draw, apply and validate a wave of attempts per active slot
        host_parallel(active.size(), cfg_.jobs, [&](size_t i) {
            MutJob& j = *active[i];
            if (!j.ctx) {
                j.dom = std::make_unique<DomTree>(DomTree::build(j.parent->kernel));
                j.ctx = std::make_unique<MutationContext>(j.parent->kernel, *j.dom, *j.rng);
            }
            j.wave.clear();
            const int k = wave_size(j.used, retries);
            j.wave.resize(static_cast<size_t>(k));
            for (int a = 0; a < k; ++a) {
                MutJob::Attempt& at = j.wave[static_cast<size_t>(a)];
                MutationResult m = random_mutation(*j.ctx);
                j.rng->get_state(at.rng_after);
                if (!m)
                    continue;
                at.kind = static_cast<int>(operator_kind(*m));
                at.edit = std::move(*m);
                ApplyResult ap = apply_edit(j.parent->kernel, at.edit);
                if (!ap.applied)
                    continue;
                at.kernel = std::move(ap.kernel);
                at.candidate = is_valid(at.kernel);
            }
        });
        // 2. one device batch for every candidate of every slot
        std::vector<const Kernel*> ks;
        std::vector<double> weight; // predicted cost: the parent's mean cost
        for (MutJob* j : active)
            for (auto& at : j->wave)
                if (at.candidate) {
                    at.verdict = static_cast<int>(ks.size());
                    ks.push_back(&at.kernel);
                    weight.push_back(j->parent->fitness ? j->parent->fitness->cost : 1.0);
                }
        counters_.host_gen_ms += ms_since(t0);
        Trace::get().mut_gen_ms += ms_since(t0);
        const auto verdicts = device_verdicts(*suite_, *exec_img_, ks, cfg_.tolerance, false, counters_,
                                              cfg_.jobs, &weight);
        const auto t_res = std::chrono::steady_clock::now();
        // 3. resolve each slot in attempt order
        for (MutJob* j : active) {
            for (auto& at : j->wave) {
                ++j->used;
                if (at.kind < 0)
                    continue;
                ++j->stats->attempts[at.kind];
                if (!at.candidate || !verdicts[static_cast<size_t>(at.verdict)].accepted)
                    continue;
                ++j->stats->accepts[at.kind];
                Individual next;
                next.kernel = std::move(at.kernel);
                next.patch = j->parent->patch;
                next.patch.push_back(at.edit);
                next.fitness = verdicts[static_cast<size_t>(at.verdict)].fitness;
                j->result = std::move(next);
                j->rng->set_state(at.rng_after);
                j->done = true;
                break;
            }
            if (!j->done && j->used >= retries) {
                ++j->stats->mut_exhausted;
                j->result = *j->parent;
                j->done = true;
            }
        }
        host_parallel(active.size(), cfg_.jobs, [&](size_t i) { active[i]->wave.clear(); });
        Trace::get().mut_resolve_ms += ms_since(t_res);
    }
}

void Engine::run_crossovers(std::vector<CxJob>& jobs) const {
    const int retries = cfg_.crossover_retries;
    for (CxJob& j : jobs) {
        if (retries <= 0) {
            ++j.stats->cx_exhausted;
            j.ra = *j.a;
            j.rb = *j.b;
            j.done = true;
        }
    }
    for (;;) {
        std::vector<CxJob*> active;
        for (CxJob& j : jobs)
            if (!j.done)
                active.push_back(&j);
        if (active.empty())
            return;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::vector<char>> valid(active.size());
        host_parallel(active.size(), cfg_.jobs, [&](size_t i) {
            CxJob& j = *active[i];
            j.wave.clear();
            const int k = std::min(j.used == 0 ? 4 : 8, retries - j.used);
            j.wave.resize(static_cast<size_t>(k));
            valid[i].assign(2 * static_cast<size_t>(k), 0);
            for (int a = 0; a < k; ++a) {
                CxJob::Attempt& at = j.wave[static_cast<size_t>(a)];
                auto [pa, pb] = crossover_messy(j.a->patch, j.b->patch, *j.rng);
                j.rng->get_state(at.rng_after);
                at.pa = apply_patch(original_, pa);
                at.pb = apply_patch(original_, pb);
                valid[i][2 * a] = is_valid(at.pa.kernel) ? 1 : 0;
                valid[i][2 * a + 1] = is_valid(at.pb.kernel) ? 1 : 0;
            }
        });
        std::vector<const Kernel*> ks;
        std::vector<double> weight; // predicted cost: the parents' mean cost
        for (size_t i = 0; i < active.size(); ++i) {
            const CxJob& j = *active[i];
            const double w = (j.a->fitness ? j.a->fitness->cost : 1.0) / 2 +
                             (j.b->fitness ? j.b->fitness->cost : 1.0) / 2;
            for (size_t a = 0; a < active[i]->wave.size(); ++a) {
                auto& at = active[i]->wave[a];
                if (valid[i][2 * a]) {
                    at.va = static_cast<int>(ks.size());
                    ks.push_back(&at.pa.kernel);
                    weight.push_back(w);
                }
                if (valid[i][2 * a + 1]) {
                    at.vb = static_cast<int>(ks.size());
                    ks.push_back(&at.pb.kernel);
                    weight.push_back(w);
                }
            }
        }
        counters_.host_gen_ms += ms_since(t0);
        Trace::get().cx_gen_ms += ms_since(t0);
        const auto verdicts = device_verdicts(*suite_, *exec_img_, ks, cfg_.tolerance, false, counters_,
                                              cfg_.jobs, &weight);
        const auto t_res = std::chrono::steady_clock::now();
        for (CxJob* j : active) {
            for (auto& at : j->wave) {
                ++j->used;
                ++j->stats->cx_attempts;
                if (at.va < 0 || !verdicts[static_cast<size_t>(at.va)].accepted)
                    continue;
                if (at.vb < 0 || !verdicts[static_cast<size_t>(at.vb)].accepted)
                    continue;
                ++j->stats->cx_accepts;
                j->ra.kernel = std::move(at.pa.kernel);
                j->ra.patch = std::move(at.pa.applied);
                j->ra.fitness = verdicts[static_cast<size_t>(at.va)].fitness;
                j->rb.kernel = std::move(at.pb.kernel);
                j->rb.patch = std::move(at.pb.applied);
                j->rb.fitness = verdicts[static_cast<size_t>(at.vb)].fitness;
                j->rng->set_state(at.rng_after);
                j->done = true;
                break;
            }
            if (!j->done && j->used >= retries) {
                ++j->stats->cx_exhausted;
                j->ra = *j->a;
                j->rb = *j->b;
                j->done = true;
            }
        }
        // the losing attempts' kernels are freed on the worker threads
        host_parallel(active.size(), cfg_.jobs, [&](size_t i) { active[i]->wave.clear(); });
        Trace::get().cx_resolve_ms += ms_since(t_res);
    }
}

Individual Engine::mutate_until_valid(const Individual& ind, Rng& rng, OperatorStats& stats) const {
    std::vector<MutJob> jobs(1);
    jobs[0].parent = &ind;
    jobs[0].rng = &rng;
    jobs[0].stats = &stats;
    run_mutations(jobs);
    return std::move(jobs[0].result);
}

std::pair<Individual, Individual> Engine::crossover_until_valid(const Individual& a,
                                                                const Individual& b, Rng& rng,
                                                                OperatorStats& stats) const {
    std::vector<CxJob> jobs(1);
    jobs[0].a = &a;
    jobs[0].b = &b;
    jobs[0].rng = &rng;
    jobs[0].stats = &stats;
    run_crossovers(jobs);
    return {std::move(jobs[0].ra), std::move(jobs[0].rb)};
}

void Engine::initialize_population() {
    const size_t pop = static_cast<size_t>(cfg_.pop_size);
    std::vector<Individual> cur(pop);
    std::vector<Rng> rngs;
    rngs.reserve(pop);
    for (size_t s = 0; s < pop; ++s) {
        cur[s].kernel = original_;
        cur[s].fitness = baseline_;
        rngs.push_back(Rng::stream(cfg_.master_seed, 0, s, kStreamInit));
    }
    std::vector<OperatorStats> slot_stats(pop);
    std::vector<std::string> failures(pop);
    std::vector<char> alive(pop, 1);
    for (int m = 0; m < cfg_.init_dist; ++m) {
        std::vector<MutJob> jobs;
        std::vector<size_t> slots;
        for (size_t s = 0; s < pop; ++s)
            if (alive[s]) {
                jobs.emplace_back();
                jobs.back().parent = &cur[s];
                jobs.back().rng = &rngs[s];
                jobs.back().stats = &slot_stats[s];
                slots.push_back(s);
            }
        if (jobs.empty())
            break;
        run_mutations(jobs);
        for (size_t i = 0; i < jobs.size(); ++i) {
            const size_t s = slots[i];
            if (jobs[i].result.patch.size() == cur[s].patch.size()) {
                failures[s] = "initialization slot " + std::to_string(s) +
                              " exhausted mutation retries at distance " + std::to_string(m);
                alive[s] = 0;
                continue;
            }
            cur[s] = std::move(jobs[i].result);
        }
    }
    population_.assign(pop, Individual{});
    for (size_t s = 0; s < pop; ++s)
        if (alive[s])
            population_[s] = std::move(cur[s]);

    OperatorStats init_stats;
    for (const auto& st : slot_stats)
        init_stats.merge(st);
    stats_.merge(init_stats);
    for (const auto& f : failures)
        if (!f.empty()) {
            std::string detail = f + " (attempts:";
            for (int i = 0; i < kOperatorCount; ++i)
                detail += " " + std::string(operator_kind_name(static_cast<OperatorKind>(i))) + "=" +
                          std::to_string(init_stats.attempts[i]);
            throw InitFailure(detail + ")");
        }
    for (const auto& ind : population_)
        archive_add(ind);
    rank_current();
    generation_ = 0;
    log_generation(init_stats);
}

void Engine::step_generation() {
    const size_t pop = static_cast<size_t>(cfg_.pop_size);
    const uint64_t gen = static_cast<uint64_t>(generation_) + 1;

    auto tp = std::chrono::steady_clock::now();
    auto lap = [&](double& acc) {
        acc += ms_since(tp);
        tp = std::chrono::steady_clock::now();
    };
    Trace& tr = Trace::get();
    Rng trng = Rng::stream(cfg_.master_seed, gen, 0, kStreamTournament);
    const std::vector<int> off_idx = tournament_select(rank_, population_.size(), pop, trng);
    const std::vector<int> elite_idx = select_best(rank_, pop / 4);
    // (copies of selected individuals: one kernel copy each, on the pool)
    std::vector<Individual> offspring(off_idx.size()), elites(elite_idx.size());
    host_parallel(off_idx.size() + elite_idx.size(), cfg_.jobs, [&](size_t i) {
        if (i < off_idx.size())
            offspring[i] = population_[static_cast<size_t>(off_idx[i])];
        else
            elites[i - off_idx.size()] = population_[static_cast<size_t>(elite_idx[i - off_idx.size()])];
    });

    Rng gx = Rng::stream(cfg_.master_seed, gen, 0, kStreamGateCross);
    Rng gm = Rng::stream(cfg_.master_seed, gen, 0, kStreamGateMutate);
    std::vector<char> cx_fire(pop / 2), mut_fire(pop);
    for (auto& f : cx_fire)
        f = gx.chance(cfg_.cross_rate) ? 1 : 0;
    for (auto& f : mut_fire)
        f = gm.chance(cfg_.mutate_rate) ? 1 : 0;

    lap(tr.select_ms);
    // Crossover: every firing pair is one speculative job.
    std::vector<OperatorStats> pair_stats(pop / 2);
    {
        std::vector<Rng> rngs;
        std::vector<CxJob> jobs;
        std::vector<size_t> pairs;
        for (size_t p = 0; p < pop / 2; ++p)
            if (cx_fire[p]) {
                pairs.push_back(p);
                rngs.push_back(Rng::stream(cfg_.master_seed, gen, p, kStreamCross));
            }
        jobs.resize(pairs.size());
        for (size_t i = 0; i < pairs.size(); ++i) {
            jobs[i].a = &offspring[2 * pairs[i]];
            jobs[i].b = &offspring[2 * pairs[i] + 1];
            jobs[i].rng = &rngs[i];
            jobs[i].stats = &pair_stats[pairs[i]];
        }
        run_crossovers(jobs);
        for (size_t i = 0; i < pairs.size(); ++i) {
            offspring[2 * pairs[i]] = std::move(jobs[i].ra);
            offspring[2 * pairs[i] + 1] = std::move(jobs[i].rb);
        }
    }
    lap(tr.cx_ms);
    // Mutation: every firing slot is one speculative job.
    std::vector<OperatorStats> mut_stats(pop);
    {
        std::vector<Rng> rngs;
        std::vector<MutJob> jobs;
        std::vector<size_t> slots;
        for (size_t i = 0; i < pop; ++i)
            if (mut_fire[i]) {
                slots.push_back(i);
                rngs.push_back(Rng::stream(cfg_.master_seed, gen, i, kStreamMutate));
            }
        jobs.resize(slots.size());
        std::vector<Individual> parents(slots.size());
        for (size_t i = 0; i < slots.size(); ++i)
            parents[i] = std::move(offspring[slots[i]]); // refilled from the job below
        for (size_t i = 0; i < slots.size(); ++i) {
            jobs[i].parent = &parents[i];
            jobs[i].rng = &rngs[i];
            jobs[i].stats = &mut_stats[slots[i]];
        }
        run_mutations(jobs);
        for (size_t i = 0; i < slots.size(); ++i)
            offspring[slots[i]] = std::move(jobs[i].result);
    }

    lap(tr.mut_ms);
    OperatorStats gen_stats;
    for (const auto& s : pair_stats)
        gen_stats.merge(s);
    for (const auto& s : mut_stats)
        gen_stats.merge(s);
    stats_.merge(gen_stats);

    std::vector<Individual> pool = std::move(elites);
    for (auto& ind : offspring)
        pool.push_back(std::move(ind));
    std::vector<FitnessVector> fits;
    fits.reserve(pool.size());
    for (const auto& ind : pool)
        fits.push_back(*ind.fitness);
    // rank_population + select_best of the pool in one device pass
    // (src/engine.cpp:258-262); only the survivor order comes back
    const std::vector<int> keep = b200::select_on_device(b200::Device::default_device(), fits, pop);
    std::vector<Individual> next;
    next.reserve(pop);
    for (int i : keep)
        next.push_back(std::move(pool[static_cast<size_t>(i)]));
    population_ = std::move(next);
    lap(tr.rank_ms);
    for (const auto& ind : population_)
        archive_add(ind);
    lap(tr.archive_ms);
    rank_current();
    ++generation_;
    log_generation(gen_stats);
}

void Engine::archive_add(const Individual& ind) {
    if (!ind.fitness)
        return;
    const FitnessVector f = *ind.fitness;
    for (const auto& e : archive_) {
        const FitnessVector& g = *e.ind.fitness;
        if (g == f || dominates(g, f))
            return;
    }
    archive_.erase(std::remove_if(archive_.begin(), archive_.end(),
                                  [&](const ArchiveEntry& e) { return dominates(f, *e.ind.fitness); }),
                   archive_.end());
    ArchiveEntry e;
    e.ind = ind;
    archive_.push_back(std::move(e));
}

void Engine::rank_current() { rank_ = rank_population(population_fitness()); }

std::vector<FitnessVector> Engine::population_fitness() const {
    std::vector<FitnessVector> fits;
    fits.reserve(population_.size());
    for (const auto& ind : population_)
        fits.push_back(*ind.fitness);
    return fits;
}

void Engine::log_generation(const OperatorStats& gs) {
    GenerationLog row;
    row.gen = generation_;
    const double inf = std::numeric_limits<double>::infinity();
    double b0 = inf, bt = inf, me = inf;
    auto see = [&](const FitnessVector& f) {
        if (f.error == 0.0)
            b0 = std::min(b0, f.cost);
        bt = std::min(bt, f.cost);
        me = std::min(me, f.error);
    };
    for (const auto& ind : population_)
        see(*ind.fitness);
    for (const auto& e : archive_)
        see(*e.ind.fitness);
    row.best_cost_err0 = b0;
    row.best_cost_tol = bt;
    row.min_error = me;
    row.front0_size = rank_.fronts.empty() ? 0 : static_cast<int>(rank_.fronts[0].size());
    row.mut_attempts = gs.total_attempts();
    row.mut_accepts = gs.total_accepts();
    row.cx_attempts = gs.cx_attempts;
    row.cx_accepts = gs.cx_accepts;
    log_.push_back(row);
}

SearchResult Engine::run(const std::vector<TestCase>& heldout) {
    const auto t_run = std::chrono::steady_clock::now();
    Trace::get() = Trace{};
    initialize_population();
    if (cfg_.budget.kind == Budget::Kind::Generations) {
        for (int g = 0; g < cfg_.budget.generations; ++g)
            step_generation();
    } else {
        const auto start = std::chrono::steady_clock::now();
        while (ms_since(start) / 1000.0 < cfg_.budget.seconds)
            step_generation();
    }
    if (!heldout.empty()) {
        b200::DeviceSuite hs(b200::Device::default_device(),
                             b200::build_suite(original_.params, heldout));
        std::vector<const Kernel*> ks;
        for (const auto& e : archive_)
            ks.push_back(&e.ind.kernel);
        const auto v = device_verdicts(hs, *exec_img_, ks, cfg_.tolerance, false, counters_, cfg_.jobs);
        for (size_t i = 0; i < archive_.size(); ++i) {
            if (v[i].accepted) {
                archive_[i].heldout_error = v[i].fitness.error;
                archive_[i].overfit = false;
            } else {
                archive_[i].heldout_error = 1.0;
                archive_[i].overfit = true;
            }
        }
    }
    if (Trace::on())
        std::fprintf(stderr,
                     "[gevo trace] run %.1f ms: verdicts %.1f (encode+gen %.1f, evaluate %.1f, "
                     "device %.1f), other host %.1f; select %.1f cx %.1f mut %.1f rank %.1f "
                     "archive %.1f (archive size %zu); cx gen %.1f resolve %.1f, mut gen %.1f "
                     "resolve %.1f\n",
                     ms_since(t_run), Trace::get().verdicts_ms, counters_.host_gen_ms,
                     Trace::get().eval_ms, counters_.device_ms,
                     ms_since(t_run) - Trace::get().verdicts_ms, Trace::get().select_ms,
                     Trace::get().cx_ms, Trace::get().mut_ms, Trace::get().rank_ms,
                     Trace::get().archive_ms, archive_.size(), Trace::get().cx_gen_ms,
                     Trace::get().cx_resolve_ms, Trace::get().mut_gen_ms, Trace::get().mut_resolve_ms);
    SearchResult r;
    r.population = population_;
    r.archive = archive_;
    r.log = log_;
    r.stats = stats_;
    r.baseline = baseline_;
    r.generations_run = generation_;
    for (size_t i = 0; i < r.archive.size(); ++i) {
        const ArchiveEntry& e = r.archive[i];
        if (e.overfit)
            continue;
        if (r.best_index < 0) {
            r.best_index = static_cast<int>(i);
            continue;
        }
        const FitnessVector& best = *r.archive[static_cast<size_t>(r.best_index)].ind.fitness;
        const FitnessVector& c = *e.ind.fitness;
        if (c.cost < best.cost || (c.cost == best.cost && c.error < best.error))
            r.best_index = static_cast<int>(i);
    }
    return r;
}

SearchResult run_search(const Kernel& original, const SearchConfig& cfg,
                        const std::vector<TestCase>& tests, const std::vector<TestCase>& heldout) {
    Engine engine(original, cfg, tests);
    return engine.run(heldout);
}

} // namespace evoir
