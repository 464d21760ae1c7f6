// Device runtime: memory, uploads, launches and read-back for the batched
// interpreter and the GPU ranking. Called from the C++ host (engine, evoir::
// wrappers) and the C ABI.
#include "../host/runtime.hpp"
#include "interp.cuh"
#include "nsga_rank.cuh"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h> // types only: the library is opened at run time (see nccl_api)

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

namespace evoir::b200 {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// Growable device allocation.
struct DevBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void reserve(size_t bytes) {
        if (bytes <= cap)
            return;
        if (ptr)
            cudaFree(ptr);
        ptr = nullptr;
        const size_t want = std::max<size_t>(bytes, cap * 3 / 2);
        check(cudaMalloc(&ptr, want), "cudaMalloc");
        cap = want;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
    ~DevBuf() {
        if (ptr)
            cudaFree(ptr);
    }
};

// Growable pinned host staging buffer.
struct PinnedBuf {
    void* ptr = nullptr;
    size_t cap = 0;
    void reserve(size_t bytes) {
        if (bytes <= cap)
            return;
        if (ptr)
            cudaFreeHost(ptr);
        const size_t want = std::max<size_t>(bytes, cap * 3 / 2);
        check(cudaMallocHost(&ptr, want), "cudaMallocHost");
        cap = want;
    }
    ~PinnedBuf() {
        if (ptr)
            cudaFreeHost(ptr);
    }
};

} // namespace

namespace {
// NCCL entry points, resolved when a communicator is first wanted: the copy
// already in the process (e.g. the one torch loaded) when there is one, else
// GEVO_NCCL_LIB or the system libnccl.so.2. Not linked at build time, so a
// process never ends up with two NCCL builds under one soname.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
};
const NcclApi& nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* e = std::getenv("GEVO_NCCL_LIB");
            h = dlopen(e ? e : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h)
            throw std::runtime_error(std::string("NCCL not found: ") + dlerror());
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.comm_destroy)
            throw std::runtime_error("NCCL library lacks an entry point");
        return a;
    }();
    return api;
}
} // namespace

// Device scratch of one evaluation stream: records, per-instance memory,
// spin-accelerator state. The device owns one (synchronous calls); every
// resident batch owns another, so batches can be evaluated concurrently on
// their own streams.
struct Scratch {
    DevBuf rec, vrec, first_fail, priv, sh_tag, sh_val;
    DevBuf ts_pos, ts_prev, ts_exec, ts_stop, ts_val, ts_tag;
    DevBuf tp_snap, gcells, gshadow, outcells, suffix, sp_vk;
    DevBuf bcost, vf, sp_base, sp_btag, sp_delta, sp_cur, sp_hvary, sp_cvary, sp_log, sp_ld;
    // bytes of per-instance scratch per launch (GEVO_SCRATCH_GB); larger
    // batches run in several launches
    size_t scratch_budget = [] {
        const char* e = std::getenv("GEVO_SCRATCH_GB");
        return (e ? static_cast<size_t>(std::max(1, std::atoi(e))) : size_t(8)) << 30;
    }();
    DevBuf cta_clock; // diagnostic per-CTA timing (GEVO_CTA_CLOCK=1)
    DevBuf regions;   // thread-parallel region ring + tickets
    DevBuf sched;     // persistent launches: queue counters, deferred items, claims, per-variant counts
};

struct DeviceImpl {
    int ordinal = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr; // created here; `stream` may be a caller's
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    DevBuf blob, counters, rank;
    gevo::RankWorkspace rws; // GPU rank_population / select_best buffers
    PinnedBuf h_rank;        // their host staging (inputs in, outputs back)
    ncclComm_t nccl = nullptr; // record exchange of a multi-GPU search
    int nccl_rank = 0, nccl_world = 0;
    DevBuf gathered;           // all-gathered variant records
    Scratch sc;
    PinnedBuf h_blob, h_vrec, h_rec;
};

struct SuiteImpl {
    DevBuf param_tag, param_payload, buf_size, buf_elem, buf_info, setup_code, setup_aux, pool,
        entry_begin, entries, static_err;
};

Device::Device(int ordinal) : impl_(std::make_unique<DeviceImpl>()) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        throw DeviceUnavailable("no CUDA device available: the B200 interpreter has no CPU path");
    }
    if (ordinal < 0) {
        const char* env = std::getenv("GEVO_DEVICE");
        if (env)
            ordinal = std::atoi(env);
        else
            check(cudaGetDevice(&ordinal), "cudaGetDevice");
    }
    impl_->ordinal = ordinal;
    check(cudaSetDevice(ordinal), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&impl_->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    impl_->stream = impl_->own_stream;
    check(cudaEventCreate(&impl_->ev0), "cudaEventCreate");
    check(cudaEventCreate(&impl_->ev1), "cudaEventCreate");
    check(cudaEventCreate(&impl_->ev2), "cudaEventCreate");
}

Device::~Device() {
    gevo::rank_release(impl_->rws);
    // (a communicator still set at exit is left to the process teardown)
    if (impl_->own_stream)
        cudaStreamDestroy(impl_->own_stream);
    cudaEventDestroy(impl_->ev0);
    cudaEventDestroy(impl_->ev1);
    cudaEventDestroy(impl_->ev2);
}

int Device::ordinal() const { return impl_->ordinal; }

void Device::set_stream(void* stream) {
    std::lock_guard<std::mutex> g(mu_);
    impl_->stream = stream ? static_cast<cudaStream_t>(stream) : impl_->own_stream;
}

Device& Device::default_device() {
    static Device* dev = new Device(-1); // intentionally leaked: outlives static teardown
    return *dev;
}

namespace {

template <typename T>
void upload(DevBuf& b, const std::vector<T>& v, cudaStream_t s) {
    b.reserve(std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty())
        check(cudaMemcpyAsync(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s),
              "upload");
}

} // namespace

DeviceSuite::DeviceSuite(Device& dev, SuiteImage image)
    : dev_(dev), image_(std::move(image)), impl_(std::make_unique<SuiteImpl>()) {
    std::lock_guard<std::mutex> g(dev_.lock());
    check(cudaSetDevice(dev_.ordinal()), "cudaSetDevice");
    cudaStream_t s = dev_.impl().stream;
    SuiteImpl& d = *impl_;
    upload(d.param_tag, image_.param_tag, s);
    upload(d.param_payload, image_.param_payload, s);
    upload(d.buf_size, image_.buf_size, s);
    upload(d.buf_elem, image_.buf_elem, s);
    // [test][param] {size << 8 | elem, word offset of the param's element 0 for
    // this test in the interleaved pool}: one 8-byte load per global access
    std::vector<uint32_t> info(image_.buf_size.size() * 2);
    for (size_t i = 0; i < image_.buf_size.size(); ++i) {
        const size_t t = i / std::max(image_.n_params, 1), p = i % std::max(image_.n_params, 1);
        const uint64_t off = image_.pool_off[p] + t;
        if (off > 0xFFFFFFFFull)
            throw std::invalid_argument("test input pool exceeds 2^32 words");
        info[2 * i] = (static_cast<uint32_t>(std::max(image_.buf_size[i], 0)) << 8) | image_.buf_elem[i];
        info[2 * i + 1] = static_cast<uint32_t>(off);
    }
    upload(d.buf_info, info, s);
    upload(d.setup_code, image_.setup_code, s);
    upload(d.setup_aux, image_.setup_aux, s);
    upload(d.pool, image_.pool, s);
    upload(d.entry_begin, image_.entry_begin, s);
    std::vector<gevo::OracleEntryDev> ents;
    for (const auto& e : image_.entries)
        ents.push_back(gevo::OracleEntryDev{e.param, e.size, e.off, e.elem, 0});
    upload(d.entries, ents, s);
    upload(d.static_err, image_.static_err, s);
    check(cudaStreamSynchronize(s), "suite upload");
}

DeviceSuite::~DeviceSuite() = default;

namespace {

// Scratch bytes one instance needs in a launch.
size_t scratch_per_instance(const SuiteImage& S, uint64_t writable_any, const ExecImage& ex,
                            bool any_sync, uint32_t max_values, uint32_t max_slots, bool vf_global) {
    size_t b = 0;
    for (int p = 0; p < S.n_params; ++p)
        if ((writable_any >> p) & 1ull)
            b += 4 * static_cast<size_t>(S.pool_rows[static_cast<size_t>(p)]);
    b += 5 * static_cast<size_t>(std::max(ex.shared_words, 0));
    if (any_sync)
        b += static_cast<size_t>(ex.threads) * (4 + 4 + 8 + 4 + 5 * static_cast<size_t>(max_values));
    b += 15 * static_cast<size_t>(max_slots) + 28 * gevo::kSpinLog; // spin accelerator
    if (vf_global)
        b += 8 * static_cast<size_t>(max_slots);
    return b;
}

// Fills everything but the batch pointers and the per-chunk window.
gevo::InterpArgs base_args(DeviceSuite& suite, const ExecImage& ex, const EvalOptions& opt) {
    gevo::InterpArgs A{};
    const SuiteImage& S = suite.image();
    SuiteImpl& d = suite.impl();
    A.n_tests = S.n_tests;
    A.n_params = S.n_params;
    A.param_tag = d.param_tag.as<uint8_t>();
    A.param_payload = d.param_payload.as<uint32_t>();
    A.buf_size = d.buf_size.as<int32_t>();
    A.buf_elem = d.buf_elem.as<uint8_t>();
    A.buf_info = d.buf_info.as<uint2>();
    A.setup_code = d.setup_code.as<uint8_t>();
    A.setup_aux = d.setup_aux.as<int32_t>();
    A.pool = d.pool.as<uint32_t>();
    A.entry_begin = d.entry_begin.as<int32_t>();
    A.entries = d.entries.as<gevo::OracleEntryDev>();
    A.static_err = d.static_err.as<uint8_t>();
    for (int p = 0; p < S.n_params; ++p)
        A.pool_off[p] = S.pool_off[static_cast<size_t>(p)];
    A.threads = ex.threads;
    A.shared_words = ex.shared_words;
    A.budget = ex.budget;
    for (int c = 0; c < GEVO_COST_CLASSES; ++c)
        A.cost[c] = ex.cost[static_cast<size_t>(c)];
    A.tolerance = opt.tolerance;
    A.early_exit = opt.early_exit ? 1 : 0;
    return A;
}

void bind_batch(gevo::InterpArgs& A, const void* dblob, const gevo_batch_header& h) {
    const char* base = static_cast<const char*>(dblob);
    A.variants = reinterpret_cast<const gevo_variant*>(base + h.off_variants);
    A.blocks = reinterpret_cast<const gevo_block*>(base + h.off_blocks);
    A.insts = reinterpret_cast<const gevo_inst*>(base + h.off_insts);
    A.arms = reinterpret_cast<const gevo_arm*>(base + h.off_arms);
    A.edges = reinterpret_cast<const gevo_edge*>(base + h.off_edges);
    A.lit_payload = reinterpret_cast<const uint32_t*>(base + h.off_lit_payload);
    A.lit_tag = reinterpret_cast<const uint8_t*>(base + h.off_lit_tag);
    A.n_variants = h.n_variants;
    A.max_slots = std::max<uint32_t>(h.max_slots, 1);
    A.lane_slots = std::max<uint32_t>(h.max_lane_slots, 1);
    A.max_lits = h.max_lits;
    A.ts_slots = std::max<uint32_t>(h.max_values, 1);
}

// Spin accelerator arms after this many instructions of one simulated thread
// (clean corpus threads run <= ~750; GEVO_SPIN_THRESHOLD=0 disables it).
int64_t spin_threshold() {
    static const int64_t v = [] {
        const char* e = std::getenv("GEVO_SPIN_THRESHOLD");
        return e ? std::atoll(e) : int64_t(256);
    }();
    return v;
}

// Spin accelerator pay factor (GEVO_SPIN_PAY): an attempt costs the lane a
// few passes over its value file in global scratch, so a partial jump that
// skipped fewer than spin_pay * n_values instructions backs off like a failed
// attempt instead of re-arming at once (0: always re-arm).
uint32_t spin_pay() {
    static const uint32_t v = [] {
        const char* e = std::getenv("GEVO_SPIN_PAY");
        return e ? static_cast<uint32_t>(std::atoi(e)) : 256u;
    }();
    return v;
}

// GEVO_TP=0 forces the sequential-lane interpreter.
bool tp_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("GEVO_TP");
        return !(e && e[0] == '0');
    }();
    return v;
}

// GEVO_CTA_CLOCK=1: the thread-parallel kernel records per-CTA timing.
bool cta_clock_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("GEVO_CTA_CLOCK");
        return e && e[0] == '1';
    }();
    return v;
}

struct CtaClockRef {
    const DevBuf* buf = nullptr;
    size_t bytes = 0;
};
CtaClockRef& last_cta_clock() {
    static CtaClockRef r;
    return r;
}

// GEVO_RECONV=0/1 forces the reconvergence gate off/on; by default it is on
// when the lanes of a warp are threads of one test.
int reconv_mode() {
    static const int v = [] {
        const char* e = std::getenv("GEVO_RECONV");
        return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    return v;
}

// GEVO_STAGE=0: the thread-parallel interpreter fetches instruction records
// from global memory (__ldg) instead of a TMA-staged shared-memory copy.
bool stage_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("GEVO_STAGE");
        return !(e && e[0] == '0');
    }();
    return v;
}

// GEVO_TP_PERSIST=1: persistent global-cell launches with the deferring work
// queue (measured no faster on config 4: speculative later tests only run in
// slots the draining batch leaves idle anyway), off by default.
bool persist_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("GEVO_TP_PERSIST");
        return e && e[0] == '1';
    }();
    return v;
}

// GEVO_TP_REGIONS=0 gives every instance its own scratch columns (one
// launch per scratch budget) instead of the per-CTA region pool.
bool regions_enabled() {
    static const bool v = [] {
        const char* e = std::getenv("GEVO_TP_REGIONS");
        return !(e && e[0] == '0');
    }();
    return v;
}

// Spin-accelerator scratch for `cols` columns (instances or lanes).
void reserve_spin(Scratch& sc, gevo::InterpArgs& A, size_t cols) {
    const size_t n = cols * A.max_slots;
    sc.sp_base.reserve(n * 4);
    sc.sp_btag.reserve(n);
    sc.sp_delta.reserve(n * 4);
    sc.sp_cur.reserve(n * 4);
    sc.sp_hvary.reserve(n);
    sc.sp_cvary.reserve(n);
    sc.sp_log.reserve(cols * gevo::kSpinLog * 5 * 4);
    sc.sp_ld.reserve(cols * gevo::kSpinLog * 4);
    sc.sp_vk.reserve(cols * gevo::kSpinLog * 4);
    A.sp_vk = sc.sp_vk.as<uint32_t>();
    A.sp_hvary = sc.sp_hvary.as<uint8_t>();
    A.sp_cvary = sc.sp_cvary.as<uint8_t>();
    A.sp_log = sc.sp_log.as<uint32_t>();
    A.sp_ld = sc.sp_ld.as<uint32_t>();
    A.sp_base = sc.sp_base.as<uint32_t>();
    A.sp_btag = sc.sp_btag.as<uint8_t>();
    A.sp_delta = sc.sp_delta.as<uint32_t>();
    A.sp_cur = sc.sp_cur.as<uint32_t>();
}

// Launches the interpreter over all variants in scratch-bounded chunks, then
// the per-variant reduction. Records land in dev.sc.rec / dev.sc.vrec.
// Where the final global buffers of the instances are after a launch
// (want_outputs): the sequential kernel's private copies (u32 words) or the
// thread-parallel kernel's memory cells (uint2, payload in .x); element e of
// writable param p of launch-local instance il is at (off[p] + e) * n_inst + il.
struct OutputWindow {
    int mode = 0; // 0 none, 1 u32 words, 2 uint2 cells
    const void* ptr = nullptr;
    size_t n_inst = 0, words = 0;
    std::vector<size_t> off;
};

int launch_all(DeviceImpl& dev, Scratch& sc, DeviceSuite& suite, gevo::InterpArgs A, const gevo_batch_header& h,
               uint64_t writable_any, const ExecImage& ex, const EvalOptions& opt,
               cudaStream_t s, OutputWindow* ow = nullptr) {
    const SuiteImage& S = suite.image();
    if (h.max_slots > gevo::kMaxSlots)
        throw std::invalid_argument("variant value file exceeds the device limit");
    const uint32_t T = static_cast<uint32_t>(std::max(S.n_tests, 1));
    const uint64_t total = static_cast<uint64_t>(h.n_variants) * static_cast<uint64_t>(S.n_tests);
    sc.rec.reserve(std::max<size_t>(total * sizeof(gevo_test_record), 16));
    sc.vrec.reserve(std::max<size_t>(h.n_variants * sizeof(gevo_variant_record), 16));
    sc.first_fail.reserve(std::max<size_t>(h.n_variants * sizeof(int32_t), 16));
    if (opt.early_exit)
        check(cudaMemsetAsync(sc.first_fail.ptr, 0x7f, h.n_variants * sizeof(int32_t), s),
              "memset first_fail");
    A.rec = sc.rec.as<gevo_test_record>();
    A.first_fail = sc.first_fail.as<int32_t>();
    int launches = 0;

    // Block costs under this launch's cost table.
    sc.bcost.reserve(std::max<size_t>(h.n_blocks * sizeof(uint4), 16));
    sc.suffix.reserve(std::max<size_t>(h.n_insts * sizeof(int64_t), 16));
    check(gevo::launch_block_cost(A.blocks, A.insts, A.variants, h.n_variants, ex.cost.data(),
                                  sc.bcost.as<uint4>(), sc.suffix.as<int64_t>(), s),
          "block_cost_kernel launch");
    ++launches;
    A.dblocks = sc.bcost.as<uint4>();
    A.suffix = sc.suffix.as<int64_t>();

    const int64_t thr = spin_threshold();
    if (!dev.counters.ptr) {
        dev.counters.reserve(48);
        check(cudaMemsetAsync(dev.counters.ptr, 0, 48, s), "counters");
    }
    A.counters = dev.counters.as<uint64_t>();
    A.cta_clock = nullptr;
    if (cta_clock_enabled()) {
        const size_t bytes = std::max<size_t>(static_cast<size_t>(h.n_variants) * T * 32, 32);
        sc.cta_clock.reserve(bytes);
        check(cudaMemsetAsync(sc.cta_clock.ptr, 0, bytes, s), "cta clock");
        A.cta_clock = sc.cta_clock.as<unsigned long long>();
        last_cta_clock() = {&sc.cta_clock, bytes};
    }

    // Thread-parallel lanes (one lane per simulated thread) whenever the
    // instance state fits on chip; the sequential-lane kernel otherwise.
    uint32_t n_cells = static_cast<uint32_t>(std::max(ex.shared_words, 0));
    for (int p = 0; p < S.n_params; ++p) {
        A.cell_off[p] = n_cells;
        if ((writable_any >> p) & 1ull)
            n_cells += static_cast<uint32_t>(S.pool_rows[static_cast<size_t>(p)]);
    }
    const uint32_t n_chunks = std::max<uint32_t>((n_cells + 31) / 32, 1);
    const uint32_t threads = static_cast<uint32_t>(std::max(ex.threads, 1));
    // on-chip instance memory first; global cells when it does not fit
    // records staged by TMA for the global-cell (256-thread) kernels, where
    // it measured +3 %; the corpus kernels keep __ldg (staging measured -4 %)
    A.stage_recs = 0;
    A.n_insts_total = h.n_insts;
    gevo::TpTables tab{A.lane_slots, A.max_slots, static_cast<uint32_t>(S.n_params), A.max_lits, 0};
    gevo::TpShape tps = gevo::tp_shape(threads, T, tab, n_cells, n_chunks, h.any_sync != 0);
    bool gc = false;
    if (tps.warps_per_cta == 0) {
        tab.stage_recs = A.stage_recs = stage_enabled() ? h.max_insts : 0;
        tps = gevo::tp_shape(threads, T, tab, 0, 0, false, true);
        gc = tps.warps_per_cta > 0;
        if (!gc)
            A.stage_recs = 0;
    }
    if (ex.threads >= 1 && !opt.sequential && tps.warps_per_cta > 0 && tp_enabled()) {
        A.tp_lanes = tps.lanes;
        const uint32_t tgroups = (T + tps.lanes - 1) / tps.lanes;
        A.n_cells = n_cells;
        A.n_chunks = n_chunks;
        A.reconv = reconv_mode() >= 0 ? static_cast<uint32_t>(reconv_mode())
                                      : static_cast<uint32_t>(tps.lanes == 1);
        const size_t per_lane = thr > 0 ? 15 * static_cast<size_t>(A.max_slots) + 28 * gevo::kSpinLog
                                        : 0;
        const size_t lanes_per_variant = static_cast<size_t>(tgroups) * 32 * tps.warps_per_cta;
        // global cells + access records: 16 bytes per cell per instance
        const size_t per_variant = std::max<size_t>(per_lane, 1) * lanes_per_variant +
                                   (gc ? 16 * static_cast<size_t>(n_cells) * T : 0);
        size_t chunk = std::max<size_t>(sc.scratch_budget / per_variant, 1);
        chunk = std::min<size_t>(chunk, std::max<uint32_t>(h.n_variants, 1));
        if (opt.want_outputs)
            chunk = std::max<uint32_t>(h.n_variants, 1); // one launch window
        // per-CTA regions: scratch for the CTAs that can be resident, one
        // launch for the whole batch (outputs read back per instance keep
        // the per-instance layout)
        A.regions = 0;
        A.persist = 0;
        if (gc && regions_enabled() && !opt.want_outputs) {
            A.regions = gevo::tp_resident_ctas(gc, tps.warps_per_cta, tps.smem);
            chunk = std::max<uint32_t>(h.n_variants, 1);
            sc.regions.reserve((static_cast<size_t>(A.regions) + 2) * 4);
            A.region_ctr = sc.regions.as<uint32_t>();
            A.region_q = A.region_ctr + 2;
            // persistent CTAs with the deferring work queue (GEVO_TP_PERSIST=1)
            if (persist_enabled()) {
                const size_t items = static_cast<size_t>(chunk) * tgroups;
                const size_t words = 4 + 2 * items + chunk;
                sc.sched.reserve(words * 4);
                A.persist = 1;
                A.n_items = static_cast<uint32_t>(items);
                A.sched = sc.sched.as<uint32_t>();
                A.defer = A.sched + 4;
                A.claim = A.defer + items;
                A.vdone = A.claim + items;
                check(cudaMemsetAsync(A.sched, 0, 16, s), "sched");
                check(cudaMemsetAsync(A.defer, 0xFF, items * 4, s), "sched");
                check(cudaMemsetAsync(A.claim, 0, (items + chunk) * 4, s), "sched");
            }
        }
        const size_t lanes = A.regions ? static_cast<size_t>(A.regions) * 32 * tps.warps_per_cta
                                       : chunk * lanes_per_variant;
        if (thr > 0) {
            reserve_spin(sc, A, lanes);
            A.spin_threshold = thr;
            A.spin_pay = spin_pay();
        }
        A.tp_snap = nullptr;
        A.out_cells = nullptr;
        A.gcells = nullptr;
        A.gshadow = nullptr;
        if (gc) {
            const size_t cols = A.regions ? static_cast<size_t>(A.regions) * tps.lanes : chunk * T;
            const size_t cells = std::max<size_t>(static_cast<size_t>(n_cells) * cols, 1);
            sc.gcells.reserve(cells * 8);
            sc.gshadow.reserve(cells * 8);
            A.gcells = sc.gcells.as<uint2>();
            A.gshadow = sc.gshadow.as<unsigned long long>();
        } else if (h.any_sync) {
            sc.tp_snap.reserve(lanes * std::max<uint32_t>(h.max_values, 1) * 8);
            A.tp_snap = sc.tp_snap.as<uint2>();
        }
        if (opt.want_outputs && ow) {
            const size_t n_inst = static_cast<size_t>(h.n_variants) * T;
            if (!gc) {
                sc.outcells.reserve(std::max<size_t>(static_cast<size_t>(n_cells) * n_inst * 8, 16));
                A.out_cells = sc.outcells.as<uint2>();
            }
            ow->mode = 2;
            ow->ptr = gc ? static_cast<const void*>(A.gcells) : static_cast<const void*>(A.out_cells);
            ow->n_inst = n_inst;
            ow->words = n_cells;
            ow->off.assign(A.cell_off, A.cell_off + S.n_params);
        }
        for (uint64_t vb = 0; vb < h.n_variants; vb += chunk) {
            gevo::InterpArgs L = A;
            L.v_begin = static_cast<uint32_t>(vb);
            L.n_var = static_cast<uint32_t>(std::min<uint64_t>(chunk, h.n_variants - vb));
            L.n_inst = L.n_var * T;
            L.n_spin = static_cast<uint32_t>(A.regions ? lanes : L.n_var * lanes_per_variant);
            if (gc && !A.regions) // (regions clear their records when taken)
                check(cudaMemsetAsync(A.gshadow, 0,
                                      static_cast<size_t>(n_cells) * L.n_inst * 8, s),
                      "access records");
            check(gevo::launch_interp_tp(L, s), "interp_tp_kernel launch");
            ++launches;
        }
        check(gevo::launch_fitness(sc.rec.as<gevo_test_record>(), h.n_variants, S.n_tests,
                                   opt.tolerance, sc.vrec.as<gevo_variant_record>(), s),
              "fitness_kernel launch");
        return launches + 1;
    }

    const gevo::LaunchShape shape = gevo::interp_shape(S.n_tests, A.max_slots);
    A.row_lanes = shape.row_lanes;
    A.vf_global = shape.vf_global ? 1 : 0;
    A.warps_per_variant = (T + 31) / 32;

    const size_t per = std::max<size_t>(
        scratch_per_instance(S, writable_any, ex, h.any_sync != 0, h.max_values, A.max_slots,
                             shape.vf_global),
        1);
    // chunk = variants per launch
    size_t chunk = std::max<size_t>(sc.scratch_budget / (per * T), 64);
    chunk = std::min<size_t>(chunk, std::max<uint32_t>(h.n_variants, 1));
    const size_t cap = chunk * T; // instances per launch window
    size_t priv_words = 0;
    for (int p = 0; p < S.n_params; ++p)
        if ((writable_any >> p) & 1ull)
            priv_words += static_cast<size_t>(S.pool_rows[static_cast<size_t>(p)]);
    sc.priv.reserve(std::max<size_t>(priv_words * cap * 4, 16));
    const size_t sw = static_cast<size_t>(std::max(ex.shared_words, 0));
    sc.sh_tag.reserve(std::max<size_t>(sw * cap, 16));
    sc.sh_val.reserve(std::max<size_t>(sw * cap * 4, 16));
    A.priv = sc.priv.as<uint32_t>();
    A.sh_tag = sc.sh_tag.as<uint8_t>();
    A.sh_val = sc.sh_val.as<uint32_t>();
    if (h.any_sync) {
        const size_t tn = static_cast<size_t>(ex.threads) * cap;
        sc.ts_pos.reserve(tn * 4);
        sc.ts_prev.reserve(tn * 4);
        sc.ts_exec.reserve(tn * 8);
        sc.ts_stop.reserve(tn * 4);
        sc.ts_val.reserve(tn * A.ts_slots * 4);
        sc.ts_tag.reserve(tn * A.ts_slots);
        A.ts_pos = sc.ts_pos.as<int32_t>();
        A.ts_prev = sc.ts_prev.as<int32_t>();
        A.ts_exec = sc.ts_exec.as<int64_t>();
        A.ts_stop = sc.ts_stop.as<uint32_t>();
        A.ts_val = sc.ts_val.as<uint32_t>();
        A.ts_tag = sc.ts_tag.as<uint8_t>();
    }
    if (shape.vf_global) {
        sc.vf.reserve(cap * A.max_slots * 8);
        A.vf = sc.vf.as<uint2>();
    }
    if (thr > 0) {
        reserve_spin(sc, A, cap);
        A.spin_threshold = thr;
        A.spin_pay = spin_pay();
    }
    if (opt.want_outputs && ow) {
        if (chunk < h.n_variants)
            throw std::invalid_argument("want_outputs needs a single-launch batch");
        ow->mode = 1;
        ow->ptr = sc.priv.ptr;
        ow->n_inst = static_cast<size_t>(h.n_variants) * T;
        ow->off.assign(static_cast<size_t>(S.n_params), 0);
        size_t words = 0;
        for (int p = 0; p < S.n_params; ++p) {
            ow->off[static_cast<size_t>(p)] = words;
            if ((writable_any >> p) & 1ull)
                words += static_cast<size_t>(S.pool_rows[static_cast<size_t>(p)]);
        }
        ow->words = words;
    }
    for (uint64_t vb = 0; vb < h.n_variants; vb += chunk) {
        gevo::InterpArgs L = A;
        L.v_begin = static_cast<uint32_t>(vb);
        L.n_var = static_cast<uint32_t>(std::min<uint64_t>(chunk, h.n_variants - vb));
        L.n_inst = L.n_var * T;
        L.n_spin = L.n_inst;
        size_t words = 0;
        for (int p = 0; p < S.n_params; ++p) {
            L.priv_off[p] = words * L.n_inst;
            if ((writable_any >> p) & 1ull)
                words += static_cast<size_t>(S.pool_rows[static_cast<size_t>(p)]);
        }
        check(gevo::launch_interp(L, s), "interp_kernel launch");
        ++launches;
    }
    check(gevo::launch_fitness(sc.rec.as<gevo_test_record>(), h.n_variants, S.n_tests,
                               opt.tolerance, sc.vrec.as<gevo_variant_record>(), s),
          "fitness_kernel launch");
    return launches + 1;
}

uint64_t writable_union(BatchImage& batch) { return batch.writable_union(); }

} // namespace

EvalResult evaluate(DeviceSuite& suite, BatchImage& batch, const ExecImage& exec,
                    const EvalOptions& opt) {
    Device& devh = suite.device();
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    cudaStream_t s = dev.stream;
    const SuiteImage& S = suite.image();
    EvalResult R;
    const gevo_batch_header h = batch.header();
    const uint64_t wr = writable_union(batch);
    const size_t bytes = h.total_bytes;

    dev.h_blob.reserve(bytes);
    batch.write_blob(static_cast<uint8_t*>(dev.h_blob.ptr)); // straight into pinned staging
    dev.blob.reserve(bytes + 64); // slack: the interpreter prefetches one record ahead
    check(cudaEventRecord(dev.ev0, s), "event");
    check(cudaMemcpyAsync(dev.blob.ptr, dev.h_blob.ptr, bytes, cudaMemcpyHostToDevice, s),
          "blob H2D");
    R.h2d_bytes = bytes;
    gevo::InterpArgs A = base_args(suite, exec, opt);
    bind_batch(A, dev.blob.ptr, h);
    check(cudaEventRecord(dev.ev1, s), "event");
    OutputWindow ow;
    R.launches = launch_all(dev, dev.sc, suite, A, h, wr, exec, opt, s, &ow);
    check(cudaEventRecord(dev.ev2, s), "event");

    if (opt.gather_count > 0 && dev.nccl) {
        // device-resident exchange: this rank's records (padded to the
        // largest shard) are all-gathered over NVLink by NCCL, then one D2H
        const size_t rb = sizeof(gevo_variant_record), m = opt.gather_count;
        if (h.n_variants > m)
            throw std::logic_error("shard larger than gather_count");
        dev.sc.vrec.reserve(m * rb);
        if (m > h.n_variants)
            check(cudaMemsetAsync(dev.sc.vrec.as<char>() + h.n_variants * rb, 0,
                                  (m - h.n_variants) * rb, s),
                  "gather pad");
        const size_t W = static_cast<size_t>(dev.nccl_world);
        dev.gathered.reserve(W * m * rb);
        if (nccl_api().all_gather(dev.sc.vrec.ptr, dev.gathered.ptr, m * rb, ncclUint8, dev.nccl, s) !=
            ncclSuccess)
            throw std::runtime_error("ncclAllGather of the variant records failed");
        R.variants.resize(W * m);
        check(cudaMemcpyAsync(R.variants.data(), dev.gathered.ptr, W * m * rb, cudaMemcpyDeviceToHost, s),
              "records D2H");
        R.d2h_bytes += W * m * rb;
    } else {
        R.variants.resize(h.n_variants);
        if (h.n_variants) {
            check(cudaMemcpyAsync(R.variants.data(), dev.sc.vrec.ptr,
                                  h.n_variants * sizeof(gevo_variant_record), cudaMemcpyDeviceToHost, s),
                  "records D2H");
            R.d2h_bytes += h.n_variants * sizeof(gevo_variant_record);
        }
    }
    const size_t total = static_cast<size_t>(h.n_variants) * S.n_tests;
    if (opt.want_tests || opt.want_outputs) {
        R.tests.resize(total);
        if (total)
            check(cudaMemcpyAsync(R.tests.data(), dev.sc.rec.ptr, total * sizeof(gevo_test_record),
                                  cudaMemcpyDeviceToHost, s),
                  "test records D2H");
        R.d2h_bytes += total * sizeof(gevo_test_record);
    }
    std::vector<uint32_t> win;
    const size_t wsz = ow.mode == 2 ? 2 : 1; // u32 per element
    if (opt.want_outputs && total && ow.mode) {
        win.resize(ow.words * ow.n_inst * wsz);
        if (!win.empty())
            check(cudaMemcpyAsync(win.data(), ow.ptr, win.size() * 4, cudaMemcpyDeviceToHost, s),
                  "outputs D2H");
    }
    check(cudaStreamSynchronize(s), "evaluate");
    float ms = 0.0f;
    check(cudaEventElapsedTime(&ms, dev.ev1, dev.ev2), "elapsed");
    R.kernel_ms = ms;

    if (opt.want_outputs && total) {
        const auto* vars = reinterpret_cast<const gevo_variant*>(static_cast<const uint8_t*>(dev.h_blob.ptr) +
                                                                 h.off_variants);
        R.outputs.assign(h.n_variants, std::vector<BufferMap>(static_cast<size_t>(S.n_tests)));
        for (uint32_t v = 0; v < h.n_variants; ++v)
            for (int t = 0; t < S.n_tests; ++t) {
                const size_t gi = static_cast<size_t>(v) * S.n_tests + t;
                if (R.tests[gi].status != GEVO_STATUS_COMPLETED)
                    continue;
                BufferMap& out = R.outputs[v][static_cast<size_t>(t)];
                for (int p = 0; p < S.n_params; ++p) {
                    const Param& prm = S.params[static_cast<size_t>(p)];
                    if (!(prm.type.is_ptr() && prm.type.space == MemSpace::Global))
                        continue;
                    const size_t tp = static_cast<size_t>(t) * S.n_params + p;
                    const int32_t n = S.buf_size[tp];
                    Buffer b;
                    b.elem = S.buf_elem[tp] == GEVO_TAG_I32 ? TypeKind::I32 : TypeKind::F32;
                    const bool mine = (vars[v].writable >> p) & 1ull;
                    for (int32_t e = 0; e < n; ++e) {
                        const uint32_t word =
                            mine ? win[((ow.off[static_cast<size_t>(p)] + static_cast<size_t>(e)) *
                                            ow.n_inst + gi) * wsz]
                                 : S.pool[S.pool_off[static_cast<size_t>(p)] +
                                          static_cast<size_t>(e) * S.n_tests + t];
                        if (b.elem == TypeKind::I32) {
                            int32_t x;
                            std::memcpy(&x, &word, 4);
                            b.i.push_back(x);
                        } else {
                            float x;
                            std::memcpy(&x, &word, 4);
                            b.f.push_back(x);
                        }
                    }
                    out[prm.name] = std::move(b);
                }
            }
    }
    return R;
}

struct ResidentBatch {
    DeviceSuite* suite;
    DevBuf blob;
    gevo_batch_header h;
    uint64_t writable;
    // concurrent evaluation: own stream, scratch and record staging
    cudaStream_t stream = nullptr;
    cudaEvent_t origin = nullptr, start = nullptr, done = nullptr;
    Scratch sc;
    PinnedBuf h_vrec, h_blob;
    int launches = 0;
    uint64_t h2d = 0; // bytes uploaded by the evaluation in flight
    bool pending = false;
    // the batch's host bytecode, page-locked in place so an uploading
    // evaluation DMAs it directly (no staging copy on the host)
    const void* reg = nullptr;
    size_t reg_size = 0;
    ~ResidentBatch() {
        // an evaluation still in flight reads the blob and writes the pinned
        // record buffer: let it finish before either is released
        if (pending && done)
            cudaEventSynchronize(done);
        if (reg)
            cudaHostUnregister(const_cast<void*>(reg));
        if (stream)
            cudaStreamDestroy(stream);
        if (origin)
            cudaEventDestroy(origin);
        if (start)
            cudaEventDestroy(start);
        if (done)
            cudaEventDestroy(done);
    }
};

std::shared_ptr<ResidentBatch> make_resident(DeviceSuite& suite, BatchImage& batch) {
    Device& devh = suite.device();
    std::lock_guard<std::mutex> g(devh.lock());
    check(cudaSetDevice(devh.ordinal()), "cudaSetDevice");
    auto rb = std::make_shared<ResidentBatch>();
    rb->suite = &suite;
    const auto& blob = batch.blob();
    rb->h = batch.header();
    rb->writable = writable_union(batch);
    rb->blob.reserve(blob.size() + 64);
    check(cudaMemcpy(rb->blob.ptr, blob.data(), blob.size(), cudaMemcpyHostToDevice), "resident");
    if (!blob.empty()) {
        if (cudaHostRegister(const_cast<uint8_t*>(blob.data()), blob.size(), cudaHostRegisterDefault) ==
            cudaSuccess) {
            rb->reg = blob.data();
            rb->reg_size = blob.size();
        } else {
            cudaGetLastError(); // not page-lockable here: uploads go through the staging copy
        }
    }
    return rb;
}

void evaluate_resident_async(ResidentBatch& rb, const ExecImage& exec, const EvalOptions& opt,
                             const std::vector<uint8_t>* upload) {
    Device& devh = rb.suite->device();
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    if (rb.pending)
        throw std::logic_error("resident batch already has an evaluation in flight");
    if (!rb.stream) {
        check(cudaStreamCreateWithFlags(&rb.stream, cudaStreamNonBlocking), "cudaStreamCreate");
        check(cudaEventCreateWithFlags(&rb.origin, cudaEventDisableTiming), "cudaEventCreate");
        check(cudaEventCreate(&rb.start), "cudaEventCreate");
        check(cudaEventCreate(&rb.done), "cudaEventCreate");
    }
    // ordered after the caller's stream (its CUDA events bracket the work)
    check(cudaEventRecord(rb.origin, dev.stream), "event");
    check(cudaStreamWaitEvent(rb.stream, rb.origin, 0), "stream wait");
    check(cudaEventRecord(rb.start, rb.stream), "event");
    rb.h2d = upload ? upload->size() : 0;
    if (upload) {
        // host bytecode of the batch, copied in this evaluation (end-to-end form)
        const void* src = upload->data();
        if (src != rb.reg || upload->size() != rb.reg_size) {
            rb.h_blob.reserve(upload->size());
            std::memcpy(rb.h_blob.ptr, upload->data(), upload->size());
            src = rb.h_blob.ptr;
        }
        check(cudaMemcpyAsync(rb.blob.ptr, src, upload->size(), cudaMemcpyHostToDevice, rb.stream),
              "blob H2D");
    }
    gevo::InterpArgs A = base_args(*rb.suite, exec, opt);
    bind_batch(A, rb.blob.ptr, rb.h);
    rb.launches = launch_all(dev, rb.sc, *rb.suite, A, rb.h, rb.writable, exec, opt, rb.stream);
    const size_t nb = rb.h.n_variants * sizeof(gevo_variant_record);
    rb.h_vrec.reserve(std::max<size_t>(nb, 16));
    if (nb)
        check(cudaMemcpyAsync(rb.h_vrec.ptr, rb.sc.vrec.ptr, nb, cudaMemcpyDeviceToHost, rb.stream),
              "records");
    check(cudaEventRecord(rb.done, rb.stream), "event");
    // (the caller's stream is ordered after `done` by wait_resident, not here:
    // a second batch launched now must not queue behind this one)
    rb.pending = true;
}

uint64_t resident_h2d(const ResidentBatch& rb) { return rb.h2d; }

bool resident_pending(const ResidentBatch& rb) { return rb.pending; }

float wait_resident(ResidentBatch& rb, std::vector<gevo_variant_record>* out, int* launches) {
    if (!rb.pending)
        throw std::logic_error("no evaluation in flight");
    check(cudaEventSynchronize(rb.done), "resident eval");
    {
        Device& devh = rb.suite->device();
        std::lock_guard<std::mutex> g(devh.lock());
        check(cudaStreamWaitEvent(devh.impl().stream, rb.done, 0), "stream wait");
    }
    rb.pending = false;
    float ms = 0;
    check(cudaEventElapsedTime(&ms, rb.start, rb.done), "elapsed");
    if (out) {
        out->resize(rb.h.n_variants);
        std::memcpy(out->data(), rb.h_vrec.ptr, rb.h.n_variants * sizeof(gevo_variant_record));
    }
    if (launches)
        *launches = rb.launches;
    return ms;
}

float evaluate_resident(ResidentBatch& rb, const ExecImage& exec, const EvalOptions& opt,
                        float* interp_ms, std::vector<gevo_variant_record>* out, int* launches) {
    Device& devh = rb.suite->device();
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    cudaStream_t s = dev.stream;
    gevo::InterpArgs A = base_args(*rb.suite, exec, opt);
    bind_batch(A, rb.blob.ptr, rb.h);
    check(cudaEventRecord(dev.ev0, s), "event");
    const int nl = launch_all(dev, dev.sc, *rb.suite, A, rb.h, rb.writable, exec, opt, s);
    if (launches)
        *launches = nl;
    check(cudaEventRecord(dev.ev2, s), "event");
    if (out) {
        out->resize(rb.h.n_variants);
        check(cudaMemcpyAsync(out->data(), dev.sc.vrec.ptr, rb.h.n_variants * sizeof(gevo_variant_record),
                              cudaMemcpyDeviceToHost, s),
              "records");
    }
    check(cudaStreamSynchronize(s), "resident eval");
    float ms = 0;
    check(cudaEventElapsedTime(&ms, dev.ev0, dev.ev2), "elapsed");
    if (interp_ms)
        *interp_ms = ms;
    return ms;
}

namespace {
void read_counters(Device& devh, uint64_t out[2], bool reset, size_t first) {
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    out[0] = out[1] = 0;
    if (!dev.counters.ptr)
        return;
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    uint64_t* c = dev.counters.as<uint64_t>() + first;
    check(cudaMemcpyAsync(out, c, 16, cudaMemcpyDeviceToHost, dev.stream), "counters");
    if (reset)
        check(cudaMemsetAsync(c, 0, 16, dev.stream), "counters");
    check(cudaStreamSynchronize(dev.stream), "counters");
}
} // namespace

void spin_counters(Device& devh, uint64_t out[2], bool reset) { read_counters(devh, out, reset, 0); }

void tp_counters(Device& devh, uint64_t out[2], bool reset) { read_counters(devh, out, reset, 2); }

void work_counters(Device& devh, uint64_t out[2], bool reset) { read_counters(devh, out, reset, 4); }

namespace {

// Uploads the fitness vectors and ranks them on the device; with keep >= 0 also
// computes select_best. Returns the number of fronts; fills `r` when given.
int32_t rank_impl(Device& devh, const std::vector<FitnessVector>& fits, bool single_group,
                  int64_t keep, ParetoRank* r, std::vector<int>* best, float* device_ms) {
    const int32_t n = static_cast<int32_t>(fits.size());
    if (r) {
        r->front.assign(fits.size(), -1);
        r->crowding.assign(fits.size(), 0.0);
        r->fronts.clear();
    }
    if (best)
        best->clear();
    if (n == 0)
        return 0;
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    cudaStream_t s = dev.stream;
    gevo::RankWorkspace& w = dev.rws;
    check(gevo::rank_reserve(w, n), "rank buffers");
    const size_t N = static_cast<size_t>(n);
    // one pinned H2D of the input span (cost, err) and one D2H of the output
    // span (crowd .. meta; select .. meta when only the selection is wanted),
    // laid out as the workspace carves them
    auto* base = reinterpret_cast<char*>(w.cost);
    const size_t err_at = reinterpret_cast<char*>(w.err) - base;
    const size_t in_bytes = err_at + N * 8;
    char* out0 = reinterpret_cast<char*>(r ? static_cast<void*>(w.crowd) : static_cast<void*>(w.select));
    const size_t out_bytes = reinterpret_cast<char*>(w.meta + gevo::kMetaCount) - out0;
    dev.h_rank.reserve(std::max(in_bytes, out_bytes));
    char* h = static_cast<char*>(dev.h_rank.ptr);
    auto* hc = reinterpret_cast<double*>(h);
    auto* he = reinterpret_cast<double*>(h + err_at);
    for (size_t i = 0; i < N; ++i) {
        hc[i] = fits[i].cost;
        he[i] = fits[i].error;
    }
    check(cudaMemcpyAsync(base, h, in_bytes, cudaMemcpyHostToDevice, s), "rank H2D");
    check(cudaEventRecord(dev.ev0, s), "event");
    check(gevo::launch_rank(w, n, single_group, static_cast<int32_t>(keep), s), "rank kernels");
    check(cudaEventRecord(dev.ev1, s), "event");
    check(cudaMemcpyAsync(h, out0, out_bytes, cudaMemcpyDeviceToHost, s), "rank D2H"); // (after the H2D)
    check(cudaStreamSynchronize(s), "rank");
    if (device_ms)
        check(cudaEventElapsedTime(device_ms, dev.ev0, dev.ev1), "elapsed");
    auto at = [&](const void* dptr) { return h + (reinterpret_cast<const char*>(dptr) - out0); };
    const auto* meta = reinterpret_cast<const int32_t*>(at(w.meta));
    const int32_t F = meta[gevo::kMetaFronts];
    if (best && keep > 0) {
        const auto* sel = reinterpret_cast<const int32_t*>(at(w.select));
        best->assign(sel, sel + keep);
    }
    if (r) {
        const auto* cr = reinterpret_cast<const double*>(at(w.crowd));
        const auto* front = reinterpret_cast<const int32_t*>(at(w.front));
        const auto* members = reinterpret_cast<const int32_t*>(at(w.members));
        const auto* offsets = reinterpret_cast<const int32_t*>(at(w.offsets));
        r->crowding.assign(cr, cr + N);
        r->front.assign(front, front + N);
        r->fronts.resize(static_cast<size_t>(F));
        for (int32_t f = 0; f < F; ++f)
            r->fronts[static_cast<size_t>(f)].assign(members + offsets[f], members + offsets[f + 1]);
    }
    return F;
}

} // namespace

ParetoRank rank_on_device(Device& devh, const std::vector<FitnessVector>& fits, bool single_group) {
    ParetoRank r;
    rank_impl(devh, fits, single_group, -1, &r, nullptr, nullptr);
    return r;
}

std::vector<int> select_on_device(Device& devh, const std::vector<FitnessVector>& fits, size_t keep,
                                  ParetoRank* rank, float* device_ms) {
    if (keep > fits.size())
        throw std::invalid_argument("select_best: keep exceeds the population");
    std::vector<int> best;
    rank_impl(devh, fits, false, static_cast<int64_t>(keep), rank, &best, device_ms);
    return best;
}


void nccl_unique_id(void* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    if (nccl_api().get_unique_id(&id) != ncclSuccess)
        throw std::runtime_error("ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
}

void set_nccl(int rank, int world, const void* id128) {
    Device& devh = Device::default_device();
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    if (dev.nccl) {
        nccl_api().comm_destroy(dev.nccl);
        dev.nccl = nullptr;
        dev.nccl_world = 0;
    }
    if (world <= 0)
        return;
    if (rank < 0 || rank >= world || !id128)
        throw std::invalid_argument("set_nccl: need 0 <= rank < world and a unique id");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (nccl_api().comm_init_rank(&dev.nccl, world, id, rank) != ncclSuccess) {
        dev.nccl = nullptr;
        throw std::runtime_error("ncclCommInitRank failed");
    }
    dev.nccl_rank = rank;
    dev.nccl_world = world;
}

int nccl_world() { return Device::default_device().impl().nccl_world; }
int nccl_rank() { return Device::default_device().impl().nccl_rank; }

size_t debug_cta_clock(Device& devh, uint64_t* out, size_t words) {
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    const CtaClockRef r = last_cta_clock();
    if (!r.buf || !r.buf->ptr)
        return 0;
    const size_t n = std::min(words, r.bytes / 8);
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    check(cudaStreamSynchronize(dev.stream), "cta clock");
    check(cudaDeviceSynchronize(), "cta clock");
    check(cudaMemcpy(out, r.buf->ptr, n * 8, cudaMemcpyDeviceToHost), "cta clock D2H");
    return n;
}

double error_on_device(Device& devh, const BufferMap& candidate, const BufferMap& oracle) {
    // Structural mismatches are decided on the host exactly like the suite
    // builder; the element-wise metric runs on the device.
    std::vector<uint32_t> cw, ow;
    std::vector<uint8_t> el;
    for (const auto& [name, want] : oracle) {
        const auto it = candidate.find(name);
        if (it == candidate.end() || it->second.elem != want.elem || it->second.size() != want.size())
            return 1.0;
        for (size_t e = 0; e < want.size(); ++e) {
            uint32_t c, o;
            if (want.elem == TypeKind::I32) {
                std::memcpy(&c, &it->second.i[e], 4);
                std::memcpy(&o, &want.i[e], 4);
            } else {
                std::memcpy(&c, &it->second.f[e], 4);
                std::memcpy(&o, &want.f[e], 4);
            }
            cw.push_back(c);
            ow.push_back(o);
            el.push_back(want.elem == TypeKind::I32 ? GEVO_TAG_I32 : GEVO_TAG_F32);
        }
    }
    if (cw.empty())
        return 0.0;
    std::lock_guard<std::mutex> g(devh.lock());
    DeviceImpl& dev = devh.impl();
    check(cudaSetDevice(dev.ordinal), "cudaSetDevice");
    cudaStream_t s = dev.stream;
    const size_t n = cw.size();
    dev.rank.reserve(n * 9 + 64);
    char* base = dev.rank.as<char>();
    uint32_t* dc = reinterpret_cast<uint32_t*>(base);
    uint32_t* dor = dc + n;
    double* dres = reinterpret_cast<double*>(base + ((8 * n + 15) & ~size_t(15)));
    uint8_t* de = reinterpret_cast<uint8_t*>(dres + 1);
    check(cudaMemcpyAsync(dc, cw.data(), n * 4, cudaMemcpyHostToDevice, s), "err H2D");
    check(cudaMemcpyAsync(dor, ow.data(), n * 4, cudaMemcpyHostToDevice, s), "err H2D");
    check(cudaMemcpyAsync(de, el.data(), n, cudaMemcpyHostToDevice, s), "err H2D");
    check(gevo::launch_error(dc, dor, de, static_cast<uint32_t>(n), dres, s), "error kernel");
    double res = 0.0;
    check(cudaMemcpyAsync(&res, dres, 8, cudaMemcpyDeviceToHost, s), "err D2H");
    check(cudaStreamSynchronize(s), "error");
    return res;
}

} // namespace evoir::b200
