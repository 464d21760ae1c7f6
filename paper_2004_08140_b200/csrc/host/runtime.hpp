// Device runtime: context (device + stream + reusable buffers), test suites
// resident in HBM, batch evaluation and GPU ranking. Host code only sees
// plain records; CUDA types stay behind this header.
#pragma once

#include "encode.hpp"
#include "evoir/nsga.hpp"

#include <memory>
#include <mutex>
#include <vector>

namespace evoir::b200 {

struct DeviceImpl;
struct SuiteImpl;

class Device {
public:
    // Throws DeviceUnavailable when CUDA has no device.
    explicit Device(int ordinal = -1);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    int ordinal() const;
    // Launch on a caller-owned stream (nullptr: back to the device's own).
    void set_stream(void* stream);
    DeviceImpl& impl() { return *impl_; }
    std::mutex& lock() { return mu_; }

    // Process-wide default device (GEVO_DEVICE env or the current CUDA device).
    static Device& default_device();

private:
    std::unique_ptr<DeviceImpl> impl_;
    std::mutex mu_;
};

// A test suite uploaded to one device (inputs, oracles, binding tables).
class DeviceSuite {
public:
    DeviceSuite(Device& dev, SuiteImage image);
    ~DeviceSuite();
    const SuiteImage& image() const { return image_; }
    SuiteImpl& impl() { return *impl_; }
    Device& device() { return dev_; }

private:
    Device& dev_;
    SuiteImage image_;
    std::unique_ptr<SuiteImpl> impl_;
};

struct EvalOptions {
    double tolerance = 0.0;
    bool early_exit = false;      // skip tests after a variant's first failure
    bool want_tests = false;      // copy per-test records back
    bool want_outputs = false;    // copy final global buffers back (small batches)
    bool sequential = false;      // force the sequential-lane interpreter
    // Multi-GPU exchange inside the evaluation: with an NCCL communicator on
    // the device (set_nccl) and gather_count > 0, the batch is this rank's
    // shard and its variant records (padded to gather_count) are all-gathered
    // on the device by ncclAllGather; EvalResult::variants then holds
    // world * gather_count records in rank order.
    size_t gather_count = 0;
};

struct EvalResult {
    std::vector<gevo_variant_record> variants;
    std::vector<gevo_test_record> tests;          // [variant * n_tests + test] when requested
    std::vector<std::vector<BufferMap>> outputs;  // [variant][test] when requested
    float kernel_ms = 0.0f;                       // interpreter + reduction, CUDA events
    uint64_t h2d_bytes = 0;
    uint64_t d2h_bytes = 0;
    int launches = 0;
};

// Evaluates every variant of `batch` on every test of `suite`.
EvalResult evaluate(DeviceSuite& suite, BatchImage& batch, const ExecImage& exec,
                    const EvalOptions& opt);

// Device-resident variant for benchmarks: the blob is uploaded once and
// re-evaluated without host transfers of programs.
struct ResidentBatch;
std::shared_ptr<ResidentBatch> make_resident(DeviceSuite& suite, BatchImage& batch);
// Runs the interpreter + reduction on a resident batch; returns kernel ms
// (CUDA events on the launch stream) and fills `interp_ms` with the share of
// the interpreter kernel alone.
// Concurrent form: launches on the batch's own stream (ordered after the work
// queued on the device's current stream) and returns; wait_resident blocks,
// orders the current stream after the batch and returns its device ms.
// Batches evaluated this way overlap on the GPU.
// `upload` (nullable): the batch's host bytecode, copied H2D as part of the
// evaluation (the blob must be the one the batch was made resident with).
void evaluate_resident_async(ResidentBatch& rb, const ExecImage& exec, const EvalOptions& opt,
                             const std::vector<uint8_t>* upload = nullptr);
float wait_resident(ResidentBatch& rb, std::vector<gevo_variant_record>* out, int* launches);
uint64_t resident_h2d(const ResidentBatch& rb);
bool resident_pending(const ResidentBatch& rb);
float evaluate_resident(ResidentBatch& rb, const ExecImage& exec, const EvalOptions& opt,
                        float* interp_ms, std::vector<gevo_variant_record>* out,
                        int* launches = nullptr);

// Spin-accelerator counters of a device: {loops jumped, instructions skipped}.
void spin_counters(Device& dev, uint64_t out[2], bool reset);
// Thread-parallel interpreter counters: {instances re-run in thread-id order
// after a same-phase cross-thread conflict, instances run}.
void tp_counters(Device& dev, uint64_t out[2], bool reset);
// {instructions the interpreters executed (spin-accelerator jumps excluded,
// work of discarded attempts and aborted threads included), 0}.
void work_counters(Device& dev, uint64_t out[2], bool reset);

// Multi-GPU exchange: one process per GPU; the engine shards
// each candidate batch across the ranks by variant and all-gathers the
// fixed-size per-variant records. `allgather` receives `bytes` from every
// rank into `recv` in rank order (NCCL over NVLink on a GPU box, gloo in CPU
// tests); the host work around it is replicated, so every rank keeps an
// identical search state.
struct Collective {
    int rank = 0;
    int world = 1;
    void (*allgather)(void* ctx, const void* send, size_t bytes, void* recv) = nullptr;
    void* ctx = nullptr;
};
void set_collective(const Collective& c);
const Collective& collective();

// NCCL communicator of the default device for the in-library record
// exchange (one process per GPU). nccl_unique_id fills 128 bytes on one
// rank, which the caller distributes; set_nccl(rank, world, id) joins the
// communicator (world <= 0 releases it). nccl_world() is 0 without one.
void nccl_unique_id(void* out128);
void set_nccl(int rank, int world, const void* id128);
int nccl_world();
int nccl_rank();

// GPU NSGA ranking (front + crowding + fronts in reference order).
ParetoRank rank_on_device(Device& dev, const std::vector<FitnessVector>& fits, bool single_group);
// rank_population + select_best(rank, keep) in one device pass (only the keep
// order comes back unless `rank` is given); device_ms = CUDA-event time of the
// ranking kernels.
std::vector<int> select_on_device(Device& dev, const std::vector<FitnessVector>& fits, size_t keep,
                                  ParetoRank* rank = nullptr, float* device_ms = nullptr);

// Diagnostic: per-CTA timing of the last thread-parallel evaluation with
// GEVO_CTA_CLOCK=1 ([variant][test] x {start ns, end ns, SM, device IR});
// returns the words copied.
size_t debug_cta_clock(Device& dev, uint64_t* out, size_t words);

// compute_error of two host buffer maps, evaluated by the device metric.
double error_on_device(Device& dev, const BufferMap& candidate, const BufferMap& oracle);

} // namespace evoir::b200
