// Host side of the device boundary: test-suite layout and variant encoding.
#pragma once

#include "../device/bytecode.h"
#include "evoir/vm.hpp"

#include <array>
#include <cstdint>
#include <string>
#include <vector>

namespace evoir::b200 {

// Test suite in device layout. Global buffers are stored test-interleaved
// ([element][test]) so the lanes of a warp, which run the same variant on
// consecutive tests with the same simulated thread id, load consecutive words.
struct SuiteImage {
    int n_tests = 0;
    int n_params = 0;
    std::vector<Param> params;
    std::vector<std::string> param_names;

    // [test][param]
    std::vector<uint8_t> param_tag;
    std::vector<uint32_t> param_payload;
    std::vector<int32_t> buf_size;
    std::vector<uint8_t> buf_elem; // GEVO_TAG_I32 / GEVO_TAG_F32
    // [param] offset (in 32-bit words) of the param's [max_size][n_tests] input block
    std::vector<uint64_t> pool_off;
    std::vector<int32_t> pool_rows; // max size over tests
    // [test] setup traps (Machine ctor, src/vm.cpp:83-112)
    std::vector<uint8_t> setup_code;
    std::vector<int32_t> setup_aux;
    // Oracle: entries grouped per test; each compares one global param against
    // one oracle block ([rows][n_tests]).
    struct OracleEntry {
        int32_t param;
        int32_t size;
        uint64_t off;
        uint8_t elem;
    };
    std::vector<OracleEntry> entries;
    std::vector<int32_t> entry_begin; // [n_tests + 1]
    std::vector<uint8_t> static_err;  // [test] 1: structural mismatch -> error 1.0
    std::vector<uint32_t> pool;       // inputs and oracles
};

SuiteImage build_suite(const std::vector<Param>& params, const std::vector<TestCase>& tests);

// Encoded population. `slot_value` maps each variant's value-file slots back
// to IR value ids so trap messages can be rebuilt on the host.
class BatchImage {
public:
    explicit BatchImage(const SuiteImage& suite);

    // Appends one variant; throws std::invalid_argument on an unsupported
    // shape (different parameter list than the suite, > GEVO_MAX_SLOTS slots).
    void add(const Kernel& k);
    // Moves every variant of `other` (same suite) to the end of this batch.
    // Lets a large batch be encoded in parallel parts and joined in order.
    void append(BatchImage&& other);
    size_t size() const { return variants_.size(); }

    // Contiguous blob in the bytecode.h layout.
    const std::vector<uint8_t>& blob();
    const gevo_batch_header& header();
    // The same bytes written straight to `dst` (header().total_bytes of them),
    // e.g. into a pinned staging buffer without the intermediate blob.
    void write_blob(uint8_t* dst);
    // Union of the variants' writable-parameter masks.
    uint64_t writable_union() const;
    // Capacity for `variants` variants of about `insts` records in all.
    void reserve(size_t variants, size_t insts);

    // Reference reason string for a trap record of variant v.
    std::string reason(size_t v, uint8_t code, int32_t aux) const;

    uint32_t max_slots() const { return max_slots_; }
    bool any_sync() const { return any_sync_; }
    uint32_t max_values() const { return max_values_; }

private:
    const SuiteImage& suite_;
    std::vector<gevo_variant> variants_;
    std::vector<gevo_block> blocks_;
    std::vector<gevo_inst> insts_;
    std::vector<gevo_edge> edges_; // parallel to insts_
    std::vector<gevo_arm> arms_;
    std::vector<uint32_t> lit_payload_;
    std::vector<uint8_t> lit_tag_;
    std::vector<std::vector<int32_t>> slot_value_; // per variant: slot -> value id
    std::vector<uint8_t> blob_; // (materialised on demand by blob())
    void layout();
    gevo_batch_header hdr_{};
    bool dirty_ = true;
    uint32_t max_slots_ = 0;
    uint32_t max_values_ = 0;
    uint32_t max_lits_ = 0;
    uint32_t max_lane_slots_ = 0;
    uint32_t max_insts_ = 0;
    bool any_sync_ = false;
};

// Reason strings shared by every path that reports a trap.
std::string reason_text(uint8_t code, const std::string& param_name, int32_t value_id);

// Launch-wide execution parameters (ExecConfig + cost table).
struct ExecImage {
    int32_t threads = 1;
    int32_t shared_words = 0;
    int64_t budget = 1000000;
    std::array<int64_t, GEVO_COST_CLASSES> cost{};
};
ExecImage exec_image(const ExecConfig& cfg);

} // namespace evoir::b200
