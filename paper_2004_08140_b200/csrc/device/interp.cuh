// Launch arguments of the batched interpreter (device side of the boundary).
#pragma once

#include "bytecode.h"

#include <cstdint>

#include <cuda_runtime.h>

namespace gevo {

struct OracleEntryDev {
    int32_t param;
    int32_t size;
    uint64_t off;
    uint32_t elem;
    uint32_t pad;
};

struct InterpArgs {
    // batch (device copies of the blob sections)
    const gevo_variant* variants;
    const gevo_block* blocks;
    const gevo_inst* insts;
    const gevo_arm* arms;
    const uint32_t* lit_payload;
    const uint8_t* lit_tag;
    uint32_t n_variants;

    // suite
    int32_t n_tests;
    int32_t n_params;
    const uint8_t* param_tag;      // [test][param]
    const uint32_t* param_payload; // [test][param]
    const int32_t* buf_size;       // [test][param]
    const uint8_t* buf_elem;       // [test][param]
    const uint8_t* setup_code;     // [test]
    const int32_t* setup_aux;      // [test]
    const uint32_t* pool;          // inputs + oracles, [row][test] blocks
    const int32_t* entry_begin;    // [test + 1]
    const OracleEntryDev* entries;
    const uint8_t* static_err;     // [test]
    uint64_t pool_off[GEVO_MAX_PARAMS];

    // execution config
    int32_t threads;
    int32_t shared_words;
    int64_t budget;
    int64_t cost[GEVO_COST_CLASSES];
    double tolerance;

    // instances handled by this launch: [inst_begin, inst_begin + n_inst)
    uint64_t inst_begin;
    uint32_t n_inst;
    uint32_t max_slots; // value-file capacity per lane (dynamic smem sizing)

    // per-instance scratch (instance-interleaved: index = row * n_inst + local)
    uint32_t* priv;                 // private copies of writable global buffers
    uint64_t priv_off[GEVO_MAX_PARAMS];
    uint8_t* sh_tag;                // simulated shared words
    uint32_t* sh_val;
    // per-(simulated thread, instance) state, only when the batch has barriers
    int32_t* ts_pos;                // block << 16 | ip
    int32_t* ts_prev;
    int64_t* ts_exec;
    uint32_t* ts_stop;              // stop kind << 16 | barrier id
    uint32_t* ts_val;               // [thread][slot][inst]
    uint8_t* ts_tag;
    uint32_t ts_slots;              // max dynamic slots (batch max n_values)

    // outputs
    gevo_test_record* rec;          // [variant * n_tests + test]
    int32_t* first_fail;            // [variant] (early-exit mode)
    int32_t early_exit;
};

// Value-file capacity limits (dynamic shared memory, 227 KB per CTA).
constexpr uint32_t kMaxSlots128 = 350;
constexpr uint32_t kMaxSlots32 = 1400;

int interp_lanes(uint32_t max_slots);
cudaError_t launch_interp(const InterpArgs& A, cudaStream_t stream);
cudaError_t launch_error(const uint32_t* cand, const uint32_t* orc, const uint8_t* elem, uint32_t n,
                         double* out, cudaStream_t stream);
cudaError_t launch_fitness(const gevo_test_record* rec, uint32_t n_variants, int32_t n_tests,
                           double tolerance, gevo_variant_record* out, cudaStream_t stream);

} // namespace gevo
