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
    const gevo_edge* edges;        // [batch instruction] pre-resolved branch phis
    const uint32_t* lit_payload;
    const uint8_t* lit_tag;
    const uint4* dblocks;          // [batch block] {start, len | nphi << 16, cost (int64)}
    const int64_t* suffix;         // [batch instruction] cost of the rest of its block
    uint32_t n_variants;

    // suite
    int32_t n_tests;
    int32_t n_params;
    const uint8_t* param_tag;      // [test][param]
    const uint32_t* param_payload; // [test][param]
    const int32_t* buf_size;       // [test][param]
    const uint8_t* buf_elem;       // [test][param]
    const uint2* buf_info;         // [test][param] {size << 8 | elem, pool word of element 0}
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

    // variants handled by this launch: [v_begin, v_begin + n_var); instance
    // il = (v - v_begin) * n_tests + test indexes the per-launch scratch.
    uint32_t v_begin;
    uint32_t n_var;
    uint32_t n_inst;                // n_var * n_tests
    uint32_t max_slots;             // value-file capacity per lane
    uint32_t warps_per_variant;     // ceil(n_tests / 32)
    uint32_t row_lanes;             // lanes per value-file row (pow2, <= 32)
    uint32_t vf_global;             // value file in global scratch (too large for smem)
    uint2* vf;                      // global value file [inst][slot] when vf_global

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

    // spin accelerator scratch ([slot][inst]); null disables it
    uint32_t* sp_base;              // payload at the reference iterate
    uint8_t* sp_btag;
    uint32_t* sp_delta;             // per-iteration stride hypothesis
    uint32_t* sp_cur;               // stride of the running abstract iterate
    uint8_t* sp_hvary;              // hypothesis: slot may vary (path-irrelevant)
    uint8_t* sp_cvary;              // abstract iterate: slot value is varying
    uint32_t* sp_log;               // [kSpinLog][col] x 5: store-log key, old payload,
                                    // old tag | flags, last stored payload, last stored tag
    uint32_t* sp_ld;                // [kSpinLog][inst] load-log keys
    uint32_t* sp_vk;                // [kSpinLog][col] memory words loaded as varying
    int64_t spin_threshold;         // per-thread executed count that arms it
    uint32_t spin_pay;              // a partial jump must skip >= spin_pay * n_values
                                    // instructions to re-arm at once (else: backoff)
    uint32_t n_spin;                // spin scratch columns (instances, or lanes for tp)

    // thread-parallel lanes (interp_tp_kernel)
    uint32_t tp_lanes;              // tests per CTA (thread-parallel kernel)
    uint32_t lane_slots;            // per-lane value-file slots: max n_values + max_phis
    uint32_t max_lits;              // max literals of a variant (CTA-shared table)
    uint2* gcells;                  // [cell][instance] global instance memory (null: on chip)
    unsigned long long* gshadow;    // [cell][instance] same-phase access records
    uint2* out_cells;               // [cell][instance] final memory of completed instances
                                    // (want_outputs, on-chip cells; null otherwise)
    uint2* tp_snap;                 // [value slot][lane] phase-start value files (multi-phase
                                    // batches; null: conflicts re-run from the initial state)
    uint32_t n_cells;               // memory cells per instance: shared words + writable rows
    uint32_t n_chunks;              // 32-bit chunks of a per-lane read / write bitset
    uint32_t cell_off[GEVO_MAX_PARAMS]; // first cell of writable global param p

    // outputs
    gevo_test_record* rec;          // [variant * n_tests + test]
    int32_t* first_fail;            // [variant] (early-exit mode)
    int32_t early_exit;
    uint64_t* counters;             // [6]: accelerated spins, jumped instructions,
                                    // tp instances re-run in id order, tp instances,
                                    // interpreted instructions, reserved (nullable)
    // thread-parallel per-CTA scratch regions: a CTA takes a free region of
    // the global cells / access records / spin and snapshot columns when it
    // starts and returns it when it ends, so scratch is sized by the CTAs
    // that can be resident, not by the batch (0: one column set per instance)
    uint32_t regions;
    uint32_t* region_q;             // [regions] free-region ring: region | generation << 16
    uint32_t* region_ctr;           // [2] acquire / release tickets
    uint32_t reconv;                // run_thread reconvergence gate (lanes of one test)
    // instruction / edge records of the CTA's variant staged in shared memory
    // by a TMA bulk copy (cp.async.bulk) at CTA start: records per CTA (the
    // batch's max_insts), 0 = fetched from global memory (__ldg)
    uint32_t stage_recs;
    uint32_t n_insts_total;         // batch instruction records (variant extents)
    // persistent thread-parallel launch (global cells): `regions` CTAs, CTA r
    // owns region r and takes work items (variant, test group) from a queue
    // in test-major order; with early exit an item whose variant's earlier
    // test groups are still running is deferred, and runs speculatively only
    // when nothing else is left (no speculative work while the GPU is full)
    uint32_t persist;
    uint32_t n_items;               // n_var * test groups
    uint32_t* sched;                // [4]: next static item, deferred count, spare
    uint32_t* defer;                // [n_items] deferred item ids (0xFFFFFFFF: not written yet)
    uint32_t* claim;                // [n_items] claim flag per deferred entry
    uint32_t* vdone;                // [n_var] finished test groups per launch-local variant
    unsigned long long* cta_clock;  // diagnostic (nullable): [variant][test] x 4 for the first
                                    // test of each thread-parallel CTA: globaltimer at CTA
                                    // start and end, SM id, device IR of the CTA
};

// Memory words one abstract iterate may store to / load from.
constexpr uint32_t kSpinLog = 8;

// Value slots a variant may use (value file in shared memory or global scratch).
constexpr uint32_t kMaxSlots = GEVO_MAX_SLOTS;

// Largest CTA of the thread-parallel interpreter.
#ifndef GEVO_TP_MAX_BLOCK
#define GEVO_TP_MAX_BLOCK 512
#endif
constexpr uint32_t kTpMaxBlock = GEVO_TP_MAX_BLOCK;

// Shared memory available to the value file of one CTA.
constexpr size_t kSmemBudget = 200 * 1024;

struct LaunchShape {
    uint32_t row_lanes;
    uint32_t warps_per_cta;
    size_t smem;
    bool vf_global;
};
LaunchShape interp_shape(int32_t n_tests, uint32_t max_slots);

// Builds the per-launch block records (block table + cost under the launch's
// cost table) that the interpreter reads with one 16-byte load per block entry.
cudaError_t launch_block_cost(const gevo_block* blocks, const gevo_inst* insts,
                              const gevo_variant* variants, uint32_t n_variants,
                              const int64_t* cost_table, uint4* out, int64_t* suffix,
                              cudaStream_t stream);
cudaError_t launch_interp(const InterpArgs& A, cudaStream_t stream);

// Thread-parallel launch shape: warps per CTA and dynamic shared memory, or
// warps_per_cta == 0 when the instance state does not fit on chip.
struct TpShape {
    uint32_t warps_per_cta;
    uint32_t lanes;         // tests per CTA (<= 32); 32 / lanes simulated threads per warp
    size_t smem;
};
struct TpTables {
    uint32_t lane_slots;    // max over variants of n_values + max_phis
    uint32_t max_slots;     // max over variants of every value-file slot
    uint32_t n_params;
    uint32_t max_lits;
    uint32_t stage_recs;    // staged instruction + edge records per CTA (0: none)
};
TpShape tp_shape(uint32_t threads, uint32_t n_tests, const TpTables& tab, uint32_t n_cells,
                 uint32_t n_chunks, bool backup, bool gc = false);
cudaError_t launch_interp_tp(const InterpArgs& A, cudaStream_t stream);
// CTAs of the thread-parallel kernel that can be resident at once for shape
// (warps, smem) on this device (the region count of a launch).
uint32_t tp_resident_ctas(bool global_cells, uint32_t warps_per_cta, size_t smem);
cudaError_t launch_error(const uint32_t* cand, const uint32_t* orc, const uint8_t* elem, uint32_t n,
                         double* out, cudaStream_t stream);
cudaError_t launch_fitness(const gevo_test_record* rec, uint32_t n_variants, int32_t n_tests,
                           double tolerance, gevo_variant_record* out, cudaStream_t stream);

} // namespace gevo
