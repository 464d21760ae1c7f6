/* gevo_b200 — C ABI of the B200 GEVO fitness-evaluation engine.
 *
 * Plain C types only (no CUDA or torch types), status-code returns, no
 * exceptions across the boundary; gevo_last_error() holds the message of the
 * last failing call on the calling thread. Strings returned through `char**`
 * are heap-allocated and released with gevo_free().
 *
 * The reference (arxiv/paper_2004_08140, `proj/`) has no FFI: its hot path is
 * a set of C++ free functions in namespace evoir. Each entry point below
 * names the reference interface it replaces (file:line under
 * /root/reference/proj). The C++ interface itself is re-exposed unchanged by
 * include/evoir/ on top of the same library.
 */
#ifndef GEVO_B200_H
#define GEVO_B200_H

#include <stddef.h>
#include <stdint.h>

#include "../paper_2004_08140_b200/csrc/device/bytecode.h" /* records, trap codes */

#ifdef __cplusplus
extern "C" {
#endif

#define GEVO_ABI_VERSION 1

/* Status codes. */
#define GEVO_SUCCESS 0
#define GEVO_E_INVALID -1     /* bad argument / parse / validation input */
#define GEVO_E_NODEVICE -2    /* no CUDA device: there is no CPU path */
#define GEVO_E_CUDA -3        /* CUDA runtime failure */
#define GEVO_E_INIT -4        /* InitFailure (engine) */

/* ExecConfig (include/evoir/vm.hpp:56-67 of the reference); cost_table in
 * CostTable field order (vm.hpp:35-53). */
typedef struct {
    int32_t threads;
    int32_t shared_words;
    int64_t instruction_budget;
    int64_t cost_table[14];
} gevo_exec_config;

/* Evaluation flags. */
#define GEVO_EVAL_EARLY_EXIT 1u /* stop a variant's remaining tests after its first failure */
#define GEVO_EVAL_TESTS 2u      /* fill per-test records */
#define GEVO_EVAL_SEQUENTIAL 4u /* force the sequential-lane interpreter (one lane runs all
                                   simulated threads of an instance in id order) */
#define GEVO_EVAL_UPLOAD 8u     /* gevo_eval_resident_async: copy the batch's host bytecode
                                   to the device as part of this evaluation */

typedef struct {
    float device_ms;       /* CUDA-event time of the interpreter + reduction launches */
    uint64_t h2d_bytes;    /* bytes copied host -> device in this call */
    uint64_t d2h_bytes;    /* bytes copied device -> host in this call */
    int32_t launches;      /* kernels launched */
    int32_t pad;
} gevo_eval_stats;

typedef struct gevo_suite gevo_suite;
typedef struct gevo_batch gevo_batch;

int gevo_abi_version(void);
int gevo_device_count(void);
const char* gevo_last_error(void);
/* Launch all work of the default device on a caller-owned cudaStream_t
 * (passed as void*; NULL restores the library's own stream), so a caller's
 * CUDA events bracket the library's launches. No reference counterpart. */
int gevo_set_stream(void* stream);
/* Diagnostics of the exact spin accelerator on the default device since the
 * last reset: out2[0] = budget-bound loops jumped, out2[1] = instructions
 * skipped by those jumps (counted in the records as executed). */
int gevo_spin_counters(uint64_t* out2, int reset);
/* Multi-GPU search (one process per GPU): the engine shards
 * every candidate batch by variant across `world` ranks and exchanges the
 * 48-byte per-variant records with `fn`, which must all-gather `bytes` from
 * every rank into `recv` (world * bytes, rank order) -- an NCCL all-gather
 * over NVLink on a GPU box. world = 1 (the default) disables sharding. No
 * reference counterpart: the reference's parallel_for (src/engine.cpp:28-62)
 * is single-process. */
typedef void (*gevo_allgather_fn)(void* ctx, const void* send, size_t bytes, void* recv);
int gevo_set_collective(int rank, int world, gevo_allgather_fn fn, void* ctx);
/* In-library multi-GPU exchange (one process per GPU): the engine's record
 * all-gather runs as ncclAllGather on the device buffers of the evaluation
 * (NVLink / NVSwitch), no host staging. One rank calls gevo_nccl_unique_id
 * (128 bytes) and distributes it; every rank then calls gevo_set_nccl with
 * its rank and the world size (world <= 0 leaves the communicator). Takes
 * precedence over gevo_set_collective. Shards are contiguous and cut at equal
 * shares of the predicted cost (the parents' mean cost). No reference
 * counterpart (src/engine.cpp:28-62 is single-process). */
int gevo_nccl_unique_id(void* out128);
int gevo_set_nccl(int rank, int world, const void* id128);
/* Thread-parallel interpreter counters since the last reset: out2[0] =
 * instances re-executed in thread-id order after a same-phase cross-thread
 * read/write conflict, out2[1] = instances run by the thread-parallel kernel. */
int gevo_tp_counters(uint64_t* out2, int reset);
/* Interpreted instructions on the default device since the last reset:
 * out2[0] = IR instructions the interpreters executed (spin-accelerator jumps
 * excluded; discarded re-run attempts and aborted threads included), out2[1]
 * reserved. Device-executed work beside the records' reference-equivalent
 * counts. */
int gevo_work_counters(uint64_t* out2, int reset);
void gevo_free(void* p);
/* Diagnostic: with GEVO_CTA_CLOCK=1 in the environment, the per-CTA timing of
 * the last thread-parallel evaluation on the default device:
 * [variant][test] x {globaltimer start ns, end ns, SM id, device IR} for the
 * first test of each CTA (zeros elsewhere). No reference counterpart. */
int gevo_debug_cta_clock(uint64_t* out, size_t words, size_t* copied);

/* ---- test suites (uploaded once, resident in HBM) ------------------------
 * Replaces the per-call test handling of evoir::execute / evaluate_fitness
 * (src/vm.cpp:83-112, 558-579): parameter binding, setup traps and oracle
 * layout are resolved once per suite. */

/* Registry benchmark (src/corpus.cpp:410 load_benchmark) with
 * generate_tests(b, n_tests, seed) (src/corpus.cpp:496). */
int gevo_suite_from_benchmark(const char* bench, int n_tests, uint64_t seed, int device,
                              gevo_suite** out);
/* Arbitrary kernel + TestCase JSON documents (src/vm.cpp:647 testcase_from_json). */
int gevo_suite_from_json(const char* kernel_ir, const char* const* tests_json, int n_tests,
                         int device, gevo_suite** out);
void gevo_suite_free(gevo_suite* s);
int gevo_suite_n_tests(const gevo_suite* s);
/* ExecConfig::for_kernel of the suite kernel (vm.hpp:61-66). */
int gevo_suite_exec_config(const gevo_suite* s, gevo_exec_config* out);
/* The suite kernel, printed (src/parser.cpp:549 print_kernel). */
int gevo_suite_kernel_ir(const gevo_suite* s, char** ir);

/* ---- populations of variants ---------------------------------------------
 * Flattened device bytecode for a whole population (bytecode.h). */
int gevo_batch_create(gevo_suite* s, gevo_batch** out);
int gevo_batch_add_ir(gevo_batch* b, const char* kernel_ir);
/* Variant = apply_patch(suite kernel, patch) (src/genome.cpp:216-227). */
int gevo_batch_add_patch(gevo_batch* b, const char* patch_json);
int gevo_batch_size(const gevo_batch* b);
/* Packed bytecode blob (host memory, owned by the batch). */
int gevo_batch_blob(gevo_batch* b, const void** data, size_t* bytes);
void gevo_batch_free(gevo_batch* b);

/* ---- evaluation ----------------------------------------------------------
 * evaluate_fitness (src/vm.cpp:558-579) over every variant x test: host
 * bytecode is copied to the device, the interpreter runs population x test x
 * simulated-thread grids, records come back. out_tests (nullable) is
 * [variant][test] and requires GEVO_EVAL_TESTS. */
int gevo_eval(gevo_batch* b, const gevo_exec_config* cfg, double tolerance, uint32_t flags,
              gevo_variant_record* out_variants, gevo_test_record* out_tests,
              gevo_eval_stats* stats);
/* Upload the bytecode once; gevo_eval_resident then re-evaluates with inputs
 * already in HBM (no program transfer). out_variants may be NULL. */
int gevo_batch_make_resident(gevo_batch* b);
int gevo_eval_resident(gevo_batch* b, const gevo_exec_config* cfg, double tolerance,
                       uint32_t flags, gevo_variant_record* out_variants, gevo_eval_stats* stats);
/* Concurrent evaluation of resident batches: _async launches the batch on its
 * own stream (after the work already queued on the library's current stream,
 * which in turn waits for it) and returns; _wait blocks until it finishes and
 * returns its records and device time. Several batches in flight overlap on
 * the GPU (their launch tails run side by side). One evaluation in flight per
 * batch. No reference counterpart (the reference evaluates one kernel at a
 * time). */
int gevo_eval_resident_async(gevo_batch* b, const gevo_exec_config* cfg, double tolerance,
                             uint32_t flags);
int gevo_eval_resident_wait(gevo_batch* b, gevo_variant_record* out_variants,
                            gevo_eval_stats* stats);
/* Reference reason string of a record (ExecResult::trap_reason /
 * EvalOutcome::reason, src/vm.cpp:513-571). */
int gevo_reason(const gevo_batch* b, int variant, uint32_t code, int32_t aux, double fail_error,
                char** text);
/* Final global buffers of every completed (variant, test) instance as JSON
 * [[{name: {"type","hex"}} | null per test] per variant] (small batches;
 * ExecResult::outputs, vm.hpp:78-85). */
int gevo_eval_outputs_json(gevo_batch* b, const gevo_exec_config* cfg, char** outputs_json);

/* evoir::execute (src/vm.cpp:500-522) as a batch of one: TestCase JSON in
 * (reference format, or "hex" element strings for bit-exact data), JSON out:
 * {"status","reason","cost","outputs"}. */
int gevo_execute(const char* kernel_ir, const char* test_json, const gevo_exec_config* cfg,
                 char** result_json);
/* evoir::evaluate_fitness (src/vm.cpp:558-579) as a batch of one: JSON out
 * {"accepted","failing_test","reason","cost","error"}. */
int gevo_evaluate_fitness(const char* kernel_ir, const char* const* tests_json, int n_tests,
                          const gevo_exec_config* cfg, double tolerance, char** outcome_json);

/* ---- ranking -------------------------------------------------------------
 * rank_population (src/nsga.cpp:88-106) on the GPU. members/offsets give
 * the fronts in reference order: front f = members[offsets[f] .. offsets[f+1]). */
int gevo_rank(const double* cost, const double* error, int32_t n, int device, int32_t* front_out,
              double* crowding_out, int32_t* members_out, int32_t* offsets_out,
              int32_t* n_fronts_out);
/* crowding_distance of one set (src/nsga.cpp:48-86). */
int gevo_crowding(const double* cost, const double* error, int32_t n, int device,
                  double* crowding_out);
/* rank_population on the GPU, then the host selection rules:
 * select_best(rank, keep) (nsga.cpp:126-148) and k binary tournaments over
 * pop_size with Rng(tournament_seed) (nsga.cpp:108-124). */
int gevo_nsga_select(const double* cost, const double* error, int32_t n, int device,
                     int32_t keep, int32_t* best_out, uint64_t tournament_seed, int32_t k,
                     int32_t* tournament_out);

/* rank_population + select_best(rank, keep) (nsga.cpp:88-106, 126-148) in one
 * device pass: only the keep order crosses back. device_ms (nullable) = CUDA-
 * event time of the ranking kernels. */
int gevo_select_best(const double* cost, const double* error, int32_t n, int device, int32_t keep,
                     int32_t* best_out, float* device_ms);

/* ---- host-side API of the search (no device work) ------------------------ */
int gevo_kernel_canonical(const char* kernel_ir, char** printed);          /* parse + print */
int gevo_kernel_validate(const char* kernel_ir, char** rules_json);        /* validate() */
int gevo_kernel_is_valid(const char* kernel_ir, int32_t* valid);           /* is_valid() */
int gevo_apply_patch(const char* kernel_ir, const char* patch_json, char** printed,
                     int32_t* n_applied);                                   /* apply_patch */
/* random_mutation (src/operators.cpp:348) on `kernel_ir` with
 * Rng::stream(master, a, b, c); returns the edit as JSON ("null" for
 * NoCandidate) and the next u64 of the stream after the draw. */
int gevo_random_mutation(const char* kernel_ir, uint64_t master, uint64_t a, uint64_t b,
                         uint64_t c, char** edit_json, uint64_t* probe);
/* Seeded inputs of a benchmark without oracles (src/corpus.cpp:429-483). */
int gevo_benchmark_inputs(const char* bench, int count, uint64_t seed, char** tests_json);
int gevo_benchmark_names(char** names_json);
int gevo_benchmark_ir(const char* bench, char** ir);
/* Bench/sweep workload: n validated mutants of a registry benchmark, drawn
 * as seeded random walks of up to max_depth accepted-by-validate edits
 * (random_mutation + apply_edit + validate, src/operators.cpp:348,
 * src/genome.cpp:212, src/validate.cpp:324), one compact patch JSON per line.
 * No evaluation: the mix keeps trapping, spinning and over-tolerance
 * variants, as the search's candidate stream does. */
int gevo_sample_candidates(const char* bench, int n, uint64_t seed, int max_depth, char** patches);
/* The same for an arbitrary kernel (IR text). */
int gevo_sample_candidates_ir(const char* kernel_ir, int n, uint64_t seed, int max_depth,
                              char** patches);
/* Test suite of an arbitrary kernel from a generator spec document
 * (src/corpus.cpp generator_spec_from_json + generate_tests_for: seeded
 * inputs, oracle = the kernel's own outputs, computed on the device). */
int gevo_suite_from_spec(const char* kernel_ir, const char* gen_json, int n_tests, uint64_t seed,
                         int device, gevo_suite** out);
/* Seeded inputs of a generator spec without oracles (TestCase JSON array). */
int gevo_spec_inputs(const char* gen_json, int count, uint64_t seed, char** tests_json);
/* Train / held-out suite seeds (src/cli_app.cpp:193-201). */
uint64_t gevo_train_seed(uint64_t master);
uint64_t gevo_heldout_seed(uint64_t master);

/* ---- end-to-end search -----------------------------------------------------
 * `evoir run --bench <bench>` (src/cli_app.cpp:203-253): returns log.csv and
 * report.json text plus device-work counters. mode: "default" | "mo". */
typedef struct {
    int64_t candidates;
    int64_t executions;
    int64_t dynamic_ir;
    int64_t launches;
    int64_t batches;
    double device_ms;
    double host_gen_ms;
    double seconds;
} gevo_run_stats;

int gevo_run_search(const char* bench, uint64_t seed, int pop, int generations, const char* mode,
                    double tolerance, int train_tests, int heldout_tests, int jobs, char** log_csv,
                    char** report_json, gevo_run_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* GEVO_B200_H */
