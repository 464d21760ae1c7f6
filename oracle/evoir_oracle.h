/* Plain-C restatement of the reference fitness path. TEST INFRASTRUCTURE ONLY.
 *
 * This is the checker the parity tests and smoke() compare the sm_100a
 * interpreter against; the product never links or calls it. It restates, in
 * C99 and from scratch, the semantics of arxiv/paper_2004_08140:
 *   - execute / Machine          src/vm.cpp:83-522
 *   - compute_error              src/vm.cpp:524-556
 *   - evaluate_fitness           src/vm.cpp:558-579
 *   - rank_population (NSGA-II)  src/nsga.cpp:9-106 (O(n^2) peel, as written)
 *   - select_best                src/nsga.cpp:126-148
 * over kernels in the canonical printed IR form (src/parser.cpp:549-624).
 *
 * Pinned against the compiled reference's golden vectors in tests/golden/
 * (tests/test_oracle.py): every vmcase, corpus suite, 1.2k+ mutant executions
 * and 300 NSGA instances are bit-identical.
 */
#ifndef EVOIR_ORACLE_H
#define EVOIR_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct eo_kernel eo_kernel;

/* elem: 0 = i32, 1 = f32 (evoir::TypeKind). */
typedef struct {
    const char* name;
    int32_t elem;
    int32_t n;
    const uint32_t* words;
} eo_buffer;

typedef struct {
    const char* name;
    int32_t kind; /* 0 i32, 1 f32, 2 bool */
    uint32_t bits;
} eo_scalar;

typedef struct {
    int32_t n_inputs;
    const eo_buffer* inputs;
    int32_t n_scalars;
    const eo_scalar* scalars;
    int32_t n_oracle;
    const eo_buffer* oracle;
} eo_test;

typedef struct {
    int32_t threads;
    int32_t shared_words;
    int64_t budget;
    int64_t cost[14];
} eo_config;

/* status: 0 completed, 1 trap, 2 budget exceeded. Outputs are written into
 * `out_words` (capacity `out_cap` words) as the concatenation of every global
 * parameter's final buffer in output-map (name) order; out_offsets/out_elems
 * describe each one (capacity: parameter count). */
typedef struct {
    int32_t status;
    int64_t cost;
    int64_t ir;
    double error;
    char reason[160];
    int32_t n_outputs;
} eo_result;

eo_kernel* eo_parse(const char* text, char* err, size_t errcap);
void eo_free(eo_kernel* k);
int32_t eo_param_count(const eo_kernel* k);

int eo_execute(const eo_kernel* k, const eo_test* t, const eo_config* cfg, eo_result* out,
               uint32_t* out_words, size_t out_cap, int32_t* out_offsets, int32_t* out_sizes,
               int32_t* out_elems, const char** out_names);

/* evaluate_fitness: returns accepted; fills failing test / reason / fitness. */
int eo_evaluate_fitness(const eo_kernel* k, const eo_test* tests, int32_t n_tests,
                        const eo_config* cfg, double tolerance, int32_t* failing_test,
                        char* reason, size_t reason_cap, double* cost, double* error,
                        int64_t* ir_ref, int32_t* execs_ref);

/* rank_population: front index + crowding per individual, fronts as
 * members[offsets[f] .. offsets[f+1]). Returns the number of fronts. */
int32_t eo_rank(const double* cost, const double* error, int32_t n, int32_t* front,
                double* crowding, int32_t* members, int32_t* offsets);
void eo_select_best(const double* cost, const double* error, int32_t n, int32_t keep,
                    int32_t* out);

#ifdef __cplusplus
}
#endif

#endif
