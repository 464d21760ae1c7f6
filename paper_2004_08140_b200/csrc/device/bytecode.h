/* Device bytecode for a population of IR variants (plain C layout, shared by
 * the host encoder csrc/host/encode.cpp and the sm_100a interpreter
 * csrc/device/interp.cu).
 *
 * One batch = one contiguous blob: header, per-variant descriptors, block
 * table, fixed 16-byte instruction records, phi arms and literal pool. The
 * host pre-resolves everything the reference's Machine::compile does per
 * execution (src/vm.cpp:166-193 of arxiv/paper_2004_08140): branch and phi
 * labels become block indices, load/store costs become cost classes chosen by
 * the pointer operand's static type, value ids become dense value-file slots.
 *
 * Value-file slot space of a variant (per simulated lane):
 *   [0, n_values)                     SSA values of the running simulated thread
 *   [n_values, +n_params)             kernel parameters (bound per test)
 *   [.., +n_lits)                     literal pool (operands and const payloads)
 *   [.., +max_phis)                   phi staging (parallel-copy semantics)
 * Operand refs >= GEVO_REF_TRAP_BASE are poisoned operands that trap on fetch.
 */
#ifndef GEVO_BYTECODE_H
#define GEVO_BYTECODE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Opcodes: identical numbering to evoir::Opcode (include/evoir/ir.hpp). */
enum {
    GEVO_OP_ADD = 0, GEVO_OP_SUB, GEVO_OP_MUL, GEVO_OP_SDIV,
    GEVO_OP_FADD, GEVO_OP_FSUB, GEVO_OP_FMUL, GEVO_OP_FDIV,
    GEVO_OP_ICMP, GEVO_OP_FCMP,
    GEVO_OP_SELECT,
    GEVO_OP_LOAD, GEVO_OP_STORE, GEVO_OP_GETINDEX,
    GEVO_OP_PHI,
    GEVO_OP_BR, GEVO_OP_SYNC, GEVO_OP_RET,
    GEVO_OP_TID, GEVO_OP_NTHREADS,
    GEVO_OP_CONST,
    GEVO_OP_COUNT,
    /* device-only: sentinel record after every block ("fell off the end of a
       block", src/vm.cpp:345-346) */
    GEVO_OP_FELL = GEVO_OP_COUNT
};

/* Cost classes: index into the 14-entry cost table (field order of
 * evoir::CostTable, include/evoir/vm.hpp). */
enum {
    GEVO_COST_ARITH = 0, GEVO_COST_CMP, GEVO_COST_SELECT, GEVO_COST_PHI, GEVO_COST_CONST,
    GEVO_COST_BR, GEVO_COST_INTRINSIC, GEVO_COST_GETINDEX, GEVO_COST_LOAD_SHARED,
    GEVO_COST_STORE_SHARED, GEVO_COST_LOAD_GLOBAL, GEVO_COST_STORE_GLOBAL, GEVO_COST_SYNC,
    GEVO_COST_RET, GEVO_COST_CLASSES
};

/* Runtime value tags (one byte per value-file slot / shared word). */
enum {
    GEVO_TAG_UNDEF = 0,     /* also: uninitialised shared word */
    GEVO_TAG_I32 = 1,
    GEVO_TAG_F32 = 2,
    GEVO_TAG_BOOL = 3,
    GEVO_TAG_PTR_SHARED = 4,
    GEVO_TAG_PTR_GLOBAL = 0x40 /* | buffer (= parameter) index, < 64 */
};
/* Tag a load/select expects for a type that can never be held (Ptr loads). */
#define GEVO_TAG_NEVER 0xFE
/* Poisoned operand slots: fetching them traps (bad param index / missing operand). */
#define GEVO_TAG_POISON_PARAM 0x20
#define GEVO_TAG_POISON_MISSING 0x21

/* Trap / status codes. Codes 1..28 map 1:1 to the reference reason strings
 * (src/vm.cpp line numbers in comments). */
enum {
    GEVO_OK = 0,
    GEVO_TRAP_MISSING_BUFFER = 1,   /* vm.cpp:93  'missing buffer for param '<name>'' */
    GEVO_TRAP_BUFFER_TYPE = 2,      /* vm.cpp:95  */
    GEVO_TRAP_MISSING_SCALAR = 3,   /* vm.cpp:105 */
    GEVO_TRAP_SCALAR_TYPE = 4,      /* vm.cpp:107 */
    GEVO_TRAP_DIVERGENCE = 5,       /* vm.cpp:137 barrier divergence */
    GEVO_TRAP_BAD_PARAM = 6,        /* vm.cpp:201 */
    GEVO_TRAP_UNDEF_VALUE = 7,      /* vm.cpp:214,217 read of undefined value %<n> (aux = slot) */
    GEVO_TRAP_BAD_OPERAND = 8,      /* vm.cpp:221 */
    GEVO_TRAP_OPERAND_TYPE = 9,     /* vm.cpp:227 */
    GEVO_TRAP_NOT_POINTER = 10,     /* vm.cpp:234 */
    GEVO_TRAP_SHARED_OOB = 11,      /* vm.cpp:242,270 */
    GEVO_TRAP_SHARED_UNINIT = 12,   /* vm.cpp:245 */
    GEVO_TRAP_SHARED_TYPE = 13,     /* vm.cpp:247 */
    GEVO_TRAP_GLOBAL_OOB = 14,      /* vm.cpp:252,276 */
    GEVO_TRAP_GLOBAL_LOAD_TYPE = 15,/* vm.cpp:254 */
    GEVO_TRAP_STORE_BOOL = 16,      /* vm.cpp:266 */
    GEVO_TRAP_GLOBAL_STORE_TYPE = 17,/* vm.cpp:278 */
    GEVO_TRAP_DEF_NO_ID = 18,       /* vm.cpp:287 */
    GEVO_TRAP_PHI_NO_INCOMING = 19, /* vm.cpp:326 */
    GEVO_TRAP_FELL_OFF = 20,        /* vm.cpp:346 */
    GEVO_TRAP_UNKNOWN_BLOCK = 21,   /* vm.cpp:375 */
    GEVO_TRAP_PHI_OUTSIDE = 22,     /* vm.cpp:380 */
    GEVO_TRAP_DIV_ZERO = 23,        /* vm.cpp:402 */
    GEVO_TRAP_DIV_OVERFLOW = 24,    /* vm.cpp:404 */
    GEVO_TRAP_SELECT_ARM = 25,      /* vm.cpp:442 */
    GEVO_TRAP_STORE_NONSCALAR = 26, /* vm.cpp:457 */
    GEVO_TRAP_GETINDEX_SPACE = 27,  /* vm.cpp:464 */
    GEVO_TRAP_UNEXPECTED_OP = 28,   /* vm.cpp:480 */
    GEVO_BUDGET_EXCEEDED = 29,      /* vm.cpp:513 instruction budget exceeded */
    GEVO_TRAP_INTERNAL = 30,        /* encoder/device contract violation (never expected) */
    GEVO_SKIPPED = 31               /* not run: an earlier test of the variant already failed */
};

/* Execution status of one (variant, test) instance. */
enum { GEVO_STATUS_COMPLETED = 0, GEVO_STATUS_TRAP = 1, GEVO_STATUS_BUDGET = 2,
       GEVO_STATUS_SKIPPED = 3 };

#define GEVO_REF_TRAP_BASE 0xFFF0u
#define GEVO_REF_BAD_PARAM 0xFFF0u   /* Param operand with out-of-range index */
#define GEVO_REF_NEG_VALUE 0xFFF1u   /* Value operand with negative id (aux carries id) */
#define GEVO_NO_RESULT 0xFFFFu

#define GEVO_MAX_PARAMS 48
#define GEVO_MAX_SLOTS 1400

/* 16-byte instruction record, laid out for a cheap decode on the device:
 * word 0 = op | aux << 8 | otag << 16 | cls << 24, word 1 = a | b << 16,
 * word 2 = res | c << 16, word 3 = t0 | t1 << 16. */
typedef struct {
    uint8_t op;      /* GEVO_OP_* */
    uint8_t aux;     /* cmp: predicate (evoir::CmpPred); select / load: tag of the result kind;
                        getindex: 1 when inst.type is ptr<shared>; br: number of targets;
                        phi: number of arms */
    uint8_t otag;    /* arithmetic / compares: tag both operands must carry */
    uint8_t cls;     /* GEVO_COST_* */
    uint16_t a;      /* operand refs */
    uint16_t b;
    uint16_t res;    /* result slot or GEVO_NO_RESULT */
    uint16_t c;      /* select: false arm; store: value; phi with > 2 arms: arm offset */
    int16_t t0;      /* br targets (block index, -1 = unknown label); phi with <= 2 arms: */
    int16_t t1;      /* predecessor block of arm a / arm b */
} gevo_inst;

typedef struct {
    int16_t pred_block; /* incoming block index (-1 = unknown label: never matches) */
    uint16_t ref;       /* operand ref */
} gevo_arm;

/* Per-instruction edge record (parallel to the instruction array; used for br):
 * the leading phis of each target block resolved for this branch's block as
 * the predecessor (src/vm.cpp:311-323 picks the first arm whose label is the
 * predecessor). phi[e][j] = operand ref | result slot << 16 for edge e (0 =
 * first target, 1 = second) and phi j < 2; ref GEVO_EDGE_NOINC = no matching
 * arm. GEVO_EDGE_NONE in phi[e][0] = not pre-resolved (> 2 phis, a phi without
 * result id, unknown target): the interpreter matches arms itself. */
typedef struct {
    uint32_t phi[2][2];
} gevo_edge;

#define GEVO_EDGE_NOINC 0xFFFEu
#define GEVO_EDGE_NONE 0xFFFFFFFFu

typedef struct {
    uint32_t start;  /* instruction index relative to the variant's inst base */
    uint16_t len;
    uint16_t nphi;   /* number of leading phis */
} gevo_block;

typedef struct {
    uint32_t inst_base;   /* into the batch instruction array */
    uint32_t block_base;  /* into the batch block array */
    uint32_t arm_base;
    uint32_t lit_base;
    uint16_t n_values;    /* dynamic SSA slots */
    uint16_t n_lits;
    uint16_t n_blocks;
    uint16_t max_phis;
    uint64_t writable;    /* bit p: global parameter p may be stored to */
    uint32_t flags;       /* bit0: has sync */
    uint32_t n_slots;     /* n_values + n_params + n_lits + max_phis */
} gevo_variant;

#define GEVO_VAR_HAS_SYNC 1u

typedef struct {
    uint32_t magic;       /* 'GEVO' */
    uint32_t version;
    uint32_t n_variants;
    uint32_t n_params;
    uint32_t n_insts;
    uint32_t n_blocks;
    uint32_t n_arms;
    uint32_t n_lits;
    uint32_t max_slots;   /* max n_slots over variants */
    uint32_t max_values;
    uint32_t any_sync;
    uint32_t max_lits;    /* max n_lits over variants */
    uint32_t max_lane_slots; /* max n_values + max_phis over variants */
    uint32_t max_insts;   /* max instruction records of a variant (sentinels included) */
    /* byte offsets of each section from the start of the blob */
    uint64_t off_variants, off_blocks, off_insts, off_arms, off_lit_payload, off_lit_tag;
    uint64_t off_edges;
    uint64_t total_bytes;
} gevo_batch_header;

#define GEVO_MAGIC 0x4F564547u
#define GEVO_VERSION 5u

/* Per-(variant, test) record written by the interpreter. */
typedef struct {
    int64_t cost;    /* cycle cost under the launch's cost table */
    int64_t ir;      /* dynamic IR instructions executed (sum over simulated threads) */
    double error;    /* compute_error vs the oracle (completed only, else -1) */
    int32_t aux;     /* trap payload: slot / param index */
    uint8_t status;  /* GEVO_STATUS_* */
    uint8_t code;    /* GEVO_OK / GEVO_TRAP_* / GEVO_BUDGET_EXCEEDED / GEVO_SKIPPED */
    uint8_t pad[2];  /* pad[0]: spin-accelerator jumps taken (diagnostic) */
} gevo_test_record;

/* Per-variant EvalOutcome (evaluate_fitness, src/vm.cpp:558-579). */
typedef struct {
    double cost_mean;    /* valid when accepted */
    double error_max;    /* valid when accepted */
    double fail_error;   /* error of the failing test when rejected over tolerance */
    int64_t ir_ref;      /* dynamic IR of the tests the reference would run */
    int32_t failing_test;/* -1 when accepted */
    int32_t execs_ref;   /* tests the reference would run (all, or up to the first failing) */
    int32_t aux;         /* trap payload of the failing test */
    uint8_t accepted;
    uint8_t code;        /* trap code of the failing test, or 0xFF: error over tolerance */
    uint8_t pad[2];
} gevo_variant_record;

#define GEVO_FAIL_TOLERANCE 0xFFu

#ifdef __cplusplus
}
#endif

#endif
