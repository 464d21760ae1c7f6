// Batched sm_100a interpreter for the evoir SSA IR.
//
// Mapping. One warp runs ONE variant: lane t executes test t (tests > 32 use
// several warps of the same variant), so the warp fetches the same 16-byte
// instruction (broadcast load), takes the same dispatch branch, reads and
// writes the same value-file row ([slot][lane] in shared memory, 8-byte
// {payload, tag} entries, conflict-free) and loads consecutive words of the
// test-interleaved input pool (coalesced). Different variants never share a
// warp, so control flow diverges only on data-dependent branches.
//
// Semantics. Inside a lane the simulated threads run exactly as the
// reference's Machine::run (src/vm.cpp:114-150 of arxiv/paper_2004_08140): one
// at a time in id order up to the next barrier or ret, then the
// barrier-divergence check. Per-instruction semantics follow run_to_barrier /
// enter_block / step (src/vm.cpp:293-482): cost and budget are charged before
// any effect, phis read all arms before writing (parallel copy), traps carry
// the reference's reason codes. Floating point is IEEE binary32
// round-to-nearest with no FMA contraction (__f*_rn, -fmad=false); the error
// metric is IEEE double.
//
// Accounting. Cost, dynamic-IR and the per-thread budget counter are charged
// a whole block at a time on entry (block costs are precomputed per launch by
// block_cost_kernel); leaving a block early (trap, sync, ret, a mid-block
// branch) refunds the instructions that did not run. A block that could
// cross the budget runs in exact per-instruction mode, so the budget trap
// fires on the same instruction as in the reference.
//
// Spin accelerator (exact). A simulated thread that passes
// `spin_threshold` executed instructions is probably spinning in a mutated
// loop until the 10^6-instruction budget (hard part 2). At a
// loop anchor block the lane snapshots the value file twice (S0, S1) and
// hypothesises that every I32/pointer slot moves by a constant stride per
// iteration and everything else is fixed. It then executes one more iteration
// while tracking strides through each instruction (add/sub/getindex add
// strides, mul by a constant scales them, compares must provably keep their
// outcome over every remaining iteration, loads/stores need fixed addresses
// and stores must not change memory, float/div/select-condition operands
// must be fixed). If the iterate S2 = S1 + stride and the tracked strides
// equal the hypothesis, the state sequence is affine with a fixed path until
// the budget runs out, so the lane jumps n whole iterations (values += n *
// stride, counters += n * per-iteration counts) and resumes exact
// interpretation, which then hits the budget trap on the reference's
// instruction. Any failed check just continues plain interpretation.
#include "interp.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>

namespace gevo {

extern __shared__ __align__(16) uint2 g_vfs[]; // value files of the CTA's warps

namespace {

constexpr int kStopRet = 1, kStopSync = 2, kStopTrap = 3, kStopAbort = 4, kStopIdle = 0;
constexpr int kStopNone = -1; // run_unit: the thread continues
// Fewest iterations a spin-accelerator jump may cover.
constexpr int64_t kSpinMinJump = 4;
// Failed spin-accelerator attempts after which a thread stops trying.
#ifndef GEVO_SPIN_ATTEMPTS
#define GEVO_SPIN_ATTEMPTS 20
#endif
constexpr uint32_t kSpinAttempts = GEVO_SPIN_ATTEMPTS;
// After a partial jump: periods of the jumped loop to wait for its anchor
// block to come round again before anchoring elsewhere.
#ifndef GEVO_PREFER_WINDOW
#define GEVO_PREFER_WINDOW 4
#endif
constexpr int64_t kPreferWindow = GEVO_PREFER_WINDOW;
// ts_stop encodings (multi-phase kernels)
constexpr uint32_t kTsFresh = 0, kTsResume = 3u << 16; // never run / resume after barrier
constexpr uint32_t kTsRet = 1u << 16, kTsSync = 2u << 16;

// Instance memory cell meta word (high half of a cell): value tag in bits
// 0..5 (cells hold only undef / i32 / f32), writer thread id + 1 in bits
// 6..15 (simulated threads <= kTpMaxBlock = 512 < 1023), phase epoch in bits
// 16..31 (an instance restarts in id order before the epoch wraps).
constexpr uint32_t kCellTag = 0x3Fu, kCellWriterShift = 6, kCellWriterMask = 0x3FFu;
__device__ __forceinline__ uint32_t cell_meta(uint32_t tag, uint32_t writer, uint32_t epoch) {
    return tag | (writer << kCellWriterShift) | (epoch << 16);
}
__device__ __forceinline__ uint32_t cell_writer(uint32_t meta) {
    return (meta >> kCellWriterShift) & kCellWriterMask;
}

// Field accessors of the 16-byte record (bytecode.h).
__device__ __forceinline__ uint32_t f_op(const uint4& r) { return r.x & 0xFF; }
__device__ __forceinline__ uint32_t f_aux(const uint4& r) { return (r.x >> 8) & 0xFF; }
__device__ __forceinline__ uint32_t f_otag(const uint4& r) { return (r.x >> 16) & 0xFF; }
__device__ __forceinline__ uint32_t f_cls(const uint4& r) { return r.x >> 24; }
__device__ __forceinline__ uint32_t f_a(const uint4& r) { return r.y & 0xFFFF; }
__device__ __forceinline__ uint32_t f_b(const uint4& r) { return r.y >> 16; }
__device__ __forceinline__ uint32_t f_res(const uint4& r) { return r.z & 0xFFFF; }
__device__ __forceinline__ uint32_t f_c(const uint4& r) { return r.z >> 16; }
__device__ __forceinline__ int32_t f_t0(const uint4& r) { return static_cast<int16_t>(r.w & 0xFFFF); }
__device__ __forceinline__ int32_t f_t1(const uint4& r) { return static_cast<int16_t>(r.w >> 16); }

__device__ __forceinline__ uint4 fetch_inst(const gevo_inst* code, uint32_t idx) {
    return __ldg(reinterpret_cast<const uint4*>(code) + idx);
}

__device__ __forceinline__ bool is_ptr_tag(uint32_t t) {
    return t == GEVO_TAG_PTR_SHARED || t >= GEVO_TAG_PTR_GLOBAL;
}

template <typename T>
__device__ __forceinline__ bool cmp(T x, T y, uint32_t pred) {
    switch (pred) {
    case 0: return x == y;
    case 1: return x != y;
    case 2: return x < y;
    case 3: return x <= y;
    case 4: return x > y;
    default: return x >= y;
    }
}

// Relative difference exactly as src/vm.cpp:526-532 (std::max / std::min
// argument order preserved for NaN behaviour), in IEEE double.
__device__ __forceinline__ double rel_diff(double c, double o) {
    const double ao = fabs(o);
    const double denom = (ao < 1e-6) ? 1e-6 : ao;
    const double d = __ddiv_rn(fabs(__dsub_rn(c, o)), denom);
    if (!isfinite(d))
        return 1.0;
    return (1.0 < d) ? 1.0 : d;
}

__device__ __forceinline__ double word_to_double(uint32_t w, uint32_t elem) {
    return elem == GEVO_TAG_I32 ? static_cast<double>(static_cast<int32_t>(w))
                                : static_cast<double>(__uint_as_float(w));
}

// Undefined / poisoned slot: every tag a slot can hold is 0 (undef), 1..4
// (i32 f32 bool ptr<shared>), 0x20 / 0x21 (poison) or 0x40 | param (ptr<global>).
__device__ __forceinline__ bool bad_tag(uint32_t t) {
    return (t - 1u > 3u) && (t < static_cast<uint32_t>(GEVO_TAG_PTR_GLOBAL));
}

// Branch-free select (the compiler may not re-branch an asm selp).
__device__ __forceinline__ uint32_t selp(bool p, uint32_t a, uint32_t b) {
    uint32_t r;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
        : "=r"(r) : "r"(a), "r"(b), "r"(static_cast<uint32_t>(p)));
    return r;
}

// Thread-parallel value files: CTA-shared parameter / literal tables (less
// shared memory per lane, one more address decision per operand) or every
// slot in the lane's own file.
#ifdef GEVO_TP_TABLES
constexpr bool kTpTables = true;
#else
constexpr bool kTpTables = false;
#endif

// Explicit shared-memory accesses by 32-bit shared-window address: the
// interpreter's value files and instance memory never go through generic
// pointers (no per-access window conversion).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint2 lds2(uint32_t a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts2(uint32_t a, uint32_t x, uint32_t y) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ uint4 lds4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t ldsb(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void stsb(uint32_t a, uint32_t x) {
    asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(x) : "memory");
}
// A value the compiler must keep rather than recompute.
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
    uint32_t y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t lds1(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts1(uint32_t a, uint32_t x) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(x) : "memory");
}
__device__ __forceinline__ unsigned long long cas64(uint32_t a, unsigned long long cmp,
                                                    unsigned long long val) {
    unsigned long long old;
    asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "r"(a), "l"(cmp), "l"(val)
                 : "memory");
    return old;
}
__device__ __forceinline__ unsigned long long lds64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

// Value file of one lane: slot s lives at shared address vsh + s * vstr
// (kM >= 1) or at index base + s * row of the global scratch array (kM == 0).
// kM: 0 = sequential lanes, value file in global scratch; 1 = sequential
// lanes, value file in shared memory; 2 = thread-parallel (one warp per
// simulated thread, instance memory in shared-memory cells, interp_tp_kernel).
// Global-cell thread-parallel lanes (256-thread data-parallel kernels) keep a
// compact value file -- 4-byte payloads and 1-byte tags in separate arrays --
// so two 256-thread CTAs fit one SM's shared memory.
#ifndef GEVO_GC_WIDE_VF
constexpr bool kGcCompactVF = true;
#else
constexpr bool kGcCompactVF = false;
#endif

// Record pointers of the global-cell lanes (empty for the other modes, so
// their lanes carry no unused fields).
struct LaneRecs {
    const uint4* rp;       // generic pointer to record 0 (the TMA-staged copy in shared
    const uint4* ep;       // memory, or global memory): one load instruction either way
};
struct LaneNoRecs {};

template <int kM>
struct Lane : std::conditional_t<kM == 3, LaneRecs, LaneNoRecs> {
    static constexpr bool kSmem = kM >= 1;
    static constexpr bool kTP = kM >= 2;
    static constexpr bool kGC = kM == 3; // instance memory cells in global memory
    static constexpr bool kCompact = kGC && kGcCompactVF;
    uint32_t vsh;    // kSmem: shared address of slot 0 (kCompact: its payload word)
    uint32_t vstr;   // kSmem: bytes from one slot to the next
    uint32_t gsh;    // kCompact: tag byte of the payload word at a = (a >> 2) + gsh (CTA-uniform)
    // kTP: only SSA values and phi staging live in the lane's value file; the
    // parameters (per test) and literals (per variant) are CTA-shared tables
    uint32_t nv;     // kTP: n_values (slots below: lane value file)
    uint32_t tsh;    // kTP: shared address of this test's parameter entry 0
    uint32_t tstr;   // kTP: bytes between parameter entries
    uint32_t lsh;    // kTP: shared address of literal 0 (slot lit_begin)
    uint32_t lit_begin;
    uint2* gvf;      // global value file (kM == 0)
    uint32_t base;   // element index of slot 0
    uint32_t row;
    // program
    const gevo_inst* code;
    const int64_t* suffix; // per-instruction cost of the rest of its block (this launch)
    const gevo_edge* edges; // per-instruction pre-resolved branch phis
    const uint4* dblk;  // block records of this variant
    const gevo_arm* arm;
    uint32_t n_values;
    uint32_t n_slots;
    uint32_t stage_base;
    uint64_t writable;
    // instance
    uint32_t v, t, il;
    uint32_t sl;     // spin-accelerator scratch column (instance, or lane when kTP)
    int32_t tid;
    const uint2* binfo;      // [param] {size << 8 | elem, pool word of element 0} of this test
    // thread-parallel (kTP)
    uint32_t csh;            // shared address of memory cell 0 of the instance
    uint32_t cstr;           // bytes from one cell to the next
    uint32_t rsh, wsh;       // shared addresses of this lane's read / write bitset chunk 0
    uint32_t bstr;           // bytes from one bitset chunk to the next
    uint32_t msh;            // shared address of the instance's min_stop
    uint32_t fsh;            // shared address of the instance's conflict flag
    uint32_t tsh_star;       // shared address of the instance's lowest conflicting thread
    uint2* gcell;            // kGC: cell 0 of the instance ([word][instance] in global memory)
    unsigned long long* gshadow; // kGC: per-word same-phase reader / writer record
    uint32_t gstr;           // kGC: elements from one word to the next (instances per launch)
    uint32_t epoch;          // phase number (max-tid-wins store rule)
    bool seq;                // sequential fallback: plain stores, no conflict tracking
    // counters
    int64_t cost;
    int64_t ir;
    uint32_t work;   // instructions this lane interpreted (diagnostic: jumps excluded,
                     // discarded attempts included)
    int32_t poll;
    uint32_t poll2;
    uint32_t jumps;   // spin-accelerator jumps (diagnostic, saturating)
    uint32_t spin_dbg;// last spin-accelerator abandon reason (diagnostic)
    // trap
    uint32_t code_out;
    int32_t aux;

    // kTP slot -> shared address: values, then params + poison (per test),
    // literals (per variant), then phi staging back in the lane's file
    __device__ __forceinline__ uint32_t tp_addr(uint32_t s) const {
        if (s < nv)
            return vsh + s * vstr;
        if (s < lit_begin)
            return tsh + (s - nv) * tstr;
        if (s < stage_base)
            return lsh + (s - lit_begin) * 8;
        return vsh + (nv + s - stage_base) * vstr;
    }
    // kCompact: row of a lane-file slot (values, then phi staging)
    __device__ __forceinline__ uint2 V(uint32_t s) const {
        if (kCompact) {
            if (!kTpTables) {
                const uint32_t a = vsh + s * 128;
                return make_uint2(lds1(a), ldsb((a >> 2) + gsh));
            }
            if (s < nv || s >= stage_base) {
                const uint32_t a = vsh + (s < nv ? s : nv + s - stage_base) * 128;
                return make_uint2(lds1(a), ldsb((a >> 2) + gsh));
            }
            return lds2(s < lit_begin ? tsh + (s - nv) * tstr : lsh + (s - lit_begin) * 8);
        }
        if (kTP && kTpTables)
            return lds2(tp_addr(s));
        if (kSmem)
            return lds2(vsh + s * vstr);
        return gvf[base + s * row];
    }
    __device__ __forceinline__ void W(uint32_t s, uint32_t payload, uint32_t tag) {
        if (kCompact) {
            if (!kTpTables) {
                const uint32_t a = vsh + s * 128;
                sts1(a, payload);
                stsb((a >> 2) + gsh, tag);
            } else if (s < nv || s >= stage_base) {
                const uint32_t a = vsh + (s < nv ? s : nv + s - stage_base) * 128;
                sts1(a, payload);
                stsb((a >> 2) + gsh, tag);
            } else {
                sts2(s < lit_begin ? tsh + (s - nv) * tstr : lsh + (s - lit_begin) * 8, payload, tag);
            }
            return;
        }
        if (kTP && kTpTables)
            sts2(tp_addr(s), payload, tag);
        else if (kSmem)
            sts2(vsh + s * vstr, payload, tag);
        else
            gvf[base + s * row] = make_uint2(payload, tag);
    }
    // instruction / branch-edge record idx of the variant (global-cell
    // kernels: the staged copy when the CTA staged it, through a generic
    // pointer; else the read-only global copy)
    __device__ __forceinline__ uint4 rec(uint32_t idx) const {
        if constexpr (kGC)
            return this->rp[idx];
        return __ldg(reinterpret_cast<const uint4*>(code) + idx);
    }
    __device__ __forceinline__ uint4 edge(uint32_t idx) const {
        if constexpr (kGC)
            return this->ep[idx];
        return __ldg(reinterpret_cast<const uint4*>(edges) + idx);
    }
    // kTP: shared address of memory cell w of the instance
    __device__ __forceinline__ uint32_t cell(uint32_t w) const { return csh + w * cstr; }
    // instance memory cell w, wherever it lives
    __device__ __forceinline__ uint2 cell_get(uint32_t w) const {
        if (kGC) {
            // volatile: bypass L1, which the compare-and-swap stores (L2) do not update
            const unsigned long long v = *reinterpret_cast<const volatile unsigned long long*>(
                gcell + static_cast<size_t>(w) * gstr);
            return make_uint2(static_cast<uint32_t>(v), static_cast<uint32_t>(v >> 32));
        }
        return lds2(cell(w));
    }
    __device__ __forceinline__ void cell_put(uint32_t w, uint32_t x, uint32_t y) const {
        if (kGC)
            *reinterpret_cast<volatile unsigned long long*>(gcell + static_cast<size_t>(w) * gstr) =
                (static_cast<unsigned long long>(y) << 32) | x;
        else
            sts2(cell(w), x, y);
    }
    __device__ __forceinline__ unsigned long long cell_cas(uint32_t w, unsigned long long cmp,
                                                           unsigned long long val) const {
        if (kGC)
            return atomicCAS(reinterpret_cast<unsigned long long*>(gcell + static_cast<size_t>(w) * gstr),
                             cmp, val);
        return cas64(cell(w), cmp, val);
    }

    __device__ __forceinline__ bool trap(uint32_t c, int32_t x = 0) {
        code_out = c;
        aux = x;
        return false;
    }
    // Trap of a generic fetch (vm.cpp:195-222) for a slot whose tag is t.
    __device__ __forceinline__ bool fetch_trap(uint32_t s, uint32_t t) {
        if (t == GEVO_TAG_UNDEF)
            return trap(GEVO_TRAP_UNDEF_VALUE, static_cast<int32_t>(s));
        if (t == GEVO_TAG_POISON_PARAM)
            return trap(GEVO_TRAP_BAD_PARAM);
        return trap(GEVO_TRAP_BAD_OPERAND);
    }
    // fetch (vm.cpp:195-222): undefined / poisoned slots trap.
    __device__ __forceinline__ bool fetch(uint32_t s, uint2& v) {
        v = V(s);
        if (bad_tag(v.y))
            return fetch_trap(s, v.y);
        return true;
    }
    // fetch_scalar (vm.cpp:224-229) failure: the first failing operand decides.
    __device__ __forceinline__ bool scalar_fail(uint32_t s, uint32_t t) {
        if (bad_tag(t))
            return fetch_trap(s, t);
        return trap(GEVO_TRAP_OPERAND_TYPE);
    }
    // fetch_ptr (vm.cpp:231-236)
    __device__ __forceinline__ bool pointer(uint32_t s, uint2& v) {
        if (!fetch(s, v))
            return false;
        if (!is_ptr_tag(v.y))
            return trap(GEVO_TRAP_NOT_POINTER);
        return true;
    }
    // set (vm.cpp:285-291)
    __device__ __forceinline__ bool set(uint32_t res, uint32_t payload, uint32_t t) {
        if (res == GEVO_NO_RESULT)
            return trap(GEVO_TRAP_DEF_NO_ID);
        W(res, payload, t);
        return true;
    }
};

struct Thread {
    int32_t block, ip, prev;
    int64_t executed;
    uint32_t bar;
    bool slow; // current block runs with per-instruction charging
    // executed count that arms the spin accelerator in the thread's next
    // phase (-1: the launch threshold). Kept across barriers, so a thread whose
    // loop contains a barrier does not restart an attempt every phase.
    int64_t spin_next = -1;
};

// Current block of a thread (decoded block record).
struct Blk {
    uint32_t start, len, nphi;
};

__device__ __forceinline__ Blk load_blk(const uint4* dblk, int32_t b, int64_t& cost) {
    const uint4 r = __ldg(dblk + b);
    Blk k;
    k.start = r.x;
    k.len = r.y & 0xFFFF;
    k.nphi = r.y >> 16;
    cost = static_cast<int64_t>((static_cast<uint64_t>(r.w) << 32) | r.z);
    return k;
}

// Spin-accelerator state of the running simulated thread.
struct Spin {
    uint32_t mode;     // 0 idle, 1 have S0, 2 abstract iterate running
    int32_t anchor;
    uint32_t skip;     // block entries to pass before choosing an anchor
    uint32_t attempts;
    int64_t next;      // executed count that arms the next attempt
    int64_t e0, c0;    // executed / lane cost at the reference iterate
    int64_t p, c;      // per-iteration instructions / cost
    int64_t H;         // iterations the abstract proof must cover
    int64_t K;         // iterations every compare of the iterate provably keeps its outcome
    int64_t Koob;      // iterations every strided load provably stays in bounds
    uint32_t nst, nld; // store / load log entries of the abstract iterate
    uint32_t retries;  // abstract iterates re-run with a widened hypothesis
    int32_t avoid;     // >= 0: block not to take as the next anchor; <= -2: block
                       // -avoid - 2 preferred as the next anchor; -1: none
    uint32_t nvk;      // memory words whose loads are varying (sp_vk)
};

// Cost of instructions [from, len) of a block (scalar arguments only: a
// reference to the lane would force it into local memory).
__device__ __noinline__ int64_t suffix_cost_of(const int64_t* cost, const gevo_inst* code,
                                               uint32_t start, uint32_t len, uint32_t from) {
    int64_t c = 0;
    for (uint32_t j = from; j < len; ++j)
        c += cost[__ldg(reinterpret_cast<const uint32_t*>(code + start + j)) >> 24];
    return c;
}

template <int kM>
__device__ __forceinline__ int64_t suffix_cost(const InterpArgs& A, const Lane<kM>& L, const Blk& b,
                                               uint32_t from) {
    if (L.suffix) // per-launch table: cost of [ip, len) for every instruction
        return from < b.len ? __ldg(L.suffix + b.start + from) : 0;
    return suffix_cost_of(A.cost, L.code, b.start, b.len, from);
}

// Charges instructions [from, len) of the current block on entry / resume.
template <int kM>
__device__ __forceinline__ void charge_block(const InterpArgs& A, Lane<kM>& L, Thread& th,
                                             const Blk& b, int64_t bcost, uint32_t from) {
    const int64_t n = static_cast<int64_t>(b.len) - from;
    if (th.executed + n <= A.budget) {
        L.cost += from == 0 ? bcost : suffix_cost(A, L, b, from);
        L.ir += n;
        L.work += static_cast<uint32_t>(n);
        th.executed += n;
        th.slow = false;
    } else {
        th.slow = true;
    }
}

// Refunds instructions [from, len) charged on entry that will not run.
template <int kM>
__device__ __forceinline__ void refund(const InterpArgs& A, Lane<kM>& L, Thread& th, const Blk& b,
                                       uint32_t from) {
    if (th.slow || from >= b.len)
        return;
    const int64_t n = static_cast<int64_t>(b.len) - from;
    L.cost -= suffix_cost(A, L, b, from);
    L.ir -= n;
    L.work -= static_cast<uint32_t>(n);
    th.executed -= n;
}

// Per-instruction charge (exact mode): cost and budget before any effect.
template <int kM>
__device__ __forceinline__ bool charge_one(const InterpArgs& A, Lane<kM>& L, Thread& th,
                                           uint32_t cls) {
    L.cost += A.cost[cls];
    ++L.ir;
    ++L.work;
    if (++th.executed > A.budget)
        return L.trap(GEVO_BUDGET_EXCEEDED);
    return true;
}

// ---- spin accelerator --------------------------------------------------------
//
// Abstract values of the iterate: affine int (stride, 0 = constant) or
// "varying" (any value; allowed only where it cannot change the path: float
// arithmetic, phi / select arms, stored values). A budget-bound spinner's
// record (status, cost, dynamic IR) depends on its path only, so varying
// values need no extrapolation; everything the path reads (branch and select
// conditions, compare operands, addresses, divisors, tags) must be affine
// with a provably constant outcome.

template <int kM>
__device__ __forceinline__ size_t sp_at(const InterpArgs& A, const Lane<kM>& L, uint32_t s) {
    return static_cast<size_t>(s) * A.n_spin + L.sl;
}

template <int kM>
__device__ __forceinline__ void spin_abandon(Spin& S, const Thread& th, Lane<kM>& L,
                                             uint32_t why) {
    ++S.attempts;
    S.skip = S.attempts & 3u;
#ifndef GEVO_SPIN_BACKOFF
#define GEVO_SPIN_BACKOFF 1 // next attempt after executed * (1 + 2^-shift): shift 1 = x1.5
#endif
    S.next = S.attempts > kSpinAttempts ? INT64_MAX : th.executed + (th.executed >> GEVO_SPIN_BACKOFF) + 64;
    if (S.mode == 2 && S.K < S.H && S.attempts <= kSpinAttempts) {
        // The anchor's loop leaves its path within K + 1 iterations (an inner
        // loop running out): try again right after that, at a block other
        // than this anchor -- typically the enclosing loop, whose iterations
        // repeat with a fixed path.
        S.next = S.e0 + (S.K + 1) * S.p + 1;
        S.skip = 0;
        S.avoid = S.anchor;
    }
    S.mode = 0;
    L.spin_dbg = why;
}

__device__ __forceinline__ bool slot_strided(uint32_t tag) {
    return tag == GEVO_TAG_I32 || is_ptr_tag(tag);
}

// Largest K in [0, H] such that (X + k*sx) pred (Y + k*sy) keeps its k = 0
// outcome for every k in [0, K] with neither side leaving the int32 range.
__device__ int64_t cmp_horizon(int32_t X, int32_t sx, int32_t Y, int32_t sy, uint32_t pred,
                               int64_t H) {
    // int32 range: |side(k)| stays representable for k <= K
    auto range = [](int64_t v, int64_t s, int64_t h) -> int64_t {
        if (s > 0)
            return min(h, (static_cast<int64_t>(INT32_MAX) - v) / s);
        if (s < 0)
            return min(h, (v - static_cast<int64_t>(INT32_MIN)) / -s);
        return h;
    };
    H = range(X, sx, range(Y, sy, H));
    const int64_t f0 = static_cast<int64_t>(X) - Y;
    const int64_t slope = static_cast<int64_t>(sx) - sy;
    if (slope == 0 || H <= 0)
        return H;
    if (pred <= 1) { // eq / ne: the outcome changes at the first root of f in [1, H]
        if (f0 == 0)
            return 0;
        if (f0 % slope != 0)
            return H;
        const int64_t r = -f0 / slope;
        return (r < 1 || r > H) ? H : r - 1;
    }
    // lt / le / gt / ge of an affine f: monotone in k, at most one change
    const bool c0 = cmp(static_cast<int64_t>(X), static_cast<int64_t>(Y), pred);
    auto same = [&](int64_t k) {
        return cmp(static_cast<int64_t>(X) + k * sx, static_cast<int64_t>(Y) + k * sy, pred) == c0;
    };
    if (same(H))
        return H;
    int64_t lo = 0, hi = H; // same(lo), !same(hi)
    while (hi - lo > 1) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (same(mid))
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

// Largest K in [0, H] such that X + k*sx and Y + k*sy stay int32 and their
// sum stays in [0, size) for every k in [0, K]; -1 when k = 0 already fails.
__device__ int64_t affine_in_bounds(int32_t X, int32_t sx, int32_t Y, int32_t sy, int32_t size,
                                    int64_t H) {
    auto range = [](int64_t v, int64_t s, int64_t h) -> int64_t {
        if (s > 0)
            return min(h, (static_cast<int64_t>(INT32_MAX) - v) / s);
        if (s < 0)
            return min(h, (v - static_cast<int64_t>(INT32_MIN)) / -s);
        return h;
    };
    H = range(X, sx, range(Y, sy, H));
    const int64_t e0 = static_cast<int64_t>(X) + Y, st = static_cast<int64_t>(sx) + sy;
    if (e0 < 0 || e0 >= size)
        return -1;
    if (st > 0)
        return min(H, (static_cast<int64_t>(size) - 1 - e0) / st);
    if (st < 0)
        return min(H, e0 / -st);
    return H;
}

template <int kM>
__device__ __forceinline__ uint32_t spin_stride(const InterpArgs& A, const Lane<kM>& L,
                                                uint32_t s) {
    return s < L.n_slots ? A.sp_cur[sp_at(A, L, s)] : 0u;
}
template <int kM>
__device__ __forceinline__ uint32_t spin_vary(const InterpArgs& A, const Lane<kM>& L,
                                              uint32_t s) {
    return s < L.n_slots ? A.sp_cvary[sp_at(A, L, s)] : 0u;
}
template <int kM>
__device__ __forceinline__ void spin_set(const InterpArgs& A, const Lane<kM>& L, uint32_t s,
                                         uint32_t stride, uint32_t vary) {
    if (s < L.n_slots) {
        A.sp_cur[sp_at(A, L, s)] = stride;
        A.sp_cvary[sp_at(A, L, s)] = static_cast<uint8_t>(vary);
    }
}

// Memory word key of a store / load of the iterate (0: not representable).
__device__ __forceinline__ uint32_t mem_key(uint32_t ptag, int64_t eff) {
    if (eff < 0 || eff >= (1 << 24))
        return 0;
    const uint32_t space = ptag == GEVO_TAG_PTR_SHARED ? 0x80u : ((ptag & 0x3F) + 1);
    return (space << 24) | static_cast<uint32_t>(eff);
}

template <int kM>
__device__ __forceinline__ size_t log_at(const InterpArgs& A, const Lane<kM>& L, uint32_t i,
                                         uint32_t field) {
    return (static_cast<size_t>(field) * kSpinLog + i) * A.n_spin + L.sl;
}

// Current memory word (payload, tag) behind a key.
template <int kM>
__device__ __forceinline__ uint2 mem_word(const InterpArgs& A, const Lane<kM>& L, uint32_t key) {
    const uint32_t eff = key & 0xFFFFFF, space = key >> 24;
    if (Lane<kM>::kTP) {
        const uint2 c = L.cell_get(space == 0x80 ? eff : A.cell_off[space - 1] + eff);
        return make_uint2(c.x, c.y & kCellTag);
    }
    if (space == 0x80) {
        const size_t at = static_cast<size_t>(eff) * A.n_inst + L.il;
        return make_uint2(A.sh_val[at], A.sh_tag[at]);
    }
    const uint32_t prm = space - 1;
    return make_uint2(A.priv[A.priv_off[prm] + static_cast<size_t>(eff) * A.n_inst + L.il], 0);
}

// Stride transfer of one instruction of the abstract iterate, called before
// its concrete execution (operands still hold their k = 0 values). Returns
// false when the instruction breaks the proof.
template <int kM>
__device__ __forceinline__ bool spin_track(const InterpArgs& A, const Lane<kM>& L,
                                           const uint4 r, Spin& S) {
    const uint32_t op = f_op(r), a = f_a(r), b = f_b(r), c = f_c(r), res = f_res(r);
    uint32_t out = 0, vout = 0;
    const uint32_t sa = spin_stride(A, L, a), sb = spin_stride(A, L, b);
    const uint32_t va = spin_vary(A, L, a), vb = spin_vary(A, L, b);
    switch (op) {
    case GEVO_OP_ADD: out = sa + sb; vout = va | vb; break;
    case GEVO_OP_SUB: out = sa - sb; vout = va | vb; break;
    case GEVO_OP_GETINDEX: out = sa + sb; vout = va | vb; break;
    case GEVO_OP_MUL:
        vout = va | vb;
        if (!vout) {
            if (sa && sb)
                vout = 1;
            else
                out = sa ? sa * L.V(b).x : sb * L.V(a).x;
        }
        break;
    case GEVO_OP_SDIV: // may trap: operands must be fixed
        if (sa | sb | va | vb)
            return false;
        break;
    case GEVO_OP_FADD: case GEVO_OP_FSUB: case GEVO_OP_FMUL: case GEVO_OP_FDIV:
    case GEVO_OP_FCMP:
        vout = (sa | sb | va | vb) ? 1u : 0u;
        break;
    case GEVO_OP_ICMP:
        if (va | vb) {
            vout = 1;
        } else if (sa | sb) {
            const uint2 x = L.V(a), y = L.V(b);
            if (x.y != GEVO_TAG_I32 || y.y != GEVO_TAG_I32)
                return false;
            const int64_t K = cmp_horizon(static_cast<int32_t>(x.x), static_cast<int32_t>(sa),
                                          static_cast<int32_t>(y.x), static_cast<int32_t>(sb),
                                          f_aux(r), S.K);
            S.K = K;
            if (K < kSpinMinJump)
                return false;
        }
        break;
    case GEVO_OP_SELECT: {
        if (sa | va)
            return false;
        const uint32_t arm = L.V(a).x ? b : c;
        out = spin_stride(A, L, arm);
        vout = spin_vary(A, L, arm);
        break;
    }
    case GEVO_OP_LOAD: case GEVO_OP_STORE: {
        if (va | vb)
            return false;
        const uint2 p = L.V(a), i = L.V(b);
        if (!is_ptr_tag(p.y) || i.y != GEVO_TAG_I32)
            return false;
        if (sa | sb) {
            // Strided load from a read-only global buffer: the value varies
            // (path-irrelevant by the other obligations) and the address stays
            // in bounds for K_oob iterations; the first out-of-bounds
            // iteration traps for sure, which bounds the jump (trap horizon).
            if (op != GEVO_OP_LOAD || p.y == GEVO_TAG_PTR_SHARED)
                return false;
            const uint32_t prm = p.y & 0x3F;
            if ((L.writable >> prm) & 1ull)
                return false;
            const int32_t size = __ldg(A.buf_size + static_cast<size_t>(L.t) * A.n_params + prm);
            const int64_t K = affine_in_bounds(static_cast<int32_t>(p.x), static_cast<int32_t>(sa),
                                               static_cast<int32_t>(i.x), static_cast<int32_t>(sb),
                                               size, S.Koob);
            if (K < 0)
                return false;
            S.Koob = K;
            vout = 1;
            break;
        }
        const int64_t eff = static_cast<int64_t>(static_cast<int32_t>(p.x)) +
                            static_cast<int32_t>(i.x);
        if (p.y == GEVO_TAG_PTR_SHARED) {
            if (eff < 0 || eff >= A.shared_words)
                return false;
        } else {
            const uint32_t prm = p.y & 0x3F;
            const int32_t size = __ldg(A.buf_size + static_cast<size_t>(L.t) * A.n_params + prm);
            if (eff < 0 || eff >= size)
                return false;
            if (!((L.writable >> prm) & 1ull)) {
                if (op == GEVO_OP_STORE)
                    return false;
                break; // read-only pool word: constant
            }
        }
        const uint32_t key = mem_key(p.y, eff);
        if (!key)
            return false;
        uint32_t hit = kSpinLog;
        for (uint32_t j = 0; j < S.nst; ++j)
            if (A.sp_log[log_at(A, L, j, 0)] == key)
                hit = j;
        if (op == GEVO_OP_LOAD) {
            bool vk = false;
            for (uint32_t k = 0; k < S.nvk; ++k)
                vk |= A.sp_vk[static_cast<size_t>(k) * A.n_spin + L.sl] == key;
            if (vk || (hit < kSpinLog && (A.sp_log[log_at(A, L, hit, 2)] & 0x100))) {
                vout = 1;
            } else {
                if (S.nld >= kSpinLog)
                    return false;
                A.sp_ld[log_at(A, L, S.nld++, 0)] = key;
            }
            break;
        }
        const uint32_t vary_store = (spin_stride(A, L, c) | spin_vary(A, L, c)) ? 0x100u : 0u;
        if (hit == kSpinLog) {
            if (S.nst >= kSpinLog)
                return false;
            const uint2 old = mem_word(A, L, key);
            A.sp_log[log_at(A, L, S.nst, 0)] = key;
            A.sp_log[log_at(A, L, S.nst, 1)] = old.x;
            A.sp_log[log_at(A, L, S.nst, 2)] = old.y | vary_store;
            hit = S.nst++;
        } else {
            A.sp_log[log_at(A, L, hit, 2)] |= vary_store;
        }
        // the thread's own last store to the word in the iterate
        const uint2 sv = L.V(c);
        A.sp_log[log_at(A, L, hit, 3)] = sv.x;
        A.sp_log[log_at(A, L, hit, 4)] = sv.y;
        return true;
    }
    case GEVO_OP_BR:
        return !(f_aux(r) == 2 && (sa | va));
    case GEVO_OP_CONST: out = sa; vout = va; break;
    default: break; // tid / nthreads / sync / ret: fixed or no result
    }
    if (res != GEVO_NO_RESULT)
        spin_set(A, L, res, vout ? 0u : out, vout);
    return true;
}

// Runs the abstract iterate again from the current anchor entry (S2 becomes
// the new S1) with the widened hypothesis: varying slots (sp_hvary) and
// varying memory words (sp_vk) stay varying.
template <int kM>
__device__ __forceinline__ void spin_restart_iterate(const InterpArgs& A, Lane<kM>& L, Thread& th,
                                                     Spin& S) {
    for (uint32_t x = 0; x < L.n_values; ++x) {
        const size_t at = sp_at(A, L, x);
        const uint32_t vary = A.sp_hvary[at];
        const uint32_t d = vary ? 0u : A.sp_delta[at];
        A.sp_delta[at] = d;
        A.sp_base[at] = L.V(x).x;
        A.sp_cur[at] = d;
        A.sp_cvary[at] = static_cast<uint8_t>(vary);
    }
    for (uint32_t x = L.n_values; x < L.n_slots; ++x) {
        A.sp_cur[sp_at(A, L, x)] = 0;
        A.sp_cvary[sp_at(A, L, x)] = 0;
    }
    S.e0 = th.executed;
    S.c0 = L.cost;
    S.nst = 0;
    S.nld = 0;
    S.H = (A.budget - th.executed) / S.p;
    S.K = S.H;
    S.Koob = S.H;
    if (S.H < 3)
        spin_abandon(S, th, L, 4);
}

// Protocol step at every completed block entry (phis done).
template <int kM>
__device__ __forceinline__ void spin_at_entry(const InterpArgs& A, Lane<kM>& L, Thread& th,
                                              Spin& S) {
    if (S.mode == 0) {
        if (th.executed < S.next)
            return;
        if (S.skip) {
            --S.skip;
            return;
        }
        // after an inner loop ran out, prefer an anchor in a block laid out
        // before it (an enclosing loop's header precedes its body) for a few
        // of its periods, then any block but the failed anchor
        if (S.avoid >= 0 && th.block >= S.avoid && th.executed < S.next + 4 * S.p + 256)
            return;
        if (th.block == S.avoid)
            return;
        // after a partial jump (the loop ran to the compare flip) the next
        // instance of the same loop is the likely spinner again (an inner
        // loop re-entered by its enclosing loop): wait for its anchor block
        // for a while before taking any other
        if (S.avoid <= -2 && th.block != -S.avoid - 2 && th.executed < S.next + kPreferWindow * S.p + 64)
            return;
        for (uint32_t x = 0; x < L.n_values; ++x) {
            const uint2 v = L.V(x);
            A.sp_base[sp_at(A, L, x)] = v.x;
            A.sp_btag[sp_at(A, L, x)] = static_cast<uint8_t>(v.y);
        }
        S.anchor = th.block;
        S.e0 = th.executed;
        S.c0 = L.cost;
        S.mode = 1;
        return;
    }
    if (th.block != S.anchor)
        return;
    if (S.mode == 1) {
        // S1: stride hypothesis from S1 - S0 (non-int changes: varying)
        const int64_t p = th.executed - S.e0;
        if (p <= 0) {
            spin_abandon(S, th, L, 1);
            return;
        }
#ifndef GEVO_SPIN_NOCHUNK
        // (snapshot words read in chunks: independent global loads in flight
        // together instead of one round trip per slot)
        constexpr uint32_t kChunk = 4;
        for (uint32_t x0 = 0; x0 < L.n_values; x0 += kChunk) {
            uint32_t bt[kChunk], bb[kChunk];
#pragma unroll
            for (uint32_t k = 0; k < kChunk; ++k)
                if (x0 + k < L.n_values) {
                    const size_t at = sp_at(A, L, x0 + k);
                    bt[k] = A.sp_btag[at];
                    bb[k] = A.sp_base[at];
                }
#pragma unroll
            for (uint32_t k = 0; k < kChunk; ++k) {
                if (x0 + k >= L.n_values)
                    break;
                const uint2 v = L.V(x0 + k);
                if (bt[k] != v.y) {
                    spin_abandon(S, th, L, 2);
                    return;
                }
                const size_t at = sp_at(A, L, x0 + k);
                uint32_t d = v.x - bb[k];
                uint8_t vary = 0;
                if (d && !slot_strided(v.y)) {
                    vary = 1;
                    d = 0;
                }
                A.sp_delta[at] = d;
                A.sp_base[at] = v.x;
                A.sp_cur[at] = d;
                A.sp_hvary[at] = vary;
                A.sp_cvary[at] = vary;
            }
        }
#else
        for (uint32_t x = 0; x < L.n_values; ++x) {
            const uint2 v = L.V(x);
            const size_t at = sp_at(A, L, x);
            if (A.sp_btag[at] != v.y) {
                spin_abandon(S, th, L, 2);
                return;
            }
            uint32_t d = v.x - A.sp_base[at];
            uint8_t vary = 0;
            if (d && !slot_strided(v.y)) {
                vary = 1;
                d = 0;
            }
            A.sp_delta[at] = d;
            A.sp_base[at] = v.x;
            A.sp_cur[at] = d;
            A.sp_hvary[at] = vary;
            A.sp_cvary[at] = vary;
        }
#endif
        for (uint32_t x = L.n_values; x < L.n_slots; ++x) {
            A.sp_cur[sp_at(A, L, x)] = 0;
            A.sp_cvary[sp_at(A, L, x)] = 0;
        }
        S.p = p;
        S.c = L.cost - S.c0;
        S.e0 = th.executed;
        S.c0 = L.cost;
        S.nst = 0;
        S.nld = 0;
        S.retries = 0;
        S.nvk = 0;
        S.H = (A.budget - th.executed) / p;
        S.K = S.H;
        S.Koob = S.H;
        if (S.H < 3) {
            spin_abandon(S, th, L, 4);
            return;
        }
        S.mode = 2;
        return;
    }
    // mode 2: the abstract iterate arrived back at the anchor (S2).
    if (th.executed - S.e0 != S.p || L.cost - S.c0 != S.c) {
        spin_abandon(S, th, L, 5);
        return;
    }
    // Slots whose observed behaviour contradicts the hypothesis (a changing
    // "fixed" slot, a broken stride) become varying and the abstract iterate
    // is re-run from S2; varying only grows, so this converges.
    bool retry = false;
    for (uint32_t x = 0; x < L.n_values; ++x) {
        const uint2 v = L.V(x);
        const size_t at = sp_at(A, L, x);
        if (A.sp_btag[at] != v.y) {
            spin_abandon(S, th, L, 6);
            return;
        }
        if (!A.sp_hvary[at] && (A.sp_cvary[at] || v.x - A.sp_base[at] != A.sp_delta[at] ||
                                A.sp_cur[at] != A.sp_delta[at])) {
            A.sp_hvary[at] = 1;
            retry = true;
        }
    }
    if (retry) {
        if (++S.retries > 4) {
            spin_abandon(S, th, L, 9);
            return;
        }
        spin_restart_iterate(A, L, th, S);
        return;
    }
    // memory: a word the iterate stores a fixed value to and also reads must
    // end the iterate with its S1 contents (each iteration then reads the same
    // value); no load reads a word that holds varying data. Words the iterate
    // only writes get the same fixed value in every iteration, so skipping
    // iterations leaves memory as running them would. The comparison uses the
    // thread's own last store (with thread-parallel lanes a concurrent writer
    // of the word can only be another thread, whose same-phase write plus this
    // read is a conflict that re-runs the instance in thread-id order).
    for (uint32_t j = 0; j < S.nst; ++j) {
        const uint32_t key = A.sp_log[log_at(A, L, j, 0)];
        const uint32_t tf = A.sp_log[log_at(A, L, j, 2)];
        bool loaded = false;
        for (uint32_t k = 0; k < S.nld; ++k)
            loaded |= A.sp_ld[log_at(A, L, k, 0)] == key;
        if (!loaded)
            continue;
        if ((tf & 0x100) || A.sp_log[log_at(A, L, j, 3)] != A.sp_log[log_at(A, L, j, 1)] ||
            A.sp_log[log_at(A, L, j, 4)] != (tf & 0xFF)) {
            // The word a load reads changes from one iteration to the next:
            // treat its loads as varying (path-irrelevant data) and run the
            // abstract iterate again; the path obligations then decide.
            if (S.nvk >= kSpinLog || ++S.retries > 4) {
                spin_abandon(S, th, L, (tf & 0x100) ? 7 : 8);
                return;
            }
            A.sp_vk[static_cast<size_t>(S.nvk++) * A.n_spin + L.sl] = key;
            spin_restart_iterate(A, L, th, S);
            return;
        }
    }
    // Jump n whole iterations. Iteration k = 0 is the abstract iterate, the jump skips k = 1..n and
    // interpretation resumes at k = n + 1. With m = min(budget-bound count,
    // last in-bounds iteration of every strided load), if the path provably
    // stays fixed through iteration m + 1 (every compare keeps its outcome),
    // the resumed iteration ends the thread by the budget or an out-of-bounds
    // trap on the reference's instruction whatever the path-irrelevant
    // ("varying") values are. Otherwise only a jump up to the first compare
    // flip is possible, and the execution it resumes may complete, so it needs
    // exact values everywhere: no varying slot, no varying store.
    const int64_t n_budget = (A.budget - th.executed) / S.p;
    const int64_t m = min(n_budget, S.Koob);
    int64_t n = m;
    if (S.K < m + 1) {
        n = S.K;
        bool vary = n < kSpinMinJump;
        for (uint32_t x = 0; x < L.n_values && !vary; ++x)
            vary = A.sp_hvary[sp_at(A, L, x)] != 0;
        for (uint32_t j = 0; j < S.nst && !vary; ++j)
            vary = (A.sp_log[log_at(A, L, j, 2)] & 0x100) != 0;
        if (vary) {
            spin_abandon(S, th, L, 10);
            return;
        }
    }
    if (n > 0) {
        for (uint32_t x = 0; x < L.n_values; ++x) {
            const size_t at = sp_at(A, L, x);
            const uint32_t d = A.sp_delta[at];
            if (d && !A.sp_hvary[at]) {
                const uint2 v = L.V(x);
                L.W(x, v.x + static_cast<uint32_t>(n) * d, v.y);
            }
        }
        th.executed += n * S.p;
        L.ir += n * S.p;
        L.cost += n * S.c;
        L.jumps = min(L.jumps + 1u, 255u);
        if (A.counters) {
            atomicAdd(reinterpret_cast<unsigned long long*>(A.counters), 1ull);
            atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 1),
                      static_cast<unsigned long long>(n * S.p));
        }
    }
    S.mode = 0;
    if (n < m || S.K < m + 1) {
        // interpret past the flip, then look for the next affine stretch
        // (re-arming only after jumps that paid for themselves measured 2x
        // slower on config 2: its loops live on many short jumps); a jump
        // short against the value file the attempt walks backs off instead
        if (n * S.p < static_cast<int64_t>(A.spin_pay) * L.n_values) {
            ++S.attempts;
            S.skip = S.attempts & 3u;
            S.next = S.attempts > kSpinAttempts ? INT64_MAX
                                                : th.executed + (th.executed >> GEVO_SPIN_BACKOFF) + 64;
        } else {
            S.skip = 0;
            S.attempts = 0;
            S.next = th.executed + 2 * S.p + 16;
        }
        S.avoid = -S.anchor - 2; // prefer this anchor next
    } else {
        S.next = INT64_MAX;
    }
}

// Phi arm for predecessor `prev` (first matching arm, vm.cpp:311-323);
// returns false when no arm matches.
template <int kM>
__device__ __forceinline__ bool phi_arm(const Lane<kM>& L, const uint4 r, int32_t prev,
                                        uint32_t& ref) {
    const uint32_t n = f_aux(r);
    if (n <= 2) {
        if (n >= 1 && f_t0(r) == prev) {
            ref = f_a(r);
            return true;
        }
        if (n == 2 && f_t1(r) == prev) {
            ref = f_b(r);
            return true;
        }
        return false;
    }
    const uint32_t* arms = reinterpret_cast<const uint32_t*>(L.arm) + f_c(r);
    for (uint32_t a = 0; a < n; ++a) {
        const uint32_t raw = __ldg(arms + a);
        if (static_cast<int16_t>(raw & 0xFFFF) == prev) {
            ref = raw >> 16;
            return true;
        }
    }
    return false;
}

// enter_block (vm.cpp:293-333): charge and stage every leading phi, then write.
template <int kM>
__device__ __forceinline__ bool enter_block(const InterpArgs& A, Lane<kM>& L, Thread& th,
                            int32_t target, Blk& b, Spin& S, uint2 edge) {
    th.prev = th.block;
    th.block = target;
    th.ip = 0;
    int64_t bcost;
    b = load_blk(L.dblk, target, bcost);
    charge_block(A, L, th, b, bcost, 0);
    const uint32_t n = b.nphi;
    if (n == 0)
        return true;
    const bool track = S.mode == 2;
    if (!th.slow && !track && edge.x != GEVO_EDGE_NONE) {
        // <= 2 phis resolved for this edge at encode time (no arm matching)
        const uint32_t ref0 = edge.x & 0xFFFF;
        uint2 v0, v1;
        if (n == 2) {
            // both arms read at once; the checks below then only re-read
            // on a failure path
            const uint32_t ref1 = edge.y & 0xFFFF;
            if (ref0 != GEVO_EDGE_NOINC && ref1 != GEVO_EDGE_NOINC) {
                v0 = L.V(ref0);
                v1 = L.V(ref1);
                if (!bad_tag(v0.y) && !bad_tag(v1.y)) {
                    th.ip = 2;
                    L.W(edge.y >> 16, v1.x, v1.y);
                    L.W(edge.x >> 16, v0.x, v0.y);
                    return true;
                }
            }
        }
        if (ref0 == GEVO_EDGE_NOINC) {
            refund(A, L, th, b, 1);
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        }
        if (!L.fetch(ref0, v0)) {
            refund(A, L, th, b, 1);
            return false;
        }
        th.ip = 1;
        if (n == 2) {
            const uint32_t ref1 = edge.y & 0xFFFF;
            if (ref1 == GEVO_EDGE_NOINC) {
                refund(A, L, th, b, 2);
                return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
            }
            if (!L.fetch(ref1, v1)) {
                refund(A, L, th, b, 2);
                return false;
            }
            th.ip = 2;
            L.W(edge.y >> 16, v1.x, v1.y);
        }
        L.W(edge.x >> 16, v0.x, v0.y);
        return true;
    }
    if (n == 2 && !th.slow && !track) {
        // loop headers: both arms read before either phi writes (parallel copy)
        const uint4 r0 = L.rec(b.start), r1 = L.rec(b.start + 1);
        uint32_t ref0, ref1;
        uint2 v0, v1;
        if (!phi_arm(L, r0, th.prev, ref0)) {
            refund(A, L, th, b, 1);
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        }
        if (!L.fetch(ref0, v0)) {
            refund(A, L, th, b, 1);
            return false;
        }
        th.ip = 1;
        if (!phi_arm(L, r1, th.prev, ref1)) {
            refund(A, L, th, b, 2);
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        }
        if (!L.fetch(ref1, v1)) {
            refund(A, L, th, b, 2);
            return false;
        }
        th.ip = 2;
        if (!L.set(f_res(r0), v0.x, v0.y) || !L.set(f_res(r1), v1.x, v1.y)) {
            refund(A, L, th, b, 2);
            return false;
        }
        return true;
    }
    if (n == 1) {
        // a single phi reads nothing another phi writes: no staging needed
        const uint4 r = L.rec(b.start);
        if (th.slow && !charge_one(A, L, th, f_cls(r)))
            return false;
        uint32_t ref;
        if (!phi_arm(L, r, th.prev, ref)) {
            refund(A, L, th, b, 1);
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        }
        uint2 v;
        if (!L.fetch(ref, v)) {
            refund(A, L, th, b, 1);
            return false;
        }
        th.ip = 1;
        if (!L.set(f_res(r), v.x, v.y)) {
            refund(A, L, th, b, 1);
            return false;
        }
        if (track)
            spin_set(A, L, f_res(r), spin_stride(A, L, ref), spin_vary(A, L, ref));
        return true;
    }
    for (uint32_t j = 0; j < n; ++j) {
        const uint4 r = L.rec(b.start + j);
        if (th.slow && !charge_one(A, L, th, f_cls(r)))
            return false;
        uint32_t ref;
        if (!phi_arm(L, r, th.prev, ref)) {
            refund(A, L, th, b, j + 1);
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        }
        uint2 v;
        if (!L.fetch(ref, v)) {
            refund(A, L, th, b, j + 1);
            return false;
        }
        L.W(L.stage_base + j, v.x, v.y);
        if (track)
            spin_set(A, L, L.stage_base + j, spin_stride(A, L, ref), spin_vary(A, L, ref));
        ++th.ip;
    }
    for (uint32_t j = 0; j < n; ++j) {
        const uint4 r = L.rec(b.start + j);
        const uint2 v = L.V(L.stage_base + j);
        if (!L.set(f_res(r), v.x, v.y)) {
            refund(A, L, th, b, n);
            return false;
        }
        if (track)
            spin_set(A, L, f_res(r), spin_stride(A, L, L.stage_base + j),
                     spin_vary(A, L, L.stage_base + j));
    }
    return true;
}

// Same-phase access bookkeeping of a thread-parallel lane. Shared-memory
// cells: per-lane read / write bitsets, checked at the phase end. Global
// cells: a per-word record {writer epoch, writer, reader epoch, reader}
// (0xFFFF = several threads) updated with one compare-and-swap; a read and a
// write of the same word by different threads in one epoch flags the
// instance right away (the CAS orders them, so one of the two sees the other).
template <int kM>
__device__ __forceinline__ void tp_note(const Lane<kM>& L, uint32_t w, bool write) {
    if (!Lane<kM>::kGC) {
        const uint32_t ba = (write ? L.wsh : L.rsh) + (w >> 5) * L.bstr;
        sts1(ba, lds1(ba) | (1u << (w & 31)));
        return;
    }
    unsigned long long* sp = L.gshadow + static_cast<size_t>(w) * L.gstr;
    const uint32_t me = static_cast<uint32_t>(L.tid), ep = L.epoch & 0xFFFF;
    unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(sp);
    for (;;) {
        uint32_t wr = static_cast<uint32_t>(cur >> 32), rd = static_cast<uint32_t>(cur);
        uint32_t& mine = write ? wr : rd;
        const uint32_t other = write ? rd : wr;
        if ((other >> 16) == ep && (other & 0xFFFF) != me) {
            sts1(L.fsh, 1u); // same-phase cross-thread read / write
            return;
        }
        uint32_t next = mine;
        if ((mine >> 16) != ep)
            next = (ep << 16) | me;
        else if ((mine & 0xFFFF) != me)
            next = (ep << 16) | 0xFFFFu;
        if (next == mine)
            return;
        mine = next;
        const unsigned long long want = (static_cast<unsigned long long>(wr) << 32) | rd;
        const unsigned long long prev = atomicCAS(sp, cur, want);
        if (prev == cur)
            return;
        cur = prev;
    }
}

// Fast path of the common memory instructions of a thread-parallel lane: all
// operands are fetched at once (independent shared-memory reads in flight
// together) and the instruction completes here when every check passes. Any
// failing check returns false before a side effect, and mem_op then runs the
// instruction with the reference's check order and trap reasons.
template <int kM>
__device__ __forceinline__ bool mem_fast(const InterpArgs& A, Lane<kM>& L, const uint4 r) {
    const uint32_t op = f_op(r), res = f_res(r);
    const bool store = op == GEVO_OP_STORE;
    const uint2 p = L.V(f_a(r)), ix = L.V(f_b(r));
    const uint2 val = store ? L.V(f_c(r)) : make_uint2(0, 0);
    if (ix.y != GEVO_TAG_I32)
        return false;
    if (store ? (val.y != GEVO_TAG_I32 && val.y != GEVO_TAG_F32) : res == GEVO_NO_RESULT)
        return false;
    const int64_t eff = static_cast<int64_t>(static_cast<int32_t>(p.x)) +
                        static_cast<int64_t>(static_cast<int32_t>(ix.x));
    uint32_t w;
    if (p.y == GEVO_TAG_PTR_SHARED) {
        if (static_cast<uint64_t>(eff) >= static_cast<uint64_t>(static_cast<uint32_t>(A.shared_words)))
            return false;
        w = static_cast<uint32_t>(eff);
        if (!store) {
            const uint2 x = L.cell_get(w);
            const uint32_t wt = x.y & kCellTag;
            if (wt != f_aux(r)) // uninitialised (tag 0) or another type
                return false;
            if (!L.seq)
                tp_note(L, w, false);
            tp_read_check(L, x.y);
            L.W(res, x.x, wt);
            return true;
        }
    } else if (p.y >= static_cast<uint32_t>(GEVO_TAG_PTR_GLOBAL)) {
        const uint32_t prm = p.y & 0x3F;
        const uint2 bi = __ldg(L.binfo + prm);
        if (static_cast<uint64_t>(eff) >= static_cast<uint64_t>(bi.x >> 8))
            return false;
        const uint32_t elem = bi.x & 0xFF;
        const bool priv = (L.writable >> prm) & 1ull;
        if (!store) {
            if (elem != f_aux(r))
                return false;
            if (!priv) {
                L.W(res, __ldg(A.pool + bi.y + static_cast<uint32_t>(eff) * static_cast<uint32_t>(A.n_tests)),
                    elem);
                return true;
            }
            w = A.cell_off[prm] + static_cast<uint32_t>(eff);
            const uint2 x = L.cell_get(w);
            if (!L.seq)
                tp_note(L, w, false);
            tp_read_check(L, x.y);
            L.W(res, x.x, x.y & kCellTag);
            return true;
        }
        if (elem != val.y || !priv)
            return false;
        w = A.cell_off[prm] + static_cast<uint32_t>(eff);
    } else {
        return false;
    }
    // store to an instance cell (as mem_op)
    if (L.seq) {
        L.cell_put(w, val.x, val.y);
        return true;
    }
    const uint32_t me = static_cast<uint32_t>(L.tid) + 1;
    const uint32_t meta = cell_meta(val.y, me, L.epoch);
    const unsigned long long want = (static_cast<unsigned long long>(meta) << 32) | val.x;
    const uint2 c0 = L.cell_get(w);
    tp_note(L, w, true);
    unsigned long long cur = (static_cast<unsigned long long>(c0.y) << 32) | c0.x;
    for (;;) {
        const uint32_t m = static_cast<uint32_t>(cur >> 32);
        if ((m >> 16) == L.epoch && cell_writer(m) > me)
            break;
        const unsigned long long prev = L.cell_cas(w, cur, want);
        if (prev == cur)
            break;
        cur = prev;
    }
    return true;
}

// A shared-memory-cell read of a concurrent phase that returned another
// simulated thread's write of this phase (the cell's writer/epoch meta): the
// reference, running threads one after another, could not have produced it
// (a higher writer runs later; a lower one may still write again), so the
// instance is flagged and the reading thread bounds the re-run's
// conflict-free prefix. Reads of phase-start or own values are clean; whether
// a lower thread writes such a word later is checked with the bitsets at the
// phase end.
template <int kM>
__device__ __forceinline__ void tp_read_check(const Lane<kM>& L, uint32_t meta) {
    if (Lane<kM>::kGC || L.seq)
        return;
    if ((meta >> 16) == (L.epoch & 0xFFFFu) && cell_writer(meta) != static_cast<uint32_t>(L.tid) + 1) {
        sts1(L.fsh, 1u);
        asm volatile("red.shared.min.s32 [%0], %1;" ::"r"(L.tsh_star), "r"(L.tid) : "memory");
    }
}

// Memory instructions (vm.cpp:238-283, 447-460): off the hot dispatch path.
template <int kM>
__device__ __forceinline__ bool mem_op(const InterpArgs& A, Lane<kM>& L, const uint4 r) {
    const uint32_t op = f_op(r);
    uint2 p;
    if (!L.pointer(f_a(r), p))
        return false;
    const uint2 ix = L.V(f_b(r));
    if (ix.y != GEVO_TAG_I32)
        return L.scalar_fail(f_b(r), ix.y);
    uint2 val = make_uint2(0, 0);
    if (op == GEVO_OP_STORE) {
        if (!L.fetch(f_c(r), val))
            return false;
        if (val.y < GEVO_TAG_I32 || val.y > GEVO_TAG_BOOL)
            return L.trap(GEVO_TRAP_STORE_NONSCALAR);
        if (val.y == GEVO_TAG_BOOL)
            return L.trap(GEVO_TRAP_STORE_BOOL);
    }
    const int64_t eff = static_cast<int64_t>(static_cast<int32_t>(p.x)) +
                        static_cast<int64_t>(static_cast<int32_t>(ix.x));
    if (Lane<kM>::kTP) {
        // Instance memory cells (shared words, then writable global buffers).
        uint32_t w;
        if (p.y == GEVO_TAG_PTR_SHARED) {
            if (eff < 0 || eff >= A.shared_words)
                return L.trap(GEVO_TRAP_SHARED_OOB);
            w = static_cast<uint32_t>(eff);
        } else {
            const uint32_t prm = p.y & 0x3F;
            const uint2 bi = __ldg(L.binfo + prm);
            const uint32_t info = bi.x;
            if (eff < 0 || eff >= static_cast<int32_t>(info >> 8))
                return L.trap(GEVO_TRAP_GLOBAL_OOB);
            const uint32_t elem = info & 0xFF;
            if (op == GEVO_OP_LOAD) {
                if (elem != f_aux(r))
                    return L.trap(GEVO_TRAP_GLOBAL_LOAD_TYPE);
                if (!((L.writable >> prm) & 1ull))
                    return L.set(f_res(r), __ldg(A.pool + bi.y +
                                                 static_cast<uint32_t>(eff) * static_cast<uint32_t>(A.n_tests)),
                                 elem);
            } else {
                if (elem != val.y)
                    return L.trap(GEVO_TRAP_GLOBAL_STORE_TYPE);
                if (!((L.writable >> prm) & 1ull))
                    return L.trap(GEVO_TRAP_INTERNAL);
            }
            w = A.cell_off[prm] + static_cast<uint32_t>(eff);
        }
        if (op == GEVO_OP_LOAD) {
            const uint2 x = L.cell_get(w);
            if (!L.seq)
                tp_note(L, w, false);
            tp_read_check(L, x.y);
            if (p.y == GEVO_TAG_PTR_SHARED) {
                const uint32_t wt = x.y & kCellTag;
                if (wt == GEVO_TAG_UNDEF)
                    return L.trap(GEVO_TRAP_SHARED_UNINIT);
                if (wt != f_aux(r))
                    return L.trap(GEVO_TRAP_SHARED_TYPE);
            }
            return L.set(f_res(r), x.x, x.y & kCellTag);
        }
        if (L.seq) {
            L.cell_put(w, val.x, val.y);
            return true;
        }
        // Same-phase stores of several simulated threads: the highest thread id
        // wins, and a thread's own stores land in program order (the
        // reference runs threads one after another, src/vm.cpp:121-142).
        const uint32_t me = static_cast<uint32_t>(L.tid) + 1;
        const uint32_t meta = cell_meta(val.y, me, L.epoch);
        const unsigned long long want = (static_cast<unsigned long long>(meta) << 32) | val.x;
        const uint2 c0 = L.cell_get(w);
        tp_note(L, w, true);
        unsigned long long cur = (static_cast<unsigned long long>(c0.y) << 32) | c0.x;
        for (;;) {
            const uint32_t m = static_cast<uint32_t>(cur >> 32);
            if ((m >> 16) == L.epoch && cell_writer(m) > me)
                break;
            const unsigned long long prev = L.cell_cas(w, cur, want);
            if (prev == cur)
                break;
            cur = prev;
        }
        return true;
    }
    if (p.y == GEVO_TAG_PTR_SHARED) {
        if (eff < 0 || eff >= A.shared_words)
            return L.trap(GEVO_TRAP_SHARED_OOB);
        const size_t at = static_cast<size_t>(eff) * A.n_inst + L.il;
        if (op == GEVO_OP_LOAD) {
            const uint32_t wt = A.sh_tag[at];
            if (wt == GEVO_TAG_UNDEF)
                return L.trap(GEVO_TRAP_SHARED_UNINIT);
            if (wt != f_aux(r))
                return L.trap(GEVO_TRAP_SHARED_TYPE);
            return L.set(f_res(r), A.sh_val[at], wt);
        }
        A.sh_tag[at] = static_cast<uint8_t>(val.y);
        A.sh_val[at] = val.x;
        return true;
    }
    const uint32_t prm = p.y & 0x3F;
    const uint2 bi = __ldg(L.binfo + prm);
    const uint32_t info = bi.x;
    if (eff < 0 || eff >= static_cast<int32_t>(info >> 8))
        return L.trap(GEVO_TRAP_GLOBAL_OOB);
    const uint32_t elem = info & 0xFF;
    const bool priv = (L.writable >> prm) & 1ull;
    if (op == GEVO_OP_LOAD) {
        if (elem != f_aux(r))
            return L.trap(GEVO_TRAP_GLOBAL_LOAD_TYPE);
        const uint32_t w =
            priv ? A.priv[A.priv_off[prm] + static_cast<size_t>(eff) * A.n_inst + L.il]
                 : __ldg(A.pool + bi.y + static_cast<size_t>(eff) * A.n_tests);
        return L.set(f_res(r), w, elem);
    }
    if (elem != val.y)
        return L.trap(GEVO_TRAP_GLOBAL_STORE_TYPE);
    if (!priv)
        return L.trap(GEVO_TRAP_INTERNAL);
    A.priv[A.priv_off[prm] + static_cast<size_t>(eff) * A.n_inst + L.il] = val.x;
    return true;
}

// Non-arithmetic straight-line instructions (select, getindex, intrinsics, const).
template <int kM>
__device__ __forceinline__ bool misc_op(const InterpArgs& A, Lane<kM>& L, const uint4 r) {
    switch (f_op(r)) {
    case GEVO_OP_SELECT: {
        // both arms are read with the condition (independent shared reads in
        // flight together); the common case completes here, anything else
        // follows the reference order below (it fetches only the chosen arm)
        const uint2 c = L.V(f_a(r)), vb = L.V(f_b(r)), vc = L.V(f_c(r));
        if (c.y == GEVO_TAG_BOOL) {
            const uint2 v = c.x ? vb : vc;
            if (v.y == f_aux(r) && f_res(r) != GEVO_NO_RESULT && !bad_tag(v.y)) {
                L.W(f_res(r), v.x, v.y);
                return true;
            }
        }
        if (c.y != GEVO_TAG_BOOL)
            return L.scalar_fail(f_a(r), c.y);
        uint2 v;
        if (!L.fetch(c.x ? f_b(r) : f_c(r), v))
            return false;
        if (v.y != f_aux(r))
            return L.trap(GEVO_TRAP_SELECT_ARM);
        return L.set(f_res(r), v.x, v.y);
    }
    case GEVO_OP_GETINDEX: {
        {
            const uint2 p = L.V(f_a(r)), ix = L.V(f_b(r));
            if ((p.y == GEVO_TAG_PTR_SHARED || p.y >= static_cast<uint32_t>(GEVO_TAG_PTR_GLOBAL)) &&
                (p.y == GEVO_TAG_PTR_SHARED ? 1u : 0u) == f_aux(r) && ix.y == GEVO_TAG_I32 &&
                f_res(r) != GEVO_NO_RESULT) {
                L.W(f_res(r), p.x + ix.x, p.y);
                return true;
            }
        }
        uint2 p;
        if (!L.pointer(f_a(r), p))
            return false;
        if ((p.y == GEVO_TAG_PTR_SHARED ? 1u : 0u) != f_aux(r))
            return L.trap(GEVO_TRAP_GETINDEX_SPACE);
        const uint2 ix = L.V(f_b(r));
        if (ix.y != GEVO_TAG_I32)
            return L.scalar_fail(f_b(r), ix.y);
        return L.set(f_res(r), p.x + ix.x, p.y);
    }
    case GEVO_OP_TID:
        return L.set(f_res(r), static_cast<uint32_t>(L.tid), GEVO_TAG_I32);
    case GEVO_OP_NTHREADS:
        return L.set(f_res(r), static_cast<uint32_t>(A.threads), GEVO_TAG_I32);
    case GEVO_OP_CONST: {
        const uint2 v = L.V(f_a(r));
        return L.set(f_res(r), v.x, v.y);
    }
    default:
        return L.trap(GEVO_TRAP_UNEXPECTED_OP);
    }
}

// add/sub/mul, fadd/fsub/fmul, icmp, fcmp: the ops of a straight-line
// arithmetic run (one bit test; op < 32 for every record)
__device__ __forceinline__ bool plain_arith(uint32_t op) {
    constexpr uint32_t kMask = (1u << GEVO_OP_ADD) | (1u << GEVO_OP_SUB) | (1u << GEVO_OP_MUL) |
                               (1u << GEVO_OP_FADD) | (1u << GEVO_OP_FSUB) | (1u << GEVO_OP_FMUL) |
                               (1u << GEVO_OP_ICMP) | (1u << GEVO_OP_FCMP);
    return (kMask >> (op & 31u)) & 1u;
}

// One scheduling unit of a simulated thread at pc: a straight-line run of
// plain arithmetic, one other instruction, or a branch with the entry of its
// target block. Returns kStopNone to continue, else the stop kind.
template <int kM>
__device__ __forceinline__ int run_unit(const InterpArgs& A, Lane<kM>& L, Thread& th, Spin& S, Blk& b,
                                        uint32_t& pc, const uint4* code,
                                        const volatile int32_t* first_fail, bool& entered) {
    {
        // (a one-ahead prefetch across units measured slower: the loop-carried
        // copy of the prefetched record waits for the load anyway)
        uint4 r = L.rec(pc);
        uint32_t op = f_op(r);
        if (th.slow || S.mode == 2) {
            // exact per-instruction charging near the budget / abstract iterate
            if (op != GEVO_OP_PHI && op != GEVO_OP_FELL) {
                if (th.slow && !charge_one(A, L, th, f_cls(r))) {
                    th.ip = static_cast<int32_t>(pc - b.start);
                    return kStopTrap;
                }
                if (S.mode == 2 && !spin_track(A, L, r, S))
                    spin_abandon(S, th, L, 0x80 | op);
            }
        }
#ifndef GEVO_NO_ARITH_RUN
        else if (plain_arith(op)) {
            // Straight-line run of plain arithmetic (block-level charging, no
            // abstract iterate): a tight loop in which only pc and the record
            // are live. It stops at the first instruction it does not handle
            // (another opcode, a division, a tag mismatch, a missing result
            // slot), which the general dispatch below then executes.
            for (;;) {
#ifndef GEVO_RUN_BRANCHY
                // next record in flight while this one executes (the sentinel
                // after every block keeps pc + 1 inside the variant)
                const uint4 nx = L.rec(pc + 1);
#endif
                const uint2 x = L.V(f_a(r)), y = L.V(f_b(r));
                const uint32_t otag = f_otag(r);
                const uint32_t res = f_res(r);
                if (x.y != otag || y.y != otag || res == GEVO_NO_RESULT)
                    break;
                const float fx = __uint_as_float(x.x), fy = __uint_as_float(y.x);
                uint32_t v, vt = otag;
                // Branch-free: every cheap result is computed and op selects one
                // (a switch, GEVO_RUN_BRANCHY, measured slower even where the
                // reconvergence gate keeps the opcode warp-uniform)
#ifdef GEVO_RUN_BRANCHY
                constexpr bool kUniformOp = true;
#else
                constexpr bool kUniformOp = false; // (kGC measured 7-10 % slower on configs 3-4)
#endif
                if constexpr (kUniformOp) {
                    switch (op) {
                    case GEVO_OP_ADD: v = x.x + y.x; break;
                    case GEVO_OP_SUB: v = x.x - y.x; break;
                    case GEVO_OP_MUL: v = x.x * y.x; break;
                    case GEVO_OP_FADD: v = __float_as_uint(__fadd_rn(fx, fy)); break;
                    case GEVO_OP_FSUB: v = __float_as_uint(__fsub_rn(fx, fy)); break;
                    case GEVO_OP_FMUL: v = __float_as_uint(__fmul_rn(fx, fy)); break;
                    case GEVO_OP_ICMP:
                        v = cmp(static_cast<int32_t>(x.x), static_cast<int32_t>(y.x), f_aux(r)) ? 1u : 0u;
                        vt = GEVO_TAG_BOOL;
                        break;
                    default: // FCMP
                        v = cmp(fx, fy, f_aux(r)) ? 1u : 0u;
                        vt = GEVO_TAG_BOOL;
                        break;
                    }
                } else {
                    // branch-free: every cheap result is computed and op selects
                    // one; a compare's predicate is a mask over (lt, eq, gt)
                    // plus an invert bit (ne = !eq, true when unordered)
                    const uint32_t o3 = op & 3u; // add/fadd 0, sub/fsub 1, mul/fmul 2
                    const uint32_t vi = selp(o3 == 0, x.x + y.x, selp(o3 == 1, x.x - y.x, x.x * y.x));
                    const uint32_t vf = selp(o3 == 0, __float_as_uint(__fadd_rn(fx, fy)),
                                             selp(o3 == 1, __float_as_uint(__fsub_rn(fx, fy)),
                                                  __float_as_uint(__fmul_rn(fx, fy))));
                    const bool icmp = op == GEVO_OP_ICMP;
                    const int32_t sx = static_cast<int32_t>(x.x), sy = static_cast<int32_t>(y.x);
                    const uint32_t ib = static_cast<uint32_t>(sx < sy) | (static_cast<uint32_t>(sx == sy) << 1) |
                                        (static_cast<uint32_t>(sx > sy) << 2);
                    const uint32_t fb = static_cast<uint32_t>(fx < fy) | (static_cast<uint32_t>(fx == fy) << 1) |
                                        (static_cast<uint32_t>(fx > fy) << 2);
                    const uint32_t bits = selp(icmp, ib, fb);
                    // eq 0x2, ne 0x2|inv, lt 0x1, le 0x3, gt 0x4, ge 0x6 (cmp() order)
                    const uint32_t m = (0x6431A2u >> (f_aux(r) * 4)) & 0xFu;
                    const uint32_t c = static_cast<uint32_t>((bits & m) != 0) ^ (m >> 3);
                    const bool is_cmp = op >= GEVO_OP_ICMP;
                    v = selp(is_cmp, c, selp(op <= GEVO_OP_MUL, vi, vf));
                    vt = selp(is_cmp, static_cast<uint32_t>(GEVO_TAG_BOOL), otag);
                }
                L.W(res, v, vt);
                ++pc;
#ifndef GEVO_RUN_BRANCHY
                r = nx;
#else
                r = L.rec(pc);
#endif
                op = f_op(r);
                if (!plain_arith(op))
                    break;
            }
        }
#endif
        bool ok;
        if (op <= GEVO_OP_FCMP) {
            // i32 / f32 arithmetic and compares: both operands carry otag
            const uint2 x = L.V(f_a(r)), y = L.V(f_b(r));
            const uint32_t otag = f_otag(r);
#ifdef GEVO_ARITH_SELP // branch-free variant (faster in the sequential kernel alone, slower overall)
            if (x.y == otag && y.y == otag && op != GEVO_OP_SDIV && op != GEVO_OP_FDIV) {
                // branch-free: every cheap result is computed, op selects one
                // (selp keeps the compiler from turning the selection back
                // into a compare-and-branch tree)
                const float fx = __uint_as_float(x.x), fy = __uint_as_float(y.x);
                const uint32_t add = x.x + y.x, sub = x.x - y.x, mul = x.x * y.x;
                const uint32_t fad = __float_as_uint(__fadd_rn(fx, fy));
                const uint32_t fsb = __float_as_uint(__fsub_rn(fx, fy));
                const uint32_t fml = __float_as_uint(__fmul_rn(fx, fy));
                // compares with C++ semantics (NaN: only != holds); bit p of
                // `cm` is the outcome of predicate p (eq ne lt le gt ge)
                const bool icmp = op == GEVO_OP_ICMP;
                const bool lt = icmp ? static_cast<int32_t>(x.x) < static_cast<int32_t>(y.x) : fx < fy;
                const bool eq = icmp ? x.x == y.x : fx == fy;
                const bool gt = icmp ? static_cast<int32_t>(x.x) > static_cast<int32_t>(y.x) : fx > fy;
                const uint32_t cm = static_cast<uint32_t>(eq) | (static_cast<uint32_t>(!eq) << 1) |
                                    (static_cast<uint32_t>(lt) << 2) |
                                    (static_cast<uint32_t>(lt || eq) << 3) |
                                    (static_cast<uint32_t>(gt) << 4) |
                                    (static_cast<uint32_t>(gt || eq) << 5);
                const uint32_t c = (cm >> f_aux(r)) & 1u;
                const uint32_t o3 = op & 3u; // add/fadd 0, sub/fsub 1, mul/fmul 2
                const uint32_t vi = selp(o3 == 0, add, selp(o3 == 1, sub, mul));
                const uint32_t vf = selp(o3 == 0, fad, selp(o3 == 1, fsb, fml));
                const bool is_cmp = op >= GEVO_OP_ICMP;
                const uint32_t v = selp(is_cmp, c, selp(op <= GEVO_OP_MUL, vi, vf));
                const uint32_t vt = selp(is_cmp, static_cast<uint32_t>(GEVO_TAG_BOOL), otag);
                const uint32_t res = f_res(r);
                if (res != GEVO_NO_RESULT) {
                    L.W(res, v, vt);
                    ++pc;
                    return kStopNone;
                }
                L.trap(GEVO_TRAP_DEF_NO_ID);
            } else
#endif
            if (x.y == otag && y.y == otag) {
                uint32_t v;
                uint32_t vt = otag;
                ok = true;
                const float fx = __uint_as_float(x.x), fy = __uint_as_float(y.x);
                switch (op) {
                case GEVO_OP_ADD: v = x.x + y.x; break;
                case GEVO_OP_SUB: v = x.x - y.x; break;
                case GEVO_OP_MUL: v = x.x * y.x; break;
                case GEVO_OP_SDIV: {
                    const int32_t sx = static_cast<int32_t>(x.x), sy = static_cast<int32_t>(y.x);
                    if (sy == 0)
                        ok = L.trap(GEVO_TRAP_DIV_ZERO);
                    else if (sx == INT32_MIN && sy == -1)
                        ok = L.trap(GEVO_TRAP_DIV_OVERFLOW);
                    v = ok ? static_cast<uint32_t>(sx / sy) : 0u;
                    break;
                }
                case GEVO_OP_FADD: v = __float_as_uint(__fadd_rn(fx, fy)); break;
                case GEVO_OP_FSUB: v = __float_as_uint(__fsub_rn(fx, fy)); break;
                case GEVO_OP_FMUL: v = __float_as_uint(__fmul_rn(fx, fy)); break;
                case GEVO_OP_FDIV: v = __float_as_uint(__fdiv_rn(fx, fy)); break;
                case GEVO_OP_ICMP:
                    v = cmp(static_cast<int32_t>(x.x), static_cast<int32_t>(y.x), f_aux(r)) ? 1u : 0u;
                    vt = GEVO_TAG_BOOL;
                    break;
                default: // FCMP
                    v = cmp(fx, fy, f_aux(r)) ? 1u : 0u;
                    vt = GEVO_TAG_BOOL;
                    break;
                }
                const uint32_t res = f_res(r);
                if (ok && res != GEVO_NO_RESULT) {
                    L.W(res, v, vt);
                    ++pc;
                    return kStopNone;
                }
                if (ok)
                    L.trap(GEVO_TRAP_DEF_NO_ID);
            } else if (x.y != otag) {
                L.scalar_fail(f_a(r), x.y);
            } else {
                L.scalar_fail(f_b(r), y.y);
            }
            ok = false;
        } else if (op == GEVO_OP_BR) {
            th.ip = static_cast<int32_t>(pc - b.start);
#ifndef GEVO_BR_EDGE_LATE
            // the edge record is in flight while the condition is read
            const uint4 er = L.edge(pc);
#endif
            int32_t target = f_t0(r);
            bool second = false;
            if (f_aux(r) == 2) {
                const uint2 c = L.V(f_a(r));
                if (c.y != GEVO_TAG_BOOL) {
                    L.scalar_fail(f_a(r), c.y);
                    refund(A, L, th, b, th.ip + 1);
                    return kStopTrap;
                }
                second = c.x == 0;
                target = second ? f_t1(r) : f_t0(r);
            }
            refund(A, L, th, b, th.ip + 1);
            if (target < 0) {
                L.trap(GEVO_TRAP_UNKNOWN_BLOCK);
                return kStopTrap;
            }
            if (Lane<kM>::kTP) {
                // a lower simulated thread already stopped the instance
                if (--L.poll <= 0) {
                    L.poll = 16;
                    if (static_cast<int32_t>(lds1(L.msh)) < L.tid)
                        return kStopAbort;
                    // global-cell instances restart from their initial state
                    // after any same-phase conflict: stop the doomed run now
                    // instead of running every thread to the phase end
#ifndef GEVO_NO_CONFLICT_ABORT
                    if (Lane<kM>::kGC && !L.seq && lds1(L.fsh))
                        return kStopAbort;
#endif
                    if (A.early_exit && (++L.poll2 & 127) == 0 &&
                        first_fail[L.v] < static_cast<int32_t>(L.t)) {
                        L.trap(GEVO_SKIPPED);
                        return kStopTrap;
                    }
                }
            } else if (A.early_exit && --L.poll <= 0) {
                L.poll = 2048;
                if (first_fail[L.v] < static_cast<int32_t>(L.t)) {
                    L.trap(GEVO_SKIPPED);
                    return kStopTrap;
                }
            }
#ifdef GEVO_BR_EDGE_LATE
            const uint4 er = L.edge(pc);
#endif
            if (!enter_block(A, L, th, target, b, S,
                             second ? make_uint2(er.z, er.w) : make_uint2(er.x, er.y)))
                return kStopTrap;
            if ((th.executed >= S.next || S.mode != 0) && !th.slow)
                spin_at_entry(A, L, th, S);
            pc = b.start + static_cast<uint32_t>(th.ip);
            // lanes running together stay together through an unconditional
            // branch; only a two-way one may split them (back to the gate)
            entered = f_aux(r) == 2;
            return kStopNone;
        } else if (op == GEVO_OP_LOAD || op == GEVO_OP_STORE) {
#ifndef GEVO_NO_MEM_FAST
            ok = (Lane<kM>::kTP && mem_fast(A, L, r)) || mem_op(A, L, r);
#else
            ok = mem_op(A, L, r);
#endif
        } else if (op == GEVO_OP_SYNC || op == GEVO_OP_RET) {
            th.ip = static_cast<int32_t>(pc - b.start);
            refund(A, L, th, b, th.ip + 1);
            th.bar = f_b(r);
            return op == GEVO_OP_SYNC ? kStopSync : kStopRet;
        } else if (op == GEVO_OP_PHI) {
            th.ip = static_cast<int32_t>(pc - b.start);
            refund(A, L, th, b, th.ip);
            L.trap(GEVO_TRAP_PHI_OUTSIDE);
            return kStopTrap;
        } else if (op == GEVO_OP_FELL) {
            th.ip = static_cast<int32_t>(pc - b.start);
            L.trap(GEVO_TRAP_FELL_OFF);
            return kStopTrap;
        } else {
            ok = misc_op(A, L, r);
        }
        if (!ok) {
            th.ip = static_cast<int32_t>(pc - b.start);
            refund(A, L, th, b, th.ip + 1);
            return kStopTrap;
        }
        ++pc;
        return kStopNone;
    }
}

// run_to_barrier (vm.cpp:340-387) + step (389-482) for one simulated thread
// from (th.block, th.ip). Returns kStopRet, kStopSync or kStopTrap.
//
// Reconvergence: the lanes of a warp that run simulated threads together
// (the same variant) advance in rounds; each round only the lanes at the
// warp's lowest pc run one unit, the others wait. Blocks are laid out in
// program order (loop headers before their bodies), so lanes that split at a
// data-dependent branch meet again at the first block both paths reach, and
// from there issue the same records together instead of serialising
// different opcodes every step. Scheduling does not change any result: each
// lane is an independent simulated thread, and same-phase cross-thread
// interactions are resolved by the timing-independent rules of the
// thread-parallel kernel.
template <int kM>
__device__ __forceinline__ int run_thread(const InterpArgs& A, Lane<kM>& L, Thread& th,
                          const volatile int32_t* first_fail) {
    Spin S;
    S.mode = 0;
    S.skip = 0;
    S.attempts = 0;
    S.next = !A.sp_base ? INT64_MAX : th.spin_next >= 0 ? th.spin_next : A.spin_threshold;
    S.avoid = -1;
    S.K = S.H = 0;
    int64_t bcost;
    Blk b = load_blk(L.dblk, th.block, bcost);
    charge_block(A, L, th, b, bcost, static_cast<uint32_t>(th.ip));
    const uint4* code = reinterpret_cast<const uint4*>(L.code);
    // pc indexes the variant's records; every block is followed by a
    // fell-off sentinel record, and the batch array is padded, so the
    // one-ahead prefetch never leaves it.
    uint32_t pc = b.start + static_cast<uint32_t>(th.ip);
    // When every live lane is at the lead pc the warp is converged and stays
    // so until a branch: it runs units up to the next block entry before the
    // next gate (one gate per block, not per unit, on converged code).
    // Starvation guard: the lowest live thread decides the instance's record
    // when it stops (higher threads are then aborted), so it must not wait
    // behind a lane spinning at lower pcs. When it has not run for 32
    // rounds, the warp follows its pc for the next 256 rounds.
    // Yield test: when over 64 gated rounds fewer than a quarter of the live
    // lanes ran per round, the lanes' paths do not meet (e.g. different loop
    // trip counts, lanes that jumped a spinning loop) and waiting only
    // serialises them: the warp runs ungated for 512 rounds, then retries.
    const bool gate = A.reconv != 0;
    unsigned live = __activemask();
    uint32_t starve = 0, follow = 0, off = 0, rounds = 0, ran = 0;
    for (;;) {
        int stop = kStopNone;
        bool run = true, together = true;
        if (gate && off) {
            --off;
        } else if (gate && (live & (live - 1))) { // (a lone live lane runs ungated)
            const int leader = __ffs(live) - 1;
            const uint32_t lead = follow ? __shfl_sync(live, pc, leader) : __reduce_min_sync(live, pc);
            run = pc == lead;
            const unsigned runs = __ballot_sync(live, run);
            together = runs == live;
            if (follow) {
                --follow;
            } else if ((runs >> leader) & 1u) {
                starve = 0;
            } else if (++starve >= 32) {
                starve = 0;
                follow = 256;
            }
            ran += 4 * __popc(runs) >= __popc(live) ? 1u : 0u;
            if (++rounds == 64) {
                if (ran < 32)
                    off = 512;
                rounds = ran = 0;
            }
        }
        if (run) {
            bool entered = false;
            const bool lone = !(live & (live - 1)); // nothing to meet: run to the stop
            do {
                entered = false;
                stop = run_unit(A, L, th, S, b, pc, code, first_fail, entered);
            } while (together && stop == kStopNone && (!entered || lone));
        }
        if (gate && (live & (live - 1)))
            live = __ballot_sync(live, stop == kStopNone);
        if (stop != kStopNone) {
            // a barrier ended the phase: an attempt in progress counts as a
            // failed one (backoff) and the armed point carries over
            if (stop == kStopSync && A.sp_base)
                th.spin_next = S.mode != 0 ? th.executed + (th.executed >> GEVO_SPIN_BACKOFF) + 64 : S.next;
            return stop;
        }
    }
}

__device__ __forceinline__ uint32_t status_of(uint32_t code) {
    return code == GEVO_BUDGET_EXCEEDED ? GEVO_STATUS_BUDGET
           : code == GEVO_SKIPPED      ? GEVO_STATUS_SKIPPED
                                       : GEVO_STATUS_TRAP;
}

template <int kM>
__device__ __forceinline__ void reset_values(Lane<kM>& L) {
    for (uint32_t s = 0; s < L.n_values; ++s)
        L.W(s, 0, GEVO_TAG_UNDEF);
}

// Machine::run for one instance (src/vm.cpp:114-150). Returns the status.
template <int kM>
__device__ __forceinline__ uint32_t run_instance(const InterpArgs& A, Lane<kM>& L, const gevo_variant& var,
                                 const volatile int32_t* first_fail) {
    const int32_t T = A.threads;
    if (!(var.flags & GEVO_VAR_HAS_SYNC)) {
        // No barrier instruction: every thread runs to ret in phase 0.
        for (int32_t tid = 0; tid < T; ++tid) {
            reset_values(L);
            L.tid = tid;
            Thread th{0, 0, -1, 0, 0, false};
            const int r = run_thread(A, L, th, first_fail);
            if (r == kStopTrap)
                return status_of(L.code_out);
            if (r != kStopRet) {
                L.trap(GEVO_TRAP_INTERNAL);
                return GEVO_STATUS_TRAP;
            }
        }
        return GEVO_STATUS_COMPLETED;
    }

    // Multi-phase: per simulated thread state and values live in scratch.
    const size_t n = A.n_inst;
    for (int32_t tid = 0; tid < T; ++tid) {
        const size_t at = static_cast<size_t>(tid) * n + L.il;
        A.ts_pos[at] = 0;
        A.ts_prev[at] = -1;
        A.ts_exec[at] = 0;
        A.ts_stop[at] = kTsFresh;
    }
    for (;;) {
        bool all_ret = true, all_sync = true;
        uint32_t stop0 = 0;
        for (int32_t tid = 0; tid < T; ++tid) {
            const size_t at = static_cast<size_t>(tid) * n + L.il;
            uint32_t st = A.ts_stop[at];
            if (st != kTsRet) {
                Thread th;
                const int32_t pos = A.ts_pos[at];
                th.block = pos >> 16;
                th.ip = pos & 0xFFFF;
                th.prev = A.ts_prev[at];
                th.executed = A.ts_exec[at];
                th.bar = 0;
                th.slow = false;
                const size_t vbase = static_cast<size_t>(tid) * A.ts_slots;
                if (st == kTsFresh) {
                    reset_values(L);
                } else {
                    for (uint32_t s = 0; s < L.n_values; ++s) {
                        const size_t sv = (vbase + s) * n + L.il;
                        L.W(s, A.ts_val[sv], A.ts_tag[sv]);
                    }
                }
                L.tid = tid;
                const int r = run_thread(A, L, th, first_fail);
                if (r == kStopTrap)
                    return status_of(L.code_out);
                A.ts_pos[at] = (th.block << 16) | th.ip;
                A.ts_prev[at] = th.prev;
                A.ts_exec[at] = th.executed;
                st = r == kStopSync ? (kTsSync | th.bar) : kTsRet;
                A.ts_stop[at] = st;
                if (r == kStopSync) {
                    for (uint32_t s = 0; s < L.n_values; ++s) {
                        const size_t sv = (vbase + s) * n + L.il;
                        const uint2 v = L.V(s);
                        A.ts_tag[sv] = static_cast<uint8_t>(v.y);
                        A.ts_val[sv] = v.x;
                    }
                }
            }
            if (tid == 0)
                stop0 = st;
            if (st != kTsRet)
                all_ret = false;
            if ((st & 0xFFFF0000u) != kTsSync || st != stop0)
                all_sync = false;
        }
        if (all_ret)
            return GEVO_STATUS_COMPLETED;
        if (!all_sync) {
            L.trap(GEVO_TRAP_DIVERGENCE);
            return GEVO_STATUS_TRAP;
        }
        for (int32_t tid = 0; tid < T; ++tid) {
            const size_t at = static_cast<size_t>(tid) * n + L.il;
            A.ts_stop[at] = kTsResume;
            A.ts_pos[at] += 1; // step past the barrier
        }
    }
}

// Error metric of one completed instance (compute_error, src/vm.cpp:536-556):
// 1.0 on any structural mismatch (resolved on the host per test), else the max
// over oracle elements of the clamped relative difference. max() is exact and
// order-free, so the per-buffer early return of the reference is not needed.
template <int kM>
__device__ __forceinline__ double instance_error(const InterpArgs& A, const Lane<kM>& L) {
    if (A.static_err[L.t])
        return 1.0;
    const uint32_t nt = static_cast<uint32_t>(A.n_tests);
    double worst = 0.0;
    for (int32_t e = A.entry_begin[L.t]; e < A.entry_begin[L.t + 1]; ++e) {
        const OracleEntryDev en = A.entries[e];
        const uint32_t p = static_cast<uint32_t>(en.param);
        const bool priv = (L.writable >> p) & 1ull;
        for (int32_t k = 0; k < en.size; ++k) {
            const uint32_t cw =
                priv ? A.priv[A.priv_off[p] + static_cast<size_t>(k) * A.n_inst + L.il]
                     : __ldg(A.pool + A.pool_off[p] + static_cast<size_t>(k) * nt + L.t);
            const uint32_t ow = __ldg(A.pool + en.off + static_cast<size_t>(k) * nt + L.t);
            const double d = rel_diff(word_to_double(cw, en.elem), word_to_double(ow, en.elem));
            worst = (worst < d) ? d : worst;
        }
        if (worst >= 1.0)
            return 1.0;
    }
    return worst;
}

} // namespace

template <int kM>
__global__ void __launch_bounds__(128) interp_kernel(const __grid_constant__ InterpArgs A) {
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + warp;
    const uint32_t vl = gw / A.warps_per_variant; // variant, local to the launch
    const uint32_t t = (gw % A.warps_per_variant) * 32 + lane;
    if (vl >= A.n_var || t >= static_cast<uint32_t>(A.n_tests))
        return;
    const uint32_t v = A.v_begin + vl;
    const uint32_t nt = static_cast<uint32_t>(A.n_tests);
    const uint32_t il = vl * nt + t;
    const uint64_t gi = static_cast<uint64_t>(v) * nt + t;

    Lane<kM> L;
    L.v = v;
    L.t = t;
    L.il = il;
    L.sl = il;
    L.seq = true;
    L.binfo = A.buf_info + static_cast<size_t>(t) * A.n_params;
    if (Lane<kM>::kSmem) {
        L.gvf = nullptr;
        L.base = warp * A.row_lanes * A.max_slots + (lane & (A.row_lanes - 1));
        L.row = A.row_lanes;
        L.vsh = smem_addr(g_vfs) + L.base * 8;
        L.vstr = A.row_lanes * 8;
    } else {
        L.gvf = A.vf;
        L.base = il;
        L.row = A.n_inst;
    }
    L.cost = 0;
    L.ir = 0;
    L.work = 0;
    L.poll = 2048;
    L.jumps = 0;
    L.spin_dbg = 0;
    L.code_out = GEVO_OK;
    L.aux = 0;
    L.writable = 0;
    L.tid = 0;

    const volatile int32_t* first_fail = A.first_fail;
    uint32_t status;
    double error = -1.0;
    const uint8_t setup = A.setup_code[t];
    if (A.early_exit && first_fail[v] < static_cast<int32_t>(t)) {
        L.code_out = GEVO_SKIPPED;
        status = GEVO_STATUS_SKIPPED;
    } else if (setup != GEVO_OK) {
        // Machine ctor failure: trap with cost 0 (src/vm.cpp:516-520).
        L.code_out = setup;
        L.aux = A.setup_aux[t];
        status = GEVO_STATUS_TRAP;
    } else {
        const gevo_variant var = A.variants[v];
        const uint32_t P = static_cast<uint32_t>(A.n_params);
        L.code = A.insts + var.inst_base;
        L.suffix = A.suffix ? A.suffix + var.inst_base : nullptr;
        L.edges = A.edges + var.inst_base;
        L.dblk = A.dblocks + var.block_base;
        L.arm = A.arms + var.arm_base;
        L.n_values = var.n_values;
        L.n_slots = var.n_slots;
        L.writable = var.writable;
        const uint32_t lit_begin = var.n_values + P + 2;
        L.stage_base = lit_begin + var.n_lits;

        // Parameters (bound per test), poison slots, literal pool.
        const size_t tp0 = static_cast<size_t>(t) * P;
        for (uint32_t p = 0; p < P; ++p)
            L.W(var.n_values + p, A.param_payload[tp0 + p], A.param_tag[tp0 + p]);
        L.W(var.n_values + P, 0, GEVO_TAG_POISON_PARAM);
        L.W(var.n_values + P + 1, 0, GEVO_TAG_POISON_MISSING);
        for (uint32_t k = 0; k < var.n_lits; ++k)
            L.W(lit_begin + k, __ldg(A.lit_payload + var.lit_base + k),
                __ldg(A.lit_tag + var.lit_base + k));
        // Private copies of the buffers this variant may store to
        // (Machine ctor copies every global buffer, src/vm.cpp:96-97; read-only
        // ones are served from the shared test pool).
        for (uint64_t m = var.writable; m; m &= m - 1) {
            const uint32_t p = static_cast<uint32_t>(__ffsll(static_cast<long long>(m)) - 1);
            const int32_t rows = A.buf_size[tp0 + p];
            for (int32_t e = 0; e < rows; ++e)
                A.priv[A.priv_off[p] + static_cast<size_t>(e) * A.n_inst + il] =
                    __ldg(A.pool + A.pool_off[p] + static_cast<size_t>(e) * nt + t);
        }
        for (int32_t w = 0; w < A.shared_words; ++w)
            A.sh_tag[static_cast<size_t>(w) * A.n_inst + il] = GEVO_TAG_UNDEF;

        status = run_instance(A, L, var, first_fail);
        if (status == GEVO_STATUS_COMPLETED)
            error = instance_error(A, L);
    }

    gevo_test_record rec;
    rec.cost = L.cost;
    rec.ir = L.ir;
    rec.error = error;
    rec.aux = L.aux;
    rec.status = static_cast<uint8_t>(status);
    rec.code = static_cast<uint8_t>(L.code_out);
    rec.pad[0] = static_cast<uint8_t>(L.jumps);
    rec.pad[1] = static_cast<uint8_t>(L.spin_dbg);
    A.rec[gi] = rec;
    if (A.counters && L.work)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 4),
                  static_cast<unsigned long long>(L.work));

    if (A.early_exit && status != GEVO_STATUS_SKIPPED &&
        (status != GEVO_STATUS_COMPLETED || error > A.tolerance))
        atomicMin(A.first_fail + v, static_cast<int32_t>(t));
}

// Interpreted-instruction counter (counters[4]): one atomic per warp.
__device__ __forceinline__ void add_work(const InterpArgs& A, uint32_t work) {
    unsigned long long w = work;
    for (int o = 16; o; o >>= 1)
        w += __shfl_xor_sync(0xffffffffu, w, o);
    if (A.counters && (threadIdx.x & 31) == 0 && w)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 4), w);
}

// ---- thread-parallel interpreter ---------------------------------------------
//
// interp_tp_kernel runs the simulated threads of an instance concurrently. A
// CTA holds one variant and Ln consecutive tests; lane l of warp w runs
// simulated thread tid = w * K + l / Ln of test l % Ln (K = 32 / Ln threads per
// warp). With many tests (the corpus: 8 threads, 16 tests) a warp covers few
// threads of many tests, whose lanes follow the same path; with many threads
// and few tests (data-parallel kernels) a warp covers consecutive threads of
// one test. The instance's mutable memory -- simulated shared words and its
// private copies of writable global buffers -- lives in shared-memory cells
// {payload, tag | writer << 8 | epoch << 16}, one column per test.
//
// Exactness. Within a phase (the stretch between two barriers) the reference
// runs threads in id order (src/vm.cpp:121-142), so thread t sees every write
// of threads < t and none of threads > t. Running them concurrently gives the
// same result whenever no word is read by one thread and written by another in
// the same phase: every read then returns the phase-start value or the
// reader's own write. Words only written by several threads (nw-sync's s[80])
// keep the value of the highest writer -- each store is a compare-and-swap
// that never overwrites a higher writer of the current epoch, and a thread's
// own stores land in program order. Every thread records the words it read and
// wrote in per-phase bitsets; at the phase end R_t & (W of any other thread)
// is checked, and any hit discards the concurrent run of that instance and
// re-executes it from the start with its threads in id order (the reference
// schedule, plain stores).
//
// Stops. The lowest thread id that traps (or exceeds its budget) decides the
// record, as in the reference, where higher threads never run after it: the
// cost and dynamic IR of threads above it in that phase are dropped, and those
// threads abandon their run early (min_stop poll). Barrier divergence is
// judged on all threads once none trapped (vm.cpp:123-137).

namespace {

enum : uint32_t { kInstPar = 0, kInstSeq = 1, kInstDone = 2 };
constexpr uint32_t kStickySeq = 2;
enum : uint32_t { kActContinue = 0, kActFinish = 1, kActRestart = 2, kActNone = 3 };

// Per-CTA scratch regions (InterpArgs::regions): a ring of free region ids
// with generation tags. Ticket k of the acquire counter takes ring entry
// k % R once its generation is k / R, i.e. after release k - R returned a
// region there; at most R CTAs are resident, so that release has been
// ticketed when ticket k is drawn and the wait is short.
__device__ uint32_t region_acquire(const InterpArgs& A) {
    const uint32_t k = atomicAdd(A.region_ctr, 1u);
    const uint32_t R = A.regions, at = k % R, gen = (k / R) & 0xFFFFu;
    const volatile uint32_t* q = A.region_q;
    for (;;) {
        const uint32_t e = q[at];
        if ((e >> 16) == gen)
            return e & 0xFFFFu;
        __nanosleep(64);
    }
}

__device__ void region_release(const InterpArgs& A, uint32_t region) {
    __threadfence(); // the CTA's scratch writes precede the hand-over
    const uint32_t k = atomicAdd(A.region_ctr + 1, 1u);
    const uint32_t R = A.regions, at = k % R, gen = ((k / R) + 1) & 0xFFFFu;
    *reinterpret_cast<volatile uint32_t*>(A.region_q + at) = region | (gen << 16);
}

__global__ void region_init_kernel(uint32_t* q, uint32_t* ctr, uint32_t R) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < R; i += gridDim.x * blockDim.x)
        q[i] = i; // generation 0
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr[0] = 0;
        ctr[1] = 0;
    }
}

struct TpInst {
    unsigned long long stage_bar; // mbarrier of the record staging copy
    uint32_t region;
    int32_t min_stop[32];
    uint32_t state[32];
    uint32_t conflict[32];
    uint32_t nconf[32]; // phases of the instance re-run after a conflict
    int32_t tstar[32];  // lowest thread whose reads overlapped another thread's writes
    int32_t seqfrom[32];// re-run: threads below run concurrently, the rest in id order
    uint32_t status[32];
    uint32_t code[32];
    int32_t aux[32];
    unsigned long long cost[32];
    unsigned long long ir[32];
    uint32_t jumps[32];
};

struct TpGeom {
    uint32_t T, Ln, K;
    // CTA-lane of simulated thread `tid` of test column j
    __device__ __forceinline__ uint32_t lane_of(uint32_t tid, uint32_t j) const {
        return (tid / K) * 32 + (tid % K) * Ln + j;
    }
};

// Instance memory cells from the test's inputs; thread tid fills words
// tid, tid + T, ...
template <int kM>
__device__ __forceinline__ void tp_init_cells(const InterpArgs& A, const Lane<kM>& L, uint32_t tid,
                                              uint32_t T) {
    if (Lane<kM>::kGC && A.regions)
        // a reused region: clear the access records of the previous CTA
        for (uint32_t w = tid; w < A.n_cells; w += T)
            L.gshadow[static_cast<size_t>(w) * L.gstr] = 0ull;
    const uint32_t SW = static_cast<uint32_t>(max(A.shared_words, 0));
    for (uint32_t w = tid; w < SW; w += T)
        L.cell_put(w, 0, GEVO_TAG_UNDEF);
    const size_t tp0 = static_cast<size_t>(L.t) * A.n_params;
    for (uint64_t m = L.writable; m; m &= m - 1) {
        const uint32_t p = static_cast<uint32_t>(__ffsll(static_cast<long long>(m)) - 1);
        const int32_t rows = A.buf_size[tp0 + p];
        const uint32_t elem = A.buf_elem[tp0 + p];
        for (int32_t e = static_cast<int32_t>(tid); e < rows; e += static_cast<int32_t>(T))
            L.cell_put(A.cell_off[p] + static_cast<uint32_t>(e),
                       __ldg(A.pool + A.pool_off[p] + static_cast<size_t>(e) * A.n_tests + L.t), elem);
    }
}

template <int kM>
__device__ __forceinline__ void tp_reset_thread(Lane<kM>& L, Thread& th) {
    for (uint32_t s = 0; s < L.n_values; ++s)
        L.W(s, 0, GEVO_TAG_UNDEF);
    L.cost = 0;
    L.ir = 0;
    L.code_out = GEVO_OK;
    L.aux = 0;
    th = Thread{0, 0, -1, 0, 0, false};
}

} // namespace

template <int kM>
#ifdef GEVO_TP_MAXNREG // register cap (occupancy experiments)
#define GEVO_TP_BOUNDS __maxnreg__(GEVO_TP_MAXNREG)
#else
#define GEVO_TP_BOUNDS __launch_bounds__(kTpMaxBlock, 1)
#endif
__device__ __forceinline__ void tp_item(const InterpArgs& A, TpInst& S, uint32_t item,
                                        uint32_t fixed_region) {
    constexpr bool kGC = kM == 3; // instance memory in global cells
    TpGeom G;
    G.T = static_cast<uint32_t>(A.threads);
    G.Ln = A.tp_lanes;
    G.K = 32 / G.Ln;
    const uint32_t T = G.T, Ln = G.Ln;
    const uint32_t w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const uint32_t sub = l / Ln, j = l % Ln;
    const uint32_t tid = w * G.K + sub;
    const bool lane_ok = sub < G.K && tid < T;

    const uint32_t nt = static_cast<uint32_t>(A.n_tests);
    // test groups major: every variant's first tests are scheduled before any
    // later ones, so the early-exit protocol (first_fail) can skip the tests
    // the reference never runs after a failure
    const uint32_t vl = item % A.n_var;
    const uint32_t tg = item / A.n_var;
    const uint32_t t = tg * Ln + j;
    const uint32_t v = A.v_begin + vl;
    const bool inst_ok = t < nt;
    const bool active = lane_ok && inst_ok;
    const bool leader = lane_ok && tid == 0;
    const uint64_t gi = static_cast<uint64_t>(v) * nt + t;

    // dynamic shared memory: value files | param table | literal table | cells |
    // R,W bitsets | per (thread, test)
    const uint32_t warps = blockDim.x >> 5;
    const uint32_t sbase = smem_addr(g_vfs);
    const uint32_t P = static_cast<uint32_t>(A.n_params);
    const uint32_t lane_slots = kTpTables ? A.lane_slots : A.max_slots;
    // compact lane files: [warp][slot][lane] payload words, then tag bytes
    const uint32_t vf_bytes = Lane<kM>::kCompact ? (warps * 32 * lane_slots * 5 + 7) & ~7u
                                                 : warps * 32 * lane_slots * 8;
    const uint32_t tab0 = sbase + vf_bytes;
    const uint32_t lit0 = tab0 + Ln * (P + 2) * 8;
    const uint32_t cell0 = lit0 + A.max_lits * 8;
    const uint32_t smem_cells = kGC ? 0 : A.n_cells;
    const uint32_t back0 = cell0 + Ln * smem_cells * 8; // phase-start copy of the cells
    const uint32_t bits0 = back0 + (A.tp_snap ? Ln * smem_cells * 8 : 0);
    const uint32_t bit_words = kGC ? 0 : A.n_chunks * blockDim.x;
    const uint32_t Q = T * Ln;
    const uint32_t pq0 = bits0 + 2 * bit_words * 4;  // kind | bar | tcode | taux (u32 x Q)
    const uint32_t err0 = (pq0 + 4 * Q * 4 + 7) & ~7u; // err (double x Q)
    const uint32_t stage0 = (err0 + Q * 8 + 15) & ~15u;  // staged records: code | edges
    const uint32_t q = tid * Ln + j;

    Lane<kM> L;
    L.gvf = nullptr;
    // (vsh goes through an opaque move: rematerialising it from the thread
    // index and the slot count at every value-file access cost ~9 SASS per IR)
    if (Lane<kM>::kCompact) {
        L.vsh = opaque(sbase + (w * 32 * lane_slots + l) * 4);
        L.vstr = 32 * 4;
        // tag array [warp][slot][lane] bytes after the payload words: the tag of
        // the word at a is at tag0 + (a - sbase) / 4
        L.gsh = sbase + warps * 32 * lane_slots * 4 - (sbase >> 2);
    } else {
        L.vsh = opaque(sbase + (w * 32 * lane_slots + l) * 8);
        L.vstr = 32 * 8;
        L.gsh = 0;
    }
    L.tsh = tab0 + j * 8;
    L.tstr = Ln * 8;
    L.lsh = lit0;
    L.base = 0;
    L.row = 0;
    L.v = v;
    L.t = inst_ok ? t : 0;
    L.il = item * 32 + j;
    L.sl = item * blockDim.x + threadIdx.x;
    L.tid = static_cast<int32_t>(tid);
    L.binfo = A.buf_info + static_cast<size_t>(L.t) * A.n_params;
    L.csh = cell0 + j * 8;
    L.cstr = Ln * 8;
    L.rsh = bits0 + threadIdx.x * 4;
    L.wsh = L.rsh + bit_words * 4;
    L.bstr = blockDim.x * 4;
    L.msh = smem_addr(S.min_stop + j);
    L.fsh = smem_addr(S.conflict + j);
    L.tsh_star = smem_addr(S.tstar + j);
    const uint32_t il = vl * nt + t; // launch-local instance (global cells)
    L.gcell = kGC ? A.gcells + il : nullptr;
    L.gshadow = kGC ? A.gshadow + il : nullptr;
    L.gstr = A.n_inst;
    L.epoch = 0;
    L.seq = false;
    L.cost = 0;
    L.ir = 0;
    L.work = 0;
    L.poll = 16;
    L.poll2 = 0;
    L.jumps = 0;
    L.spin_dbg = 0;
    L.code_out = GEVO_OK;
    L.aux = 0;
    L.writable = 0;
    L.n_values = 0;

    const volatile int32_t* first_fail = A.first_fail;
    unsigned long long clk0 = 0;
    if (A.cta_clock && threadIdx.x == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk0));
    if (threadIdx.x < 32) {
        const uint32_t c = threadIdx.x; // instance column
        const uint32_t tc = tg * Ln + c;
        S.cost[c] = 0;
        S.ir[c] = 0;
        S.jumps[c] = 0;
        S.nconf[c] = 0;
        S.seqfrom[c] = 0;
        S.aux[c] = 0;
        S.code[c] = GEVO_OK;
        if (c >= Ln || tc >= nt) {
            S.state[c] = kInstDone;
            S.status[c] = GEVO_STATUS_SKIPPED;
        } else if (A.early_exit && first_fail[v] < static_cast<int32_t>(tc)) {
            S.state[c] = kInstDone;
            S.status[c] = GEVO_STATUS_SKIPPED;
            S.code[c] = GEVO_SKIPPED;
        } else if (A.setup_code[tc] != GEVO_OK) {
            // Machine ctor failure: trap with cost 0 (src/vm.cpp:516-520).
            S.state[c] = kInstDone;
            S.status[c] = GEVO_STATUS_TRAP;
            S.code[c] = A.setup_code[tc];
            S.aux[c] = A.setup_aux[tc];
        } else {
            S.state[c] = kInstPar;
        }
    }
    __syncthreads();
    if (A.regions) {
        // this CTA's scratch columns (global cells + access records, spin and
        // snapshot state): a free region, when any of its instances runs
        if (threadIdx.x == 0) {
            bool any = false;
            for (uint32_t c = 0; c < Ln; ++c)
                any |= S.state[c] != kInstDone;
            // (a persistent CTA owns its region)
            S.region = !any ? 0xFFFFFFFFu : fixed_region != 0xFFFFFFFFu ? fixed_region : region_acquire(A);
        }
        __syncthreads();
        const uint32_t rg = S.region;
        if (rg != 0xFFFFFFFFu) {
            // a region holds its instances' cells contiguously, [cell][test]:
            // consecutive threads touching consecutive words coalesce
            const size_t base = static_cast<size_t>(rg) * A.n_cells * Ln + j;
            L.gcell = kGC ? A.gcells + base : nullptr;
            L.gshadow = kGC ? A.gshadow + base : nullptr;
            L.gstr = Ln;
            L.sl = rg * blockDim.x + threadIdx.x;
        }
    }

    const gevo_variant var = A.variants[v];
    // Stage the variant's instruction and branch-edge records in shared memory
    // with two TMA bulk copies (one elected thread, an mbarrier counting the
    // bytes); the interpreter then fetches every record with ld.shared.
    uint32_t n_recs = 0;
    if (A.stage_recs && __syncthreads_or(S.state[j] != kInstDone && active)) {
        const uint32_t end = v + 1 < A.v_begin + A.n_var ? A.variants[v + 1].inst_base : A.n_insts_total;
        n_recs = min(end - var.inst_base, A.stage_recs);
        const uint32_t bar = smem_addr(&S.stage_bar);
        if (threadIdx.x == 0) {
            const uint32_t bytes = n_recs * 16;
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(2 * bytes)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(stage0), "l"(A.insts + var.inst_base), "r"(bytes), "r"(bar)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(stage0 + A.stage_recs * 16), "l"(A.edges + var.inst_base), "r"(bytes), "r"(bar)
                         : "memory");
        }
    }
    // CTA-shared tables: the variant's literals, each test's parameters
    for (uint32_t k = threadIdx.x; k < var.n_lits; k += blockDim.x)
        sts2(lit0 + k * 8, __ldg(A.lit_payload + var.lit_base + k), __ldg(A.lit_tag + var.lit_base + k));
    Thread th{0, 0, -1, 0, 0, false};
    Thread th_snap = th;
    int64_t cost_commit = 0, ir_commit = 0;
    bool first_phase = true; // of this instance: a conflict re-runs from the initial state
    const bool snap = A.tp_snap && (var.flags & GEVO_VAR_HAS_SYNC);
    if (active && S.state[j] != kInstDone) {
        L.code = A.insts + var.inst_base;
        L.suffix = A.suffix ? A.suffix + var.inst_base : nullptr;
        L.edges = A.edges + var.inst_base;
        if constexpr (Lane<kM>::kGC) {
            L.rp = reinterpret_cast<const uint4*>(L.code);
            L.ep = reinterpret_cast<const uint4*>(L.edges);
        }
        L.dblk = A.dblocks + var.block_base;
        L.arm = A.arms + var.arm_base;
        L.n_values = var.n_values;
        L.n_slots = var.n_slots;
        L.writable = var.writable;
        L.nv = var.n_values;
        L.lit_begin = var.n_values + P + 2;
        L.stage_base = L.lit_begin + var.n_lits;
        if (!kTpTables)
            for (uint32_t k = 0; k < var.n_lits; ++k)
                L.W(L.lit_begin + k, __ldg(A.lit_payload + var.lit_base + k),
                    __ldg(A.lit_tag + var.lit_base + k));
        if (tid == 0 || !kTpTables) {
            const size_t tp0 = static_cast<size_t>(t) * P;
            for (uint32_t p = 0; p < P; ++p)
                L.W(var.n_values + p, A.param_payload[tp0 + p], A.param_tag[tp0 + p]);
            L.W(var.n_values + P, 0, GEVO_TAG_POISON_PARAM);
            L.W(var.n_values + P + 1, 0, GEVO_TAG_POISON_MISSING);
        }
        tp_reset_thread(L, th);
        tp_init_cells(A, L, tid, T);
    }

    if (n_recs) {
        __syncthreads(); // the barrier is initialised before anyone waits on it
        const uint32_t bar = smem_addr(&S.stage_bar);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                         : "=r"(done)
                         : "r"(bar)
                         : "memory");
        if constexpr (Lane<kM>::kGC) {
            const char* g0 = reinterpret_cast<const char*>(g_vfs) + (stage0 - sbase); // generic
            L.rp = reinterpret_cast<const uint4*>(g0);
            L.ep = reinterpret_cast<const uint4*>(g0 + A.stage_recs * 16);
        }
    }
    for (;;) { // phases, CTA-uniform
        ++L.epoch;
        const uint32_t st = active ? S.state[j] : kInstDone;
        if (st == kInstPar) {
            if (!kGC)
                for (uint32_t k = 0; k < A.n_chunks; ++k) {
                    sts1(L.rsh + k * L.bstr, 0);
                    sts1(L.wsh + k * L.bstr, 0);
                }
            if (!kGC && snap && !first_phase) {
                // phase-start state, restored if this phase must run in id order
                th_snap = th;
                for (uint32_t x = 0; x < L.n_values; ++x)
                    A.tp_snap[static_cast<size_t>(x) * A.n_spin + L.sl] = L.V(x);
                for (uint32_t x = tid; x < A.n_cells; x += T) {
                    const uint2 c = lds2(L.cell(x));
                    sts2(back0 + (x * Ln + j) * 8, c.x, c.y);
                }
            }
        }
        if (leader) {
            S.min_stop[j] = INT32_MAX;
            S.conflict[j] = 0;
            S.tstar[j] = INT32_MAX;
        }
        __syncthreads();
        int kind = kStopIdle;
        // round 0 runs the concurrent instances; when some instance follows the
        // reference schedule, rounds 1..T run its threads one after another,
        // stopping at the first trap (one run_thread call site: inlined)
        const bool any_seq = __syncthreads_or(st == kInstSeq);
        const uint32_t rounds = any_seq ? T + 1 : 1;
        for (uint32_t u = 0; u < rounds; ++u) {
            // a re-run phase first repeats its conflict-free prefix (threads
            // below seqfrom: none of them read a word another thread wrote, so
            // concurrently they reproduce their reference results) and then
            // runs the remaining threads one after another
            const bool go = u == 0 ? (st == kInstPar ||
                                      (st == kInstSeq && static_cast<int32_t>(tid) < S.seqfrom[j]))
                                   : (st == kInstSeq && tid == u - 1 &&
                                      static_cast<int32_t>(tid) >= S.seqfrom[j] &&
                                      S.min_stop[j] == INT32_MAX);
            if (go) {
                L.seq = u != 0;
                kind = run_thread(A, L, th, first_fail);
                if (kind == kStopTrap) {
                    if (u == 0)
                        atomicMin(S.min_stop + j, static_cast<int32_t>(tid));
                    else
                        S.min_stop[j] = static_cast<int32_t>(tid);
                }
            }
            if (any_seq)
                __syncthreads();
        }
        if (lane_ok) {
            sts1(pq0 + q * 4, static_cast<uint32_t>(kind));
            sts1(pq0 + (Q + q) * 4, th.bar);
            sts1(pq0 + (2 * Q + q) * 4, L.code_out);
            sts1(pq0 + (3 * Q + q) * 4, static_cast<uint32_t>(L.aux));
        }
        __syncthreads();
        if (!kGC && st == kInstPar) {
            // Words this thread read that another thread wrote in the phase.
            // Written by a LOWER thread: the reference shows that write, so
            // the phase conflicts. Written only by higher threads: the reads
            // saw phase-start values (a higher thread's write, had it been
            // seen, was flagged by tp_read_check) -- no conflict, but the
            // thread is then not part of a re-run's conflict-free prefix.
            uint32_t lo = 0, hi = 0;
            for (uint32_t k = 0; k < A.n_chunks && !lo; ++k) {
                const uint32_t r = lds1(L.rsh + k * L.bstr);
                if (!r)
                    continue;
                const uint32_t wk = bits0 + (bit_words + k * blockDim.x) * 4;
                for (uint32_t u = 0; u < T; ++u) {
                    const uint32_t o = r & lds1(wk + G.lane_of(u, j) * 4);
                    lo |= u < tid ? o : 0u;
                    hi |= u > tid ? o : 0u;
                }
            }
            if (lo)
                S.conflict[j] = 1;
            if (lo | hi)
                atomicMin(S.tstar + j, static_cast<int32_t>(tid));
        }
        __syncthreads();
        // Phase verdict of instance j (every thread of it derives the same one).
        uint32_t act = kActNone, ts = T, status = 0;
        if (st != kInstDone) {
            act = kActContinue;
            if (S.conflict[j] || (st == kInstPar && L.epoch >= 0xFFFFu)) {
                act = kActRestart;
            } else {
                for (uint32_t u = 0; u < T; ++u)
                    if (lds1(pq0 + (u * Ln + j) * 4) == kStopTrap) {
                        ts = u;
                        break;
                    }
                if (ts < T) {
                    act = kActFinish;
                    const uint32_t c = lds1(pq0 + (2 * Q + ts * Ln + j) * 4);
                    status = c == GEVO_BUDGET_EXCEEDED ? GEVO_STATUS_BUDGET
                             : c == GEVO_SKIPPED      ? GEVO_STATUS_SKIPPED
                                                      : GEVO_STATUS_TRAP;
                } else {
                    bool all_ret = true, same = true;
                    const uint32_t b0 = lds1(pq0 + (Q + j) * 4);
                    for (uint32_t u = 0; u < T; ++u) {
                        const uint32_t k = lds1(pq0 + (u * Ln + j) * 4);
                        all_ret &= k == kStopRet;
                        same &= k == kStopSync && lds1(pq0 + (Q + u * Ln + j) * 4) == b0;
                    }
                    if (all_ret) {
                        act = kActFinish;
                        status = GEVO_STATUS_COMPLETED;
                    } else if (!same) {
                        act = kActFinish;
                        status = GEVO_STATUS_TRAP;
                        ts = T + 1; // divergence
                    }
                }
            }
        }
        __syncthreads(); // verdict inputs read; shared state may change now
        if (act == kActRestart) {
            if (A.counters && leader)
                atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 2), 1ull);
            if (first_phase || kGC) {
                tp_reset_thread(L, th);
                tp_init_cells(A, L, tid, T);
                cost_commit = ir_commit = 0;
            } else {
                // back to the phase start (snap is set: only multi-phase variants get here)
                th = th_snap;
                for (uint32_t x = 0; x < L.n_values; ++x) {
                    const uint2 sv = A.tp_snap[static_cast<size_t>(x) * A.n_spin + L.sl];
                    L.W(x, sv.x, sv.y);
                }
                for (uint32_t x = tid; x < A.n_cells; x += T) {
                    const uint2 c = lds2(back0 + (x * Ln + j) * 8);
                    sts2(L.cell(x), c.x, c.y);
                }
                L.cost = cost_commit;
                L.ir = ir_commit;
                L.code_out = GEVO_OK;
                L.aux = 0;
            }
            if (leader) {
                S.state[j] = kInstSeq;
                ++S.nconf[j];
                // global-cell instances restart from their initial state (not
                // the conflicting phase's start) and learn of conflicts at the
                // access: fully in id order
                // (and a multi-phase instance without a snapshot would restart
                // from phase 0, where the prefix bound does not apply)
                S.seqfrom[j] = (kGC || S.tstar[j] == INT32_MAX ||
                                (!snap && (var.flags & GEVO_VAR_HAS_SYNC)))
                                   ? 0
                                   : S.tstar[j];
            }
        } else if (act == kActFinish) {
            const bool mine = ts >= T || tid <= ts;
            atomicAdd(S.cost + j, static_cast<unsigned long long>(mine ? L.cost : cost_commit));
            atomicAdd(S.ir + j, static_cast<unsigned long long>(mine ? L.ir : ir_commit));
            atomicAdd(S.jumps + j, L.jumps);
            if (leader) {
                S.state[j] = kInstDone;
                S.status[j] = status;
                if (ts < T) {
                    S.code[j] = lds1(pq0 + (2 * Q + ts * Ln + j) * 4);
                    S.aux[j] = static_cast<int32_t>(lds1(pq0 + (3 * Q + ts * Ln + j) * 4));
                } else if (ts == T + 1) {
                    S.code[j] = GEVO_TRAP_DIVERGENCE;
                    S.aux[j] = 0;
                } else {
                    S.code[j] = GEVO_OK;
                    S.aux[j] = 0;
                }
            }
        } else if (act == kActContinue) {
            ++th.ip; // step past the barrier
            cost_commit = L.cost;
            ir_commit = L.ir;
            // the next phase runs concurrently again (a single-phase variant
            // never continues; a re-run phase 0 has no snapshot to return to),
            // unless the instance keeps conflicting: after kStickySeq re-runs
            // its remaining phases go straight to thread-id order (typically a
            // barrier inside a loop whose every iteration conflicts), saving
            // the discarded concurrent attempt and its snapshot
            if (snap) {
                first_phase = false;
                if (leader)
                    S.state[j] = S.nconf[j] >= kStickySeq ? kInstSeq : kInstPar;
                if (leader)
                    S.seqfrom[j] = 0;
            }
        }
        if (__syncthreads_and(!active || S.state[j] == kInstDone))
            break;
    }

    if (A.cta_clock && threadIdx.x == 0) {
        unsigned long long clk1;
        uint32_t smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(clk1));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* c = A.cta_clock + (static_cast<size_t>(v) * nt + tg * Ln) * 4;
        c[0] = clk0;
        c[1] = clk1;
        c[2] = smid;
        c[3] = S.ir[0];
    }
    // compute_error (src/vm.cpp:536-556) of completed instances: max over
    // oracle elements, spread over the instance's threads (max is order-free).
    double worst = 0.0;
    const bool done_ok = inst_ok && S.status[j] == GEVO_STATUS_COMPLETED;
    if (!kGC && A.out_cells && lane_ok && done_ok)
        for (uint32_t x = tid; x < A.n_cells; x += T)
            A.out_cells[static_cast<size_t>(x) * A.n_inst + il] = L.cell_get(x);
    if (lane_ok && done_ok && !A.static_err[t]) {
        for (int32_t e = A.entry_begin[t]; e < A.entry_begin[t + 1]; ++e) {
            const OracleEntryDev en = A.entries[e];
            const uint32_t p = static_cast<uint32_t>(en.param);
            const bool priv = (L.writable >> p) & 1ull;
            for (int32_t k = static_cast<int32_t>(tid); k < en.size; k += static_cast<int32_t>(T)) {
                const uint32_t cw = priv ? L.cell_get(A.cell_off[p] + static_cast<uint32_t>(k)).x
                                         : __ldg(A.pool + A.pool_off[p] +
                                                 static_cast<size_t>(k) * nt + t);
                const uint32_t ow = __ldg(A.pool + en.off + static_cast<size_t>(k) * nt + t);
                const double d = rel_diff(word_to_double(cw, en.elem), word_to_double(ow, en.elem));
                worst = (worst < d) ? d : worst;
            }
        }
    }
    double* errs = reinterpret_cast<double*>(reinterpret_cast<char*>(g_vfs) + (err0 - sbase));
    if (lane_ok)
        errs[q] = worst;
    __syncthreads();
    add_work(A, lane_ok ? L.work : 0u);
    if (A.regions && fixed_region == 0xFFFFFFFFu && threadIdx.x == 0 && S.region != 0xFFFFFFFFu)
        region_release(A, S.region);
    if (!leader || !inst_ok)
        return;
    double error = -1.0;
    if (done_ok) {
        if (A.static_err[t]) {
            error = 1.0;
        } else {
            error = 0.0;
            for (uint32_t u = 0; u < T; ++u) {
                const double e = errs[u * Ln + j];
                error = (error < e) ? e : error;
            }
        }
    }
    const uint32_t status = S.status[j];
    gevo_test_record rec;
    rec.cost = static_cast<int64_t>(S.cost[j]);
    rec.ir = static_cast<int64_t>(S.ir[j]);
    rec.error = error;
    rec.aux = S.aux[j];
    rec.status = static_cast<uint8_t>(status);
    rec.code = static_cast<uint8_t>(S.code[j]);
    rec.pad[0] = static_cast<uint8_t>(min(S.jumps[j], 255u));
    rec.pad[1] = 0;
    A.rec[gi] = rec;
    if (A.counters)
        atomicAdd(reinterpret_cast<unsigned long long*>(A.counters + 3), 1ull);
    if (A.early_exit && status != GEVO_STATUS_SKIPPED &&
        (status != GEVO_STATUS_COMPLETED || error > A.tolerance))
        atomicMin(A.first_fail + v, static_cast<int32_t>(t));
}

constexpr uint32_t kNoItem = 0xFFFFFFFFu;

// Work item a CTA may run now: the first test group, a group whose variant
// already failed an earlier test (a skip), or one whose earlier groups are
// all finished.
__device__ __forceinline__ bool tp_ready(const InterpArgs& A, uint32_t k) {
    const uint32_t vl = k % A.n_var, tg = k / A.n_var;
    if (tg == 0 || !A.early_exit)
        return true;
    const volatile int32_t* ff = A.first_fail;
    if (ff[A.v_begin + vl] < static_cast<int32_t>(tg * A.tp_lanes))
        return true;
    return reinterpret_cast<const volatile uint32_t*>(A.vdone)[vl] >= tg;
}

// Persistent scheduler (thread 0 of a CTA): static test-major order, blocked
// items deferred; then the deferred ones, ready first, else speculatively.
__device__ uint32_t tp_next_item(const InterpArgs& A) {
    for (;;) {
        const uint32_t k = atomicAdd(A.sched, 1u);
        if (k >= A.n_items)
            break;
        if (tp_ready(A, k))
            return k;
        const uint32_t slot = atomicAdd(A.sched + 1, 1u);
        reinterpret_cast<volatile uint32_t*>(A.defer)[slot] = k;
    }
    const volatile uint32_t* defer = A.defer;
    const volatile uint32_t* claim = A.claim;
    for (;;) {
        const uint32_t nd = reinterpret_cast<const volatile uint32_t*>(A.sched)[1];
        int32_t spec = -1;
        for (uint32_t e = 0; e < nd; ++e) {
            if (claim[e])
                continue;
            const uint32_t k = defer[e];
            if (k == kNoItem)
                continue; // being written by the CTA that deferred it (it drains it)
            if (tp_ready(A, k)) {
                if (atomicExch(A.claim + e, 1u) == 0u)
                    return k;
            } else if (spec < 0) {
                spec = static_cast<int32_t>(e);
            }
        }
        if (spec < 0)
            return kNoItem;
        if (atomicExch(A.claim + spec, 1u) == 0u)
            return defer[spec];
    }
}

template <int kM>
__global__ void GEVO_TP_BOUNDS interp_tp_kernel(const __grid_constant__ InterpArgs A) {
    __shared__ TpInst S;
    __shared__ uint32_t next_item;
    for (uint32_t round = 0;; ++round) {
        uint32_t it;
        if (A.persist) {
            if (threadIdx.x == 0)
                next_item = tp_next_item(A);
            __syncthreads();
            it = next_item;
            if (it == kNoItem)
                return;
        } else {
            if (round)
                return;
            it = blockIdx.x;
        }
        tp_item<kM>(A, S, it, A.persist ? blockIdx.x : 0xFFFFFFFFu);
        if (A.persist) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence(); // records and first_fail before the group counts as done
                atomicAdd(A.vdone + it % A.n_var, 1u);
            }
        }
    }
}

// Per-launch block records: {start, len | nphi << 16, cost of the block under
// the launch's cost table} (one thread per variant).
struct CostTableArg {
    int64_t c[GEVO_COST_CLASSES];
};

__global__ void block_cost_kernel(const gevo_variant* __restrict__ variants,
                                  const gevo_block* __restrict__ blocks,
                                  const gevo_inst* __restrict__ insts, uint32_t n_variants,
                                  const CostTableArg ct, uint4* __restrict__ out,
                                  int64_t* __restrict__ suffix) {
    // one warp per variant, one lane per block: each lane sums its block's
    // instruction classes back to front (the suffix costs refund() reads)
    const uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (v >= n_variants)
        return;
    const gevo_variant var = variants[v];
    for (uint32_t b = lane; b < var.n_blocks; b += 32) {
        const gevo_block g = blocks[var.block_base + b];
        int64_t c = 0;
        for (uint32_t j = g.len; j-- > 0;) {
            c += ct.c[insts[var.inst_base + g.start + j].cls];
            if (suffix)
                suffix[var.inst_base + g.start + j] = c;
        }
        const uint64_t u = static_cast<uint64_t>(c);
        out[var.block_base + b] =
            make_uint4(g.start, static_cast<uint32_t>(g.len) | (static_cast<uint32_t>(g.nphi) << 16),
                       static_cast<uint32_t>(u), static_cast<uint32_t>(u >> 32));
    }
}

// evaluate_fitness reduction (src/vm.cpp:558-579): one warp per variant,
// lane = test (chunks of 32). The first failing test comes from a ballot;
// dynamic IR is an exact integer sum; the error maximum uses the reference's
// comparison per element first (a NaN error never becomes the maximum, as in
// the in-order loop) and is order-free after that; the cost mean divides the
// in-order double sum of integer costs, which is exact -- hence equal to the
// int64 sum -- while every partial sum stays below 2^53 (checked; otherwise
// lane 0 adds in test order).
__global__ void fitness_kernel(const gevo_test_record* __restrict__ rec, uint32_t n_variants,
                               int32_t n_tests, double tolerance,
                               gevo_variant_record* __restrict__ out) {
    const uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int32_t lane = static_cast<int32_t>(threadIdx.x & 31);
    if (v >= n_variants)
        return;
    gevo_variant_record r{};
    r.failing_test = -1;
    r.accepted = 1;
    r.code = GEVO_OK;
    int64_t ir = 0, cost = 0, execs = 0;
    double worst = 0.0;
    bool exact = true;
    const gevo_test_record* vr = rec + static_cast<size_t>(v) * n_tests;
    for (int32_t base = 0; base < n_tests; base += 32) {
        const int32_t t = base + lane;
        const bool have = t < n_tests;
        gevo_test_record x{};
        if (have)
            x = vr[t];
        const bool fail = have && (x.status != GEVO_STATUS_COMPLETED || x.error > tolerance);
        const unsigned fm = __ballot_sync(0xffffffffu, fail);
        const int32_t first = fm ? __ffs(fm) - 1 : 32;
        const bool counted = have && lane <= first; // executed by the reference
        const bool passed = have && lane < first;
        int64_t c_ir = counted ? x.ir : 0, c_cost = passed ? x.cost : 0;
        double w = passed ? ((0.0 < x.error) ? x.error : 0.0) : 0.0;
        exact &= !passed || (x.cost >= 0 && x.cost < (int64_t(1) << 52));
        for (int o = 16; o; o >>= 1) {
            c_ir += __shfl_xor_sync(0xffffffffu, c_ir, o);
            c_cost += __shfl_xor_sync(0xffffffffu, c_cost, o);
            const double wo = __shfl_xor_sync(0xffffffffu, w, o);
            w = (w < wo) ? wo : w;
        }
        ir += c_ir;
        cost += c_cost;
        execs += fm ? first + 1 : min(32, n_tests - base);
        worst = (worst < w) ? w : worst;
        if (fm) {
            const int32_t ft = base + first;
            const gevo_test_record y = vr[ft];
            r.accepted = 0;
            r.failing_test = ft;
            if (y.status != GEVO_STATUS_COMPLETED) {
                r.code = y.code;
                r.aux = y.aux;
            } else {
                r.code = GEVO_FAIL_TOLERANCE;
                r.fail_error = y.error;
            }
            break;
        }
    }
    exact = __all_sync(0xffffffffu, exact) && cost < (int64_t(1) << 53);
    if (lane != 0)
        return;
    r.execs_ref = execs;
    r.ir_ref = ir;
    if (r.accepted) {
        double total = 0.0;
        if (exact) {
            total = static_cast<double>(cost);
        } else {
            for (int32_t t = 0; t < n_tests; ++t)
                total = __dadd_rn(total, static_cast<double>(vr[t].cost));
        }
        r.cost_mean = __ddiv_rn(total, static_cast<double>(n_tests));
        r.error_max = worst;
    }
    out[v] = r;
}

// Element-wise error metric for evoir::compute_error on host maps (structural
// mismatches are resolved by the caller). One CTA, max-reduction in shared memory.
__global__ void error_kernel(const uint32_t* __restrict__ cand, const uint32_t* __restrict__ orc,
                             const uint8_t* __restrict__ elem, uint32_t n, double* out) {
    __shared__ double red[256];
    double worst = 0.0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double d = rel_diff(word_to_double(cand[i], elem[i]), word_to_double(orc[i], elem[i]));
        worst = (worst < d) ? d : worst;
    }
    red[threadIdx.x] = worst;
    __syncthreads();
    for (uint32_t w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const double o = red[threadIdx.x + w];
            red[threadIdx.x] = (red[threadIdx.x] < o) ? o : red[threadIdx.x];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0)
        *out = red[0];
}

cudaError_t launch_error(const uint32_t* cand, const uint32_t* orc, const uint8_t* elem, uint32_t n,
                         double* out, cudaStream_t stream) {
    error_kernel<<<1, 256, 0, stream>>>(cand, orc, elem, n, out);
    return cudaGetLastError();
}

LaunchShape interp_shape(int32_t n_tests, uint32_t max_slots) {
    LaunchShape s;
    uint32_t row = 1;
    while (row < 32 && row < static_cast<uint32_t>(n_tests))
        row <<= 1;
    s.row_lanes = row;
    const size_t per_warp = static_cast<size_t>(row) * 8 * max_slots;
    s.vf_global = per_warp > kSmemBudget;
    if (s.vf_global) {
        s.warps_per_cta = 4;
        s.smem = 0;
        return s;
    }
    uint32_t w = 4;
    while (w > 1 && per_warp * w > kSmemBudget)
        w >>= 1;
    s.warps_per_cta = w;
    s.smem = per_warp * w;
    return s;
}

cudaError_t launch_block_cost(const gevo_block* blocks, const gevo_inst* insts,
                              const gevo_variant* variants, uint32_t n_variants,
                              const int64_t* cost_table, uint4* out, int64_t* suffix,
                              cudaStream_t stream) {
    if (n_variants == 0)
        return cudaSuccess;
    CostTableArg ct;
    for (int i = 0; i < GEVO_COST_CLASSES; ++i)
        ct.c[i] = cost_table[i];
    block_cost_kernel<<<(n_variants + 3) / 4, 128, 0, stream>>>(variants, blocks, insts,
                                                                    n_variants, ct, out, suffix);
    return cudaGetLastError();
}

cudaError_t launch_interp(const InterpArgs& A, cudaStream_t stream) {
    if (A.n_var == 0)
        return cudaSuccess;
    const LaunchShape s = interp_shape(A.n_tests, A.max_slots);
    const uint64_t warps = static_cast<uint64_t>(A.n_var) * A.warps_per_variant;
    const unsigned grid = static_cast<unsigned>((warps + s.warps_per_cta - 1) / s.warps_per_cta);
    if (s.vf_global) {
        interp_kernel<0><<<grid, 32 * s.warps_per_cta, 0, stream>>>(A);
        return cudaGetLastError();
    }
    const cudaError_t e = cudaFuncSetAttribute(
        interp_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s.smem));
    if (e != cudaSuccess)
        return e;
    interp_kernel<1><<<grid, 32 * s.warps_per_cta, s.smem, stream>>>(A);
    return cudaGetLastError();
}

size_t tp_smem_bytes(uint32_t threads, uint32_t lanes, const TpTables& tab, uint32_t n_cells,
                     uint32_t n_chunks, bool backup, bool gc) {
    const uint32_t K = 32 / lanes;
    const size_t warps = (threads + K - 1) / K;
    const size_t Q = static_cast<size_t>(threads) * lanes;
    const size_t vf = warps * 32 * (kTpTables ? tab.lane_slots : tab.max_slots);
    const bool compact = gc && kGcCompactVF;
    size_t b = static_cast<size_t>(tab.stage_recs) * 32 + 16 + // staged code + edge records
               (compact ? (vf * 5 + 7) & ~size_t(7) : vf * 8) +
               (static_cast<size_t>(lanes) * (tab.n_params + 2) + tab.max_lits) * 8 +
               static_cast<size_t>(lanes) * n_cells * 8 * (backup ? 2 : 1) +
               2 * static_cast<size_t>(n_chunks) * warps * 32 * 4 + 4 * Q * 4;
    return ((b + 7) & ~size_t(7)) + Q * 8;
}

TpShape tp_shape(uint32_t threads, uint32_t n_tests, const TpTables& tab, uint32_t n_cells,
                 uint32_t n_chunks, bool backup, bool gc) {
    TpShape s{0, 0, 0};
    if (threads < 1 || threads > kTpMaxBlock)
        return s;
    // most tests per CTA first (fuller, converged warps), fewer when the
    // block or its on-chip state would not fit
    static const uint32_t cap = [] {
        const char* e = std::getenv("GEVO_TP_LANES"); // tests per CTA upper bound (tuning)
        return e ? static_cast<uint32_t>(std::max(1, std::min(32, std::atoi(e)))) : 32u;
    }();
    // kernels of a warp or more of threads fill whole warps with one test per
    // CTA: no lanes of a later test run speculatively beside an earlier
    // test's, and the early-exit protocol skips the later tests' CTAs
    const uint32_t top = threads >= 32 ? 1u : min(max(n_tests, 1u), cap);
    for (uint32_t ln = top; ln >= 1; --ln) {
        const uint32_t K = 32 / ln;
        const uint32_t warps = (threads + K - 1) / K;
        if (warps * 32 > kTpMaxBlock)
            continue;
        const size_t bytes = tp_smem_bytes(threads, ln, tab, n_cells, n_chunks, backup, gc);
        if (bytes <= kSmemBudget) {
            s.warps_per_cta = warps;
            s.lanes = ln;
            s.smem = bytes;
            return s;
        }
    }
    return s;
}

uint32_t tp_resident_ctas(bool global_cells, uint32_t warps_per_cta, size_t smem) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const void* fn = global_cells ? reinterpret_cast<const void*>(interp_tp_kernel<3>)
                                  : reinterpret_cast<const void*>(interp_tp_kernel<2>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, static_cast<int>(32 * warps_per_cta), smem);
    return static_cast<uint32_t>(std::max(per_sm, 1) * std::max(sms, 1));
}

cudaError_t launch_interp_tp(const InterpArgs& A, cudaStream_t stream) {
    if (A.n_inst == 0)
        return cudaSuccess;
    const bool gc = A.gcells != nullptr;
    const TpShape s = tp_shape(static_cast<uint32_t>(A.threads), static_cast<uint32_t>(A.n_tests),
                               TpTables{A.lane_slots, A.max_slots, static_cast<uint32_t>(A.n_params), A.max_lits,
                                        A.stage_recs},
                               gc ? 0 : A.n_cells, gc ? 0 : A.n_chunks, A.tp_snap != nullptr, gc);
    if (s.warps_per_cta == 0 || s.lanes != A.tp_lanes)
        return cudaErrorInvalidConfiguration;
    // persistent launches: one CTA per region, items from the queue
    const unsigned grid = A.persist ? A.regions
                                    : A.n_var * ((static_cast<uint32_t>(A.n_tests) + s.lanes - 1) / s.lanes);
    static const int carveout = [] {
        const char* e = std::getenv("GEVO_TP_CARVEOUT"); // shared-memory carveout % (tuning)
        return e ? std::atoi(e) : -1;
    }();
    if (carveout >= 0) {
        cudaFuncSetAttribute(interp_tp_kernel<2>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
        cudaFuncSetAttribute(interp_tp_kernel<3>, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    }
    if (A.regions)
        region_init_kernel<<<(A.regions + 255) / 256, 256, 0, stream>>>(A.region_q, A.region_ctr,
                                                                       A.regions);
    if (gc) {
        const cudaError_t e = cudaFuncSetAttribute(
            interp_tp_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s.smem));
        if (e != cudaSuccess)
            return e;
        interp_tp_kernel<3><<<grid, 32 * s.warps_per_cta, s.smem, stream>>>(A);
        return cudaGetLastError();
    }
    const cudaError_t e = cudaFuncSetAttribute(
        interp_tp_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(s.smem));
    if (e != cudaSuccess)
        return e;
    interp_tp_kernel<2><<<grid, 32 * s.warps_per_cta, s.smem, stream>>>(A);
    return cudaGetLastError();
}

cudaError_t launch_fitness(const gevo_test_record* rec, uint32_t n_variants, int32_t n_tests,
                           double tolerance, gevo_variant_record* out, cudaStream_t stream) {
    const unsigned grid = (n_variants + 3) / 4;
    if (grid == 0)
        return cudaSuccess;
    fitness_kernel<<<grid, 128, 0, stream>>>(rec, n_variants, n_tests, tolerance, out);
    return cudaGetLastError();
}

} // namespace gevo
