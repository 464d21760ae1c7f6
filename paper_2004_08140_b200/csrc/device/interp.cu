// Batched sm_100a interpreter for the evoir SSA IR.
//
// One CUDA thread ("lane") executes one (variant, test) instance. Lanes are
// ordered variant-major, so the lanes of a warp run the same variant on
// consecutive tests: they fetch the same 16-byte instruction (broadcast), take
// the same dispatch branch, read/write the same value-file slot (conflict-free
// [slot][lane] shared-memory layout) and load consecutive words of the
// test-interleaved input pool (coalesced).
//
// Inside a lane the simulated threads run exactly as the reference's
// Machine::run (src/vm.cpp:114-150 of arxiv/paper_2004_08140): one at a time
// in id order up to the next barrier or ret, then the barrier-divergence check.
// Per-instruction semantics follow run_to_barrier / enter_block / step
// (src/vm.cpp:293-482): cost and budget are charged before any effect, phis
// read all arms before writing (parallel copy), traps carry the reference's
// reason codes. Floating point is IEEE binary32 round-to-nearest with no FMA
// contraction (__f*_rn intrinsics, -fmad=false), double for the error metric.
#include "interp.cuh"

#include <cuda_runtime.h>

namespace gevo {

namespace {

constexpr int kStopRet = 1, kStopSync = 2, kStopTrap = 3;
// ts_stop encodings (multi-phase kernels)
constexpr uint32_t kTsFresh = 0, kTsResume = 3u << 16; // never run / resume after barrier
constexpr uint32_t kTsRet = 1u << 16, kTsSync = 2u << 16;

struct Inst {
    uint32_t op, cls, want, res, a, b, c;
    int32_t t0, t1;
};

__device__ __forceinline__ Inst load_inst(const gevo_inst* code, uint32_t idx) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(code) + idx);
    Inst in;
    in.op = r.x & 0xFF;
    in.cls = (r.x >> 8) & 0xFF;
    in.want = (r.x >> 16) & 0xFF;
    in.res = r.y & 0xFFFF;
    in.a = r.y >> 16;
    in.b = r.z & 0xFFFF;
    in.c = r.z >> 16;
    in.t0 = static_cast<int16_t>(r.w & 0xFFFF);
    in.t1 = static_cast<int16_t>(r.w >> 16);
    return in;
}

__device__ __forceinline__ gevo_block load_block(const gevo_block* blk, int b) {
    const uint2 r = __ldg(reinterpret_cast<const uint2*>(blk) + b);
    gevo_block g;
    g.start = r.x;
    g.len = static_cast<uint16_t>(r.y & 0xFFFF);
    g.nphi = static_cast<uint16_t>(r.y >> 16);
    return g;
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

struct Lane {
    // value file (already offset by lane; slot s at s * stride)
    uint32_t* pay;
    uint8_t* tag;
    int stride;
    // program
    const gevo_inst* code;
    const gevo_block* blk;
    const gevo_arm* arm;
    uint32_t n_values;
    uint32_t stage_base;
    uint64_t writable;
    // instance
    uint32_t v, t, il;
    int32_t tid;
    // counters
    int64_t cost;
    int64_t ir;
    int32_t poll;
    // trap
    uint32_t code_out;
    int32_t aux;

    __device__ __forceinline__ uint32_t& P(uint32_t s) { return pay[s * stride]; }
    __device__ __forceinline__ uint8_t& G(uint32_t s) { return tag[s * stride]; }

    __device__ __forceinline__ bool trap(uint32_t c, int32_t x = 0) {
        code_out = c;
        aux = x;
        return false;
    }

    // Generic fetch (vm.cpp:195-222): undefined / poisoned slots trap.
    __device__ __forceinline__ bool fetch(uint32_t s, uint32_t& t, uint32_t& p) {
        t = G(s);
        p = P(s);
        if (t == GEVO_TAG_UNDEF)
            return trap(GEVO_TRAP_UNDEF_VALUE, static_cast<int32_t>(s));
        if (t == GEVO_TAG_POISON_PARAM)
            return trap(GEVO_TRAP_BAD_PARAM);
        if (t == GEVO_TAG_POISON_MISSING)
            return trap(GEVO_TRAP_BAD_OPERAND);
        return true;
    }
    // fetch_scalar (vm.cpp:224-229)
    __device__ __forceinline__ bool scalar(uint32_t s, uint32_t want, uint32_t& p) {
        const uint32_t t = G(s);
        p = P(s);
        if (t == want)
            return true;
        uint32_t tt, pp;
        if (!fetch(s, tt, pp))
            return false;
        return trap(GEVO_TRAP_OPERAND_TYPE);
    }
    // fetch_ptr (vm.cpp:231-236)
    __device__ __forceinline__ bool pointer(uint32_t s, uint32_t& t, uint32_t& off) {
        if (!fetch(s, t, off))
            return false;
        if (!is_ptr_tag(t))
            return trap(GEVO_TRAP_NOT_POINTER);
        return true;
    }
    // set (vm.cpp:285-291)
    __device__ __forceinline__ bool set(uint32_t res, uint32_t t, uint32_t p) {
        if (res == GEVO_NO_RESULT)
            return trap(GEVO_TRAP_DEF_NO_ID);
        G(res) = static_cast<uint8_t>(t);
        P(res) = p;
        return true;
    }
};

struct Thread {
    int32_t block, ip, prev;
    int64_t executed;
    uint32_t bar;
};

__device__ __forceinline__ bool charge(Lane& L, Thread& th, const int64_t* s_cost, uint32_t cls,
                                       int64_t budget) {
    L.cost += s_cost[cls];
    ++L.ir;
    if (++th.executed > budget)
        return L.trap(GEVO_BUDGET_EXCEEDED);
    return true;
}

// enter_block (vm.cpp:293-333): charge and stage every leading phi, then write.
__device__ bool enter_block(const InterpArgs& A, Lane& L, Thread& th, const int64_t* s_cost,
                            int target, gevo_block& b) {
    th.prev = th.block;
    th.block = target;
    th.ip = 0;
    b = load_block(L.blk, target);
    const uint32_t n = b.nphi;
    for (uint32_t j = 0; j < n; ++j) {
        const Inst phi = load_inst(L.code, b.start + j);
        if (!charge(L, th, s_cost, phi.cls, A.budget))
            return false;
        bool matched = false;
        for (uint32_t a = 0; a < phi.b; ++a) {
            const uint32_t raw = __ldg(reinterpret_cast<const uint32_t*>(L.arm) + phi.a + a);
            const int32_t from = static_cast<int16_t>(raw & 0xFFFF);
            if (from != th.prev)
                continue;
            uint32_t t, p;
            if (!L.fetch(raw >> 16, t, p))
                return false;
            L.G(L.stage_base + j) = static_cast<uint8_t>(t);
            L.P(L.stage_base + j) = p;
            matched = true;
            break;
        }
        if (!matched)
            return L.trap(GEVO_TRAP_PHI_NO_INCOMING);
        ++th.ip;
    }
    for (uint32_t j = 0; j < n; ++j) {
        const Inst phi = load_inst(L.code, b.start + j);
        if (!L.set(phi.res, L.G(L.stage_base + j), L.P(L.stage_base + j)))
            return false;
    }
    return true;
}

// run_to_barrier (vm.cpp:340-387) + step (389-482). Returns kStopRet,
// kStopSync or kStopTrap (L.code_out set).
__device__ int run_thread(const InterpArgs& A, Lane& L, Thread& th, const int64_t* s_cost,
                          const volatile int32_t* first_fail) {
    gevo_block b = load_block(L.blk, th.block);
    for (;;) {
        if (th.ip >= static_cast<int32_t>(b.len)) {
            L.trap(GEVO_TRAP_FELL_OFF);
            return kStopTrap;
        }
        const Inst in = load_inst(L.code, b.start + static_cast<uint32_t>(th.ip));
        if (in.op == GEVO_OP_PHI) {
            L.trap(GEVO_TRAP_PHI_OUTSIDE);
            return kStopTrap;
        }
        if (!charge(L, th, s_cost, in.cls, A.budget))
            return kStopTrap;

        bool ok = true;
        switch (in.op) {
        case GEVO_OP_SYNC:
            th.bar = in.b;
            return kStopSync;
        case GEVO_OP_RET:
            return kStopRet;
        case GEVO_OP_BR: {
            int target = in.t0;
            if (in.want == 2) {
                uint32_t c;
                if (!L.scalar(in.a, GEVO_TAG_BOOL, c))
                    return kStopTrap;
                target = c ? in.t0 : in.t1;
            }
            if (target < 0) {
                L.trap(GEVO_TRAP_UNKNOWN_BLOCK);
                return kStopTrap;
            }
            if (A.early_exit && --L.poll <= 0) {
                L.poll = 2048;
                if (first_fail[L.v] < static_cast<int32_t>(L.t)) {
                    L.trap(GEVO_SKIPPED);
                    return kStopTrap;
                }
            }
            if (!enter_block(A, L, th, s_cost, target, b))
                return kStopTrap;
            continue;
        }
        case GEVO_OP_ADD: case GEVO_OP_SUB: case GEVO_OP_MUL: case GEVO_OP_SDIV: {
            uint32_t x, y;
            if (!L.scalar(in.a, GEVO_TAG_I32, x) || !L.scalar(in.b, GEVO_TAG_I32, y))
                return kStopTrap;
            uint32_t r;
            if (in.op == GEVO_OP_ADD) {
                r = x + y;
            } else if (in.op == GEVO_OP_SUB) {
                r = x - y;
            } else if (in.op == GEVO_OP_MUL) {
                r = x * y;
            } else {
                const int32_t sx = static_cast<int32_t>(x), sy = static_cast<int32_t>(y);
                if (sy == 0) {
                    L.trap(GEVO_TRAP_DIV_ZERO);
                    return kStopTrap;
                }
                if (sx == INT32_MIN && sy == -1) {
                    L.trap(GEVO_TRAP_DIV_OVERFLOW);
                    return kStopTrap;
                }
                r = static_cast<uint32_t>(sx / sy);
            }
            ok = L.set(in.res, GEVO_TAG_I32, r);
            break;
        }
        case GEVO_OP_FADD: case GEVO_OP_FSUB: case GEVO_OP_FMUL: case GEVO_OP_FDIV: {
            uint32_t x, y;
            if (!L.scalar(in.a, GEVO_TAG_F32, x) || !L.scalar(in.b, GEVO_TAG_F32, y))
                return kStopTrap;
            const float fx = __uint_as_float(x), fy = __uint_as_float(y);
            float r;
            if (in.op == GEVO_OP_FADD)
                r = __fadd_rn(fx, fy);
            else if (in.op == GEVO_OP_FSUB)
                r = __fsub_rn(fx, fy);
            else if (in.op == GEVO_OP_FMUL)
                r = __fmul_rn(fx, fy);
            else
                r = __fdiv_rn(fx, fy);
            ok = L.set(in.res, GEVO_TAG_F32, __float_as_uint(r));
            break;
        }
        case GEVO_OP_ICMP: {
            uint32_t x, y;
            if (!L.scalar(in.a, GEVO_TAG_I32, x) || !L.scalar(in.b, GEVO_TAG_I32, y))
                return kStopTrap;
            ok = L.set(in.res, GEVO_TAG_BOOL,
                       cmp(static_cast<int32_t>(x), static_cast<int32_t>(y), in.want) ? 1u : 0u);
            break;
        }
        case GEVO_OP_FCMP: {
            uint32_t x, y;
            if (!L.scalar(in.a, GEVO_TAG_F32, x) || !L.scalar(in.b, GEVO_TAG_F32, y))
                return kStopTrap;
            ok = L.set(in.res, GEVO_TAG_BOOL,
                       cmp(__uint_as_float(x), __uint_as_float(y), in.want) ? 1u : 0u);
            break;
        }
        case GEVO_OP_SELECT: {
            uint32_t c, t, p;
            if (!L.scalar(in.a, GEVO_TAG_BOOL, c) || !L.fetch(c ? in.b : in.c, t, p))
                return kStopTrap;
            if (t != in.want) {
                L.trap(GEVO_TRAP_SELECT_ARM);
                return kStopTrap;
            }
            ok = L.set(in.res, t, p);
            break;
        }
        case GEVO_OP_LOAD: case GEVO_OP_STORE: {
            uint32_t pt, off, idx;
            if (!L.pointer(in.a, pt, off) || !L.scalar(in.b, GEVO_TAG_I32, idx))
                return kStopTrap;
            uint32_t vt = 0, vp = 0;
            if (in.op == GEVO_OP_STORE) {
                if (!L.fetch(in.c, vt, vp))
                    return kStopTrap;
                if (vt < GEVO_TAG_I32 || vt > GEVO_TAG_BOOL) {
                    L.trap(GEVO_TRAP_STORE_NONSCALAR);
                    return kStopTrap;
                }
                if (vt == GEVO_TAG_BOOL) {
                    L.trap(GEVO_TRAP_STORE_BOOL);
                    return kStopTrap;
                }
            }
            const int64_t eff = static_cast<int64_t>(static_cast<int32_t>(off)) +
                                static_cast<int64_t>(static_cast<int32_t>(idx));
            const uint32_t nt = static_cast<uint32_t>(A.n_tests);
            if (pt == GEVO_TAG_PTR_SHARED) {
                if (eff < 0 || eff >= A.shared_words) {
                    L.trap(GEVO_TRAP_SHARED_OOB);
                    return kStopTrap;
                }
                const size_t at = static_cast<size_t>(eff) * A.n_inst + L.il;
                if (in.op == GEVO_OP_LOAD) {
                    const uint32_t wt = A.sh_tag[at];
                    if (wt == GEVO_TAG_UNDEF) {
                        L.trap(GEVO_TRAP_SHARED_UNINIT);
                        return kStopTrap;
                    }
                    if (wt != in.want) {
                        L.trap(GEVO_TRAP_SHARED_TYPE);
                        return kStopTrap;
                    }
                    ok = L.set(in.res, wt, A.sh_val[at]);
                } else {
                    A.sh_tag[at] = static_cast<uint8_t>(vt);
                    A.sh_val[at] = vp;
                }
                break;
            }
            const uint32_t p = pt & 0x3F;
            const size_t tp = static_cast<size_t>(L.t) * A.n_params + p;
            const int32_t size = __ldg(A.buf_size + tp);
            if (eff < 0 || eff >= size) {
                L.trap(GEVO_TRAP_GLOBAL_OOB);
                return kStopTrap;
            }
            const uint32_t elem = __ldg(A.buf_elem + tp);
            const bool priv = (L.writable >> p) & 1ull;
            if (in.op == GEVO_OP_LOAD) {
                if (elem != in.want) {
                    L.trap(GEVO_TRAP_GLOBAL_LOAD_TYPE);
                    return kStopTrap;
                }
                const uint32_t w =
                    priv ? A.priv[A.priv_off[p] + static_cast<size_t>(eff) * A.n_inst + L.il]
                         : __ldg(A.pool + A.pool_off[p] + static_cast<size_t>(eff) * nt + L.t);
                ok = L.set(in.res, elem, w);
            } else {
                if (elem != vt) {
                    L.trap(GEVO_TRAP_GLOBAL_STORE_TYPE);
                    return kStopTrap;
                }
                if (!priv) {
                    L.trap(GEVO_TRAP_INTERNAL);
                    return kStopTrap;
                }
                A.priv[A.priv_off[p] + static_cast<size_t>(eff) * A.n_inst + L.il] = vp;
            }
            break;
        }
        case GEVO_OP_GETINDEX: {
            uint32_t pt, off, idx;
            if (!L.pointer(in.a, pt, off))
                return kStopTrap;
            if ((pt == GEVO_TAG_PTR_SHARED ? 1u : 0u) != in.want) {
                L.trap(GEVO_TRAP_GETINDEX_SPACE);
                return kStopTrap;
            }
            if (!L.scalar(in.b, GEVO_TAG_I32, idx))
                return kStopTrap;
            ok = L.set(in.res, pt, off + idx);
            break;
        }
        case GEVO_OP_TID:
            ok = L.set(in.res, GEVO_TAG_I32, static_cast<uint32_t>(L.tid));
            break;
        case GEVO_OP_NTHREADS:
            ok = L.set(in.res, GEVO_TAG_I32, static_cast<uint32_t>(A.threads));
            break;
        case GEVO_OP_CONST:
            ok = L.set(in.res, L.G(in.a), L.P(in.a));
            break;
        default:
            L.trap(GEVO_TRAP_UNEXPECTED_OP);
            return kStopTrap;
        }
        if (!ok)
            return kStopTrap;
        ++th.ip;
    }
}

} // namespace


// Error metric of one completed instance (compute_error, src/vm.cpp:536-556):
// 1.0 on any structural mismatch (resolved on the host per test), else the max
// over oracle elements of the clamped relative difference. max() is exact and
// order-free, so the per-buffer early return of the reference is not needed.
__device__ double instance_error(const InterpArgs& A, const Lane& L) {
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

__device__ __forceinline__ void reset_values(Lane& L) {
    for (uint32_t s = 0; s < L.n_values; ++s)
        L.G(s) = GEVO_TAG_UNDEF;
}

// Machine::run for one instance (src/vm.cpp:114-150). Returns the status.
__device__ uint32_t run_instance(const InterpArgs& A, Lane& L, const gevo_variant& var,
                                 const int64_t* s_cost, const volatile int32_t* first_fail) {
    const int32_t T = A.threads;
    if (!(var.flags & GEVO_VAR_HAS_SYNC)) {
        // No barrier instruction: every thread runs to ret in phase 0.
        for (int32_t tid = 0; tid < T; ++tid) {
            reset_values(L);
            L.tid = tid;
            Thread th{0, 0, -1, 0, 0};
            const int r = run_thread(A, L, th, s_cost, first_fail);
            if (r == kStopTrap)
                return L.code_out == GEVO_BUDGET_EXCEEDED ? GEVO_STATUS_BUDGET
                       : L.code_out == GEVO_SKIPPED      ? GEVO_STATUS_SKIPPED
                                                         : GEVO_STATUS_TRAP;
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
                const size_t vbase = static_cast<size_t>(tid) * A.ts_slots;
                if (st == kTsFresh) {
                    reset_values(L);
                } else {
                    for (uint32_t s = 0; s < L.n_values; ++s) {
                        const size_t sv = (vbase + s) * n + L.il;
                        L.G(s) = A.ts_tag[sv];
                        L.P(s) = A.ts_val[sv];
                    }
                }
                L.tid = tid;
                const int r = run_thread(A, L, th, s_cost, first_fail);
                if (r == kStopTrap)
                    return L.code_out == GEVO_BUDGET_EXCEEDED ? GEVO_STATUS_BUDGET
                           : L.code_out == GEVO_SKIPPED      ? GEVO_STATUS_SKIPPED
                                                             : GEVO_STATUS_TRAP;
                A.ts_pos[at] = (th.block << 16) | th.ip;
                A.ts_prev[at] = th.prev;
                A.ts_exec[at] = th.executed;
                st = r == kStopSync ? (kTsSync | th.bar) : kTsRet;
                A.ts_stop[at] = st;
                if (r == kStopSync) {
                    for (uint32_t s = 0; s < L.n_values; ++s) {
                        const size_t sv = (vbase + s) * n + L.il;
                        A.ts_tag[sv] = L.G(s);
                        A.ts_val[sv] = L.P(s);
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

template <int kLanes>
__global__ void __launch_bounds__(kLanes) interp_kernel(const __grid_constant__ InterpArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ int64_t s_cost[GEVO_COST_CLASSES];
    if (threadIdx.x < GEVO_COST_CLASSES)
        s_cost[threadIdx.x] = A.cost[threadIdx.x];
    __syncthreads();

    const uint32_t il = blockIdx.x * kLanes + threadIdx.x;
    if (il >= A.n_inst)
        return;
    const uint64_t gi = A.inst_begin + il;
    const uint32_t nt = static_cast<uint32_t>(A.n_tests);

    Lane L;
    L.v = static_cast<uint32_t>(gi / nt);
    L.t = static_cast<uint32_t>(gi % nt);
    L.il = il;
    L.stride = kLanes;
    L.pay = reinterpret_cast<uint32_t*>(smem) + threadIdx.x;
    L.tag = smem + static_cast<size_t>(4) * kLanes * A.max_slots + threadIdx.x;
    L.cost = 0;
    L.ir = 0;
    L.poll = 2048;
    L.code_out = GEVO_OK;
    L.aux = 0;
    L.writable = 0;
    L.tid = 0;

    const volatile int32_t* first_fail = A.first_fail;
    uint32_t status;
    double error = -1.0;
    const uint8_t setup = A.setup_code[L.t];
    if (A.early_exit && first_fail[L.v] < static_cast<int32_t>(L.t)) {
        L.code_out = GEVO_SKIPPED;
        status = GEVO_STATUS_SKIPPED;
    } else if (setup != GEVO_OK) {
        // Machine ctor failure: trap with cost 0 (src/vm.cpp:516-520).
        L.code_out = setup;
        L.aux = A.setup_aux[L.t];
        status = GEVO_STATUS_TRAP;
    } else {
        const gevo_variant var = A.variants[L.v];
        const uint32_t P = static_cast<uint32_t>(A.n_params);
        L.code = A.insts + var.inst_base;
        L.blk = A.blocks + var.block_base;
        L.arm = A.arms + var.arm_base;
        L.n_values = var.n_values;
        L.writable = var.writable;
        const uint32_t lit_begin = var.n_values + P + 2;
        L.stage_base = lit_begin + var.n_lits;

        // Parameters (bound per test), poison slots, literal pool.
        const size_t tp0 = static_cast<size_t>(L.t) * P;
        for (uint32_t p = 0; p < P; ++p) {
            L.G(var.n_values + p) = A.param_tag[tp0 + p];
            L.P(var.n_values + p) = A.param_payload[tp0 + p];
        }
        L.G(var.n_values + P) = GEVO_TAG_POISON_PARAM;
        L.G(var.n_values + P + 1) = GEVO_TAG_POISON_MISSING;
        for (uint32_t k = 0; k < var.n_lits; ++k) {
            L.G(lit_begin + k) = __ldg(A.lit_tag + var.lit_base + k);
            L.P(lit_begin + k) = __ldg(A.lit_payload + var.lit_base + k);
        }
        // Private copies of the buffers this variant may store to
        // (Machine ctor copies every global buffer, src/vm.cpp:96-97; read-only
        // ones are served from the shared test pool).
        for (uint64_t m = var.writable; m; m &= m - 1) {
            const uint32_t p = static_cast<uint32_t>(__ffsll(static_cast<long long>(m)) - 1);
            const int32_t rows = A.buf_size[tp0 + p];
            for (int32_t e = 0; e < rows; ++e)
                A.priv[A.priv_off[p] + static_cast<size_t>(e) * A.n_inst + il] =
                    __ldg(A.pool + A.pool_off[p] + static_cast<size_t>(e) * nt + L.t);
        }
        for (int32_t w = 0; w < A.shared_words; ++w)
            A.sh_tag[static_cast<size_t>(w) * A.n_inst + il] = GEVO_TAG_UNDEF;

        status = run_instance(A, L, var, s_cost, first_fail);
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
    rec.pad[0] = rec.pad[1] = 0;
    A.rec[gi] = rec;

    if (A.early_exit && status != GEVO_STATUS_SKIPPED &&
        (status != GEVO_STATUS_COMPLETED || error > A.tolerance))
        atomicMin(A.first_fail + L.v, static_cast<int32_t>(L.t));
}

// evaluate_fitness reduction (src/vm.cpp:558-579), one thread per variant,
// tests in order so the double sum and the first failure match the reference.
__global__ void fitness_kernel(const gevo_test_record* __restrict__ rec, uint32_t n_variants,
                               int32_t n_tests, double tolerance,
                               gevo_variant_record* __restrict__ out) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_variants)
        return;
    gevo_variant_record r{};
    r.failing_test = -1;
    r.accepted = 1;
    r.code = GEVO_OK;
    double total = 0.0, worst = 0.0;
    for (int32_t t = 0; t < n_tests; ++t) {
        const gevo_test_record x = rec[static_cast<size_t>(v) * n_tests + t];
        r.execs_ref += 1;
        r.ir_ref += x.ir;
        if (x.status != GEVO_STATUS_COMPLETED) {
            r.accepted = 0;
            r.failing_test = t;
            r.code = x.code;
            r.aux = x.aux;
            break;
        }
        if (x.error > tolerance) {
            r.accepted = 0;
            r.failing_test = t;
            r.code = GEVO_FAIL_TOLERANCE;
            r.fail_error = x.error;
            break;
        }
        worst = (worst < x.error) ? x.error : worst;
        total = __dadd_rn(total, static_cast<double>(x.cost));
    }
    if (r.accepted) {
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

// Lanes per CTA: 128 while the value file fits (5 B per slot per lane),
// 32 for very large variants.
int interp_lanes(uint32_t max_slots) { return max_slots <= kMaxSlots128 ? 128 : 32; }

cudaError_t launch_interp(const InterpArgs& A, cudaStream_t stream) {
    const int lanes = interp_lanes(A.max_slots);
    const size_t smem = static_cast<size_t>(5) * lanes * A.max_slots;
    const unsigned grid = (A.n_inst + lanes - 1) / lanes;
    if (grid == 0)
        return cudaSuccess;
    if (lanes == 128) {
        cudaFuncSetAttribute(interp_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        interp_kernel<128><<<grid, 128, smem, stream>>>(A);
    } else {
        cudaFuncSetAttribute(interp_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem));
        interp_kernel<32><<<grid, 32, smem, stream>>>(A);
    }
    return cudaGetLastError();
}

cudaError_t launch_fitness(const gevo_test_record* rec, uint32_t n_variants, int32_t n_tests,
                           double tolerance, gevo_variant_record* out, cudaStream_t stream) {
    const unsigned grid = (n_variants + 127) / 128;
    if (grid == 0)
        return cudaSuccess;
    fitness_kernel<<<grid, 128, 0, stream>>>(rec, n_variants, n_tests, tolerance, out);
    return cudaGetLastError();
}

} // namespace gevo
