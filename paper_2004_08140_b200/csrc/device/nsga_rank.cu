// GPU NSGA-II ranking over (cost, error) -- rank_population and select_best
// of arxiv/paper_2004_08140 (src/nsga.cpp:9-148), bit-identical.
//
// The reference peels fronts with an O(n^2) dominance count (nsga.cpp:15-46),
// then sorts every front twice for crowding (nsga.cpp:48-86). Here:
//
//  1. Order-preserving 64-bit keys of both objectives, and two lexicographic
//     orders by stable radix sorts: A = (cost, error, index) and
//     B = (error, cost, index). Every dominator of a point precedes it in A.
//  2. Identical points form groups (they never dominate each other and share a
//     front); groups carry the dense ranks of their cost and error.
//  3. Fronts of the groups, in one CTA, by the cheaper of two exact schemes:
//     * levels: walk the distinct values of one objective (C costs or D
//       errors) in ascending order. Inside a level the groups are sorted by
//       the other objective, and front_t = t + max_{i<=t}(B_i + 1 - i), where
//       B_i is the highest front among lower levels at or below group i's
//       position (a prefix-max array over positions). Each level is two
//       block-wide max-scans; total O(g + min(C,D) * max(C,D) / 1024) steps.
//     * staircase: the front of a point is the length of its longest
//       dominance chain = the number of staircase levels whose minimum error
//       is <= its error (patience sorting over A). One warp per point with a
//       32-ary search of the staircase; used when both objectives have many
//       distinct values (then the level walk would be quadratic).
//     Either scheme yields the unique partition the reference's peel yields.
//  4. Front sizes by histogram + exclusive scan; members (ascending index per
//     front, nsga.cpp:32-43) by a stable radix sort of the indices by front.
//  5. Crowding: each front's cost order (key, other, index) is A restricted to
//     the front and its error order is B restricted to it, so a stable sort of
//     A (and of B) by front gives both orders and every member's position in
//     O(1); the reference's double operations are replayed per member, cost
//     objective first (nsga.cpp:57-85).
//  6. select_best(keep): the fronts before the cut front are taken whole in
//     ascending index order; the cut front is ordered by (crowding desc,
//     index asc) with a stable segmented radix sort (nsga.cpp:126-148).
//
// Nothing synchronises with the host: every data-dependent size (groups,
// fronts, the cut front) stays on the device.
#include "nsga_rank.cuh"

#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>

namespace gevo {

namespace {

constexpr int kThreads = 256;
constexpr int kFrontThreads = 1024;
// staircase levels kept in shared memory by the front kernel (int32 each)
constexpr int kStairSmem = 48 * 1024;

__device__ __forceinline__ uint64_t ord64(double x) {
    // total order of finite/infinite doubles as unsigned integers; -0 == +0
    // like the reference's double comparisons
    uint64_t b = static_cast<uint64_t>(__double_as_longlong(x == 0.0 ? 0.0 : x));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void key_kernel(const double* __restrict__ cost, const double* __restrict__ err, int32_t n,
                           uint64_t* __restrict__ kc, uint64_t* __restrict__ ke,
                           int32_t* __restrict__ iota) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        kc[i] = ord64(cost[i]);
        ke[i] = ord64(err[i]);
        iota[i] = i;
    }
}

__global__ void gather_u64(const uint64_t* __restrict__ key, const int32_t* __restrict__ idx, int32_t n,
                           uint64_t* __restrict__ out) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n)
        out[p] = key[idx[p]];
}

__global__ void gather_u32(const int32_t* __restrict__ key, const int32_t* __restrict__ idx, int32_t n,
                           uint32_t* __restrict__ out) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < n)
        out[p] = static_cast<uint32_t>(key[idx[p]]);
}

// Group / distinct-value flags over both orders (1 at the start of a run).
__global__ void flags_kernel(const uint64_t* __restrict__ kc, const uint64_t* __restrict__ ke,
                             const int32_t* __restrict__ A, const int32_t* __restrict__ B, int32_t n,
                             int32_t* __restrict__ gflag, int32_t* __restrict__ cflag,
                             int32_t* __restrict__ eflag, int32_t* __restrict__ bflag,
                             int32_t* __restrict__ posA, int32_t* __restrict__ posB) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    const int32_t i = A[p];
    posA[i] = p;
    if (p == 0) {
        gflag[p] = cflag[p] = 1;
    } else {
        const int32_t h = A[p - 1];
        const bool dc = kc[i] != kc[h];
        cflag[p] = dc;
        gflag[p] = dc || ke[i] != ke[h];
    }
    const int32_t j = B[p];
    posB[j] = p;
    if (p == 0) {
        eflag[p] = bflag[p] = 1;
    } else {
        const int32_t h = B[p - 1];
        const bool de = ke[j] != ke[h];
        eflag[p] = de;
        bflag[p] = de || kc[j] != kc[h];
    }
}

// Per-group dense ranks (inclusive scans of the flags are 1-based ids) and
// the groups listed in (error, cost) order.
__global__ void group_kernel(const int32_t* __restrict__ A, const int32_t* __restrict__ B, int32_t n,
                             const int32_t* __restrict__ gid, const int32_t* __restrict__ cpos,
                             const int32_t* __restrict__ epos, const int32_t* __restrict__ bgid,
                             const int32_t* __restrict__ posA, const int32_t* __restrict__ posB,
                             int32_t* __restrict__ grp_c, int32_t* __restrict__ grp_e,
                             int32_t* __restrict__ gB, int32_t* __restrict__ meta) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    if (p == 0 || gid[p] != gid[p - 1]) {
        const int32_t g = gid[p] - 1;
        grp_c[g] = cpos[p] - 1;
        grp_e[g] = epos[posB[A[p]]] - 1;
    }
    if (p == 0 || bgid[p] != bgid[p - 1])
        gB[bgid[p] - 1] = gid[posA[B[p]]] - 1;
    if (p == n - 1) {
        meta[kMetaGroups] = gid[p];
        meta[kMetaCosts] = cpos[p];
        meta[kMetaErrors] = epos[p];
    }
}

using FrontScan = cub::BlockScan<int32_t, kFrontThreads>;

// The A-order list of groups is the identity (list == nullptr).
__device__ __forceinline__ int32_t list_at(const int32_t* list, int32_t k) { return list ? list[k] : k; }

struct MaxOp {
    __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

// Level walk (see the file comment). `list` holds the groups in (level, pos)
// order; lvl_start is scratch of nlev + 1 entries; pq/uq hold npos entries.
__device__ void level_walk(const int32_t* __restrict__ list, const int32_t* __restrict__ level,
                           const int32_t* __restrict__ pos, int32_t g, int32_t nlev, int32_t npos,
                           int32_t* __restrict__ lvl_start, int32_t* __restrict__ pq,
                           int32_t* __restrict__ uq, int32_t* __restrict__ fg,
                           FrontScan::TempStorage& ts, int32_t& fmax) {
    const int tid = threadIdx.x;
    for (int32_t k = tid; k < npos; k += kFrontThreads)
        pq[k] = uq[k] = -1;
    for (int32_t k = tid; k < g; k += kFrontThreads)
        if (k == 0 || level[list_at(list, k)] != level[list_at(list, k - 1)])
            lvl_start[level[list_at(list, k)]] = k;
    if (tid == 0)
        lvl_start[nlev] = g;
    __syncthreads();
    int32_t top = -1;
    for (int32_t d = 0; d < nlev; ++d) {
        const int32_t s = lvl_start[d], e = lvl_start[d + 1];
        int32_t carry = INT32_MIN;
        for (int32_t base = s; base < e; base += kFrontThreads) {
            const int32_t t = base - s + tid;
            const bool in = base + tid < e;
            int32_t G = 0, p = 0, a = INT32_MIN;
            if (in) {
                G = list_at(list, base + tid);
                p = pos[G];
                a = pq[p] + 1 - t;
            }
            int32_t m, agg;
            FrontScan(ts).InclusiveScan(a, m, MaxOp(), agg);
            m = max(m, carry);
            if (in) {
                const int32_t f = t + m;
                fg[G] = f;
                uq[p] = f;
                top = max(top, f);
            }
            carry = max(carry, agg);
            __syncthreads();
        }
        // pq = max(pq, prefix max of this level's fronts by position)
        const int32_t p0 = pos[list_at(list, s)];
        carry = -1;
        for (int32_t base = p0; base < npos; base += kFrontThreads) {
            const int32_t c = base + tid;
            const int32_t u = c < npos ? uq[c] : -1;
            int32_t m, agg;
            FrontScan(ts).InclusiveScan(u, m, MaxOp(), agg);
            m = max(m, carry);
            if (c < npos) {
                pq[c] = max(pq[c], m);
                uq[c] = -1;
            }
            carry = max(carry, agg);
            __syncthreads();
        }
    }
    atomicMax(&fmax, top);
}

// Staircase over the groups in A order (one warp). stair is non-decreasing;
// the front of a group is the number of levels whose minimum error is <= its
// error (upper_bound), found with a 32-ary search.
__device__ void staircase(const int32_t* __restrict__ grp_e, int32_t g, volatile int32_t* stair,
                          int32_t* __restrict__ fg, int32_t& fmax) {
    const int lane = threadIdx.x & 31;
    int32_t F = 0;
    for (int32_t base = 0; base < g; base += 32) {
        const int32_t mine = base + lane < g ? grp_e[base + lane] : 0;
        const int32_t cnt = min(32, g - base);
        int32_t outf = 0;
        for (int32_t k = 0; k < cnt; ++k) {
            const int32_t e = __shfl_sync(0xffffffffu, mine, k);
            int32_t lo = 0, hi = F;
            while (hi - lo > 32) {
                const int32_t step = (hi - lo + 31) >> 5;
                const int32_t x = lo + (lane + 1) * step - 1;
                const bool le = x < hi && stair[x] <= e;
                const int32_t c = __popc(__ballot_sync(0xffffffffu, le));
                const int32_t nlo = lo + c * step;
                hi = min(hi, lo + (c + 1) * step - 1);
                lo = nlo;
            }
            const int32_t x = lo + lane;
            const bool le = x < hi && stair[x] <= e;
            const int32_t r = lo + __popc(__ballot_sync(0xffffffffu, le));
            if (lane == 0)
                stair[r] = e;
            __syncwarp();
            if (r == F)
                ++F;
            if (lane == k)
                outf = r;
        }
        if (lane < cnt)
            fg[base + lane] = outf;
    }
    if (lane == 0)
        atomicMax(&fmax, F - 1);
}

__global__ void __launch_bounds__(kFrontThreads, 1)
    front_kernel(const int32_t* __restrict__ grp_c, const int32_t* __restrict__ grp_e,
                 const int32_t* __restrict__ gB, bool single_group, int32_t* __restrict__ lvl,
                 int32_t* __restrict__ pq, int32_t* __restrict__ uq, int32_t* __restrict__ gstair,
                 int32_t* __restrict__ fg, int32_t* __restrict__ meta) {
    __shared__ FrontScan::TempStorage ts;
    __shared__ int32_t fmax, strategy;
    extern __shared__ int32_t sstair[];
    const int32_t g = meta[kMetaGroups], C = meta[kMetaCosts], D = meta[kMetaErrors];
    if (threadIdx.x == 0) {
        fmax = -1;
        if (single_group) {
            strategy = 3;
        } else {
            // block-scan steps of the level walk vs warp steps of the staircase
            const int32_t nl = min(C, D), np = max(C, D);
            const double walk = static_cast<double>(nl) * ((np + kFrontThreads - 1) / kFrontThreads + 2);
            const double stair = static_cast<double>(g) / 8.0;
            strategy = walk <= stair ? (C <= D ? 0 : 1) : 2;
        }
    }
    __syncthreads();
    const int32_t st = strategy;
    if (st == 3) {
        for (int32_t k = threadIdx.x; k < g; k += kFrontThreads)
            fg[k] = 0;
        if (threadIdx.x == 0)
            fmax = g > 0 ? 0 : -1;
    } else if (st == 0) {
        // cost levels: A order is (cost, error) -- the groups 0..g-1 in order
        level_walk(nullptr, grp_c, grp_e, g, C, D, lvl, pq, uq, fg, ts, fmax);
    } else if (st == 1) {
        level_walk(gB, grp_e, grp_c, g, D, C, lvl, pq, uq, fg, ts, fmax);
    } else if (threadIdx.x < 32) {
        staircase(grp_e, g, g <= kStairSmem ? sstair : gstair, fg, fmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        meta[kMetaFronts] = fmax + 1;
        meta[kMetaStrategy] = st;
    }
}

__global__ void scatter_front_kernel(const int32_t* __restrict__ A, const int32_t* __restrict__ gid,
                                     const int32_t* __restrict__ fg, int32_t n,
                                     int32_t* __restrict__ front, int32_t* __restrict__ cnt) {
    const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n)
        return;
    const int32_t f = fg[gid[p] - 1];
    front[A[p]] = f;
    atomicAdd(&cnt[f], 1);
}

__global__ void pos_kernel(const int32_t* __restrict__ ocost, const int32_t* __restrict__ oerr,
                           int32_t n, int32_t* __restrict__ pos_c, int32_t* __restrict__ pos_e) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n) {
        pos_c[ocost[q]] = q;
        pos_e[oerr[q]] = q;
    }
}

__global__ void crowd_kernel(const double* __restrict__ cost, const double* __restrict__ err,
                             const int32_t* __restrict__ front, const int32_t* __restrict__ offsets,
                             const int32_t* __restrict__ ocost, const int32_t* __restrict__ oerr,
                             const int32_t* __restrict__ pos_c, const int32_t* __restrict__ pos_e,
                             int32_t n, double* __restrict__ crowd) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int32_t f = front[i];
    const int32_t b = offsets[f], m = offsets[f + 1] - b;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    if (m <= 2) {
        crowd[i] = inf;
        return;
    }
    // cost objective (key cost, tie error, then index)
    const int32_t q1 = pos_c[i], p1 = q1 - b;
    double d = 0.0;
    const double lo1 = cost[ocost[b]], hi1 = cost[ocost[b + m - 1]];
    if (p1 == 0 || p1 == m - 1)
        d = inf;
    else if (hi1 > lo1)
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(cost[ocost[q1 + 1]], cost[ocost[q1 - 1]]),
                                   __dsub_rn(hi1, lo1)));
    // error objective; members already at +inf are skipped
    const int32_t q2 = pos_e[i], p2 = q2 - b;
    const double lo2 = err[oerr[b]], hi2 = err[oerr[b + m - 1]];
    if (p2 == 0 || p2 == m - 1)
        d = inf;
    else if (hi2 > lo2 && d != inf)
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(err[oerr[q2 + 1]], err[oerr[q2 - 1]]),
                                   __dsub_rn(hi2, lo2)));
    crowd[i] = d;
}

// select_best: the cut front f* is the first whose end passes keep.
__global__ void cut_kernel(const int32_t* __restrict__ offsets, int32_t keep, int32_t* __restrict__ meta,
                           int32_t* __restrict__ seg) {
    const int32_t F = meta[kMetaFronts];
    int32_t lo = 0, hi = F; // first f with offsets[f + 1] > keep
    while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (offsets[mid + 1] > keep)
            hi = mid;
        else
            lo = mid + 1;
    }
    meta[kMetaCut] = lo;
    seg[0] = offsets[lo];
    seg[1] = lo < F ? offsets[lo + 1] : offsets[lo];
}

__global__ void crowd_key_kernel(const double* __restrict__ crowd, const int32_t* __restrict__ members,
                                 int32_t n, uint64_t* __restrict__ key) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < n)
        key[q] = ord64(crowd[members[q]]);
}

__global__ void select_kernel(const int32_t* __restrict__ members, const int32_t* __restrict__ sorted,
                              const int32_t* __restrict__ seg, int32_t keep,
                              int32_t* __restrict__ out) {
    const int32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < keep)
        out[q] = q < seg[0] ? members[q] : sorted[q];
}

// ---- small pools: the whole ranking in one CTA ---------------------------
//
// For pools of up to kSmallN members (a search ranks pools of 1.25 x pop
// every generation) the multi-kernel pipeline above is launch-bound. Here one
// CTA does everything in shared memory with O(n^2 / 1024) counting passes:
// lexicographic positions, fronts by the staircase (one warp), ascending-index
// members, per-front cost / error positions, crowding and select_best.
constexpr int kSmallN = 2048;
constexpr int kSmallThreads = 1024;

__device__ __forceinline__ bool lex_less(double a0, double b0, int32_t i0, double a1, double b1,
                                         int32_t i1) {
    if (a0 != a1)
        return a0 < a1;
    if (b0 != b1)
        return b0 < b1;
    return i0 < i1;
}

__global__ void __launch_bounds__(kSmallThreads, 1)
    rank_small_kernel(const double* __restrict__ gcost, const double* __restrict__ gerr, int32_t n,
                      bool single_group, int32_t keep, int32_t* __restrict__ front_out,
                      int32_t* __restrict__ members_out, int32_t* __restrict__ offsets_out,
                      double* __restrict__ crowd_out, int32_t* __restrict__ select_out,
                      int32_t* __restrict__ meta) {
    extern __shared__ double sm[];
    double* cost = sm;
    double* err = sm + n;
    int32_t* A = reinterpret_cast<int32_t*>(sm + 2 * n); // A order: index at each position
    int32_t* B = A + n;        // B order
    int32_t* posA = B + n;     // position of each index in A
    int32_t* posB = posA + n;
    int32_t* front = posB + n;
    int32_t* off = front + n;  // [n + 1] front offsets
    int32_t* ocost = off + n + 1;
    int32_t* oerr = ocost + n;
    int32_t* stair = oerr + n;
    __shared__ int32_t sF, sCut;
    const int tid = threadIdx.x;
    for (int32_t i = tid; i < n; i += kSmallThreads) {
        cost[i] = gcost[i];
        err[i] = gerr[i];
    }
    __syncthreads();
    // 1. lexicographic positions (cost, error, index) and (error, cost, index)
    for (int32_t i = tid; i < n; i += kSmallThreads) {
        const double ci = cost[i], ei = err[i];
        int32_t pa = 0, pb = 0;
        for (int32_t j = 0; j < n; ++j) {
            const double cj = cost[j], ej = err[j];
            pa += lex_less(cj, ej, j, ci, ei, i);
            pb += lex_less(ej, cj, j, ei, ci, i);
        }
        posA[i] = pa;
        posB[i] = pb;
        A[pa] = i;
        B[pb] = i;
    }
    __syncthreads();
    // 2. fronts: the staircase over the A order (identical points share a
    //    front), one warp, 32-ary search of the staircase
    if (tid < 32) {
        const int lane = tid;
        int32_t F = 0, last = -1;
        if (single_group) {
            for (int32_t p = lane; p < n; p += 32)
                front[A[p]] = 0;
            F = 1;
        } else {
            for (int32_t p = 0; p < n; ++p) {
                const int32_t i = A[p];
                const double c = cost[i], e = err[i];
                if (p > 0 && c == cost[A[p - 1]] && e == err[A[p - 1]]) {
                    if (lane == 0)
                        front[i] = last;
                    continue;
                }
                int32_t lo = 0, hi = F;
                while (hi - lo > 32) {
                    const int32_t step = (hi - lo + 31) >> 5;
                    const int32_t x = lo + (lane + 1) * step - 1;
                    const bool le = x < hi && err[stair[x]] <= e;
                    const int32_t cnt = __popc(__ballot_sync(0xffffffffu, le));
                    const int32_t nlo = lo + cnt * step;
                    hi = min(hi, lo + (cnt + 1) * step - 1);
                    lo = nlo;
                }
                const int32_t x = lo + lane;
                const bool le = x < hi && err[stair[x]] <= e;
                const int32_t r = lo + __popc(__ballot_sync(0xffffffffu, le));
                if (lane == 0) {
                    stair[r] = i; // (the staircase holds the index of its minimum)
                    front[i] = r;
                }
                __syncwarp();
                if (r == F)
                    ++F;
                last = r;
            }
        }
        if (lane == 0)
            sF = F;
    }
    __syncthreads();
    const int32_t F = sF;
    // 3. front sizes -> offsets (count, then a serial prefix over F <= n)
    for (int32_t f = tid; f <= n; f += kSmallThreads)
        off[f] = 0;
    __syncthreads();
    for (int32_t i = tid; i < n; i += kSmallThreads)
        atomicAdd(&off[front[i] + 1], 1);
    __syncthreads();
    if (tid == 0)
        for (int32_t f = 1; f <= F; ++f)
            off[f] += off[f - 1];
    __syncthreads();
    // 4. members (ascending index per front) and per-front positions in the
    //    cost / error orders
    for (int32_t i = tid; i < n; i += kSmallThreads) {
        const int32_t f = front[i];
        int32_t pm = 0, pc = 0, pe = 0;
        for (int32_t j = 0; j < n; ++j) {
            if (front[j] != f)
                continue;
            pm += j < i;
            pc += posA[j] < posA[i];
            pe += posB[j] < posB[i];
        }
        members_out[off[f] + pm] = i;
        ocost[off[f] + pc] = i;
        oerr[off[f] + pe] = i;
    }
    __syncthreads();
    // posA / posB now: each member's slot in its front's cost / error order
    for (int32_t q = tid; q < n; q += kSmallThreads) {
        posA[ocost[q]] = q;
        posB[oerr[q]] = q;
    }
    __syncthreads();
    // 5. crowding (nsga.cpp:48-86), cost objective first
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    for (int32_t i = tid; i < n; i += kSmallThreads) {
        const int32_t f = front[i], b = off[f], m = off[f + 1] - b;
        double d = 0.0;
        if (m <= 2) {
            d = inf;
        } else {
            const int32_t q1 = posA[i], p1 = q1 - b;
            const double lo1 = cost[ocost[b]], hi1 = cost[ocost[b + m - 1]];
            if (p1 == 0 || p1 == m - 1)
                d = inf;
            else if (hi1 > lo1)
                d = __dadd_rn(d, __ddiv_rn(__dsub_rn(cost[ocost[q1 + 1]], cost[ocost[q1 - 1]]),
                                           __dsub_rn(hi1, lo1)));
            const int32_t q2 = posB[i], p2 = q2 - b;
            const double lo2 = err[oerr[b]], hi2 = err[oerr[b + m - 1]];
            if (p2 == 0 || p2 == m - 1)
                d = inf;
            else if (hi2 > lo2 && d != inf)
                d = __dadd_rn(d, __ddiv_rn(__dsub_rn(err[oerr[q2 + 1]], err[oerr[q2 - 1]]),
                                           __dsub_rn(hi2, lo2)));
        }
        crowd_out[i] = d;
        front_out[i] = f;
    }
    for (int32_t f = tid; f <= F; f += kSmallThreads)
        offsets_out[f] = off[f];
    // 6. select_best(keep): whole fronts in ascending index order, the cut
    //    front by (crowding desc, index asc) (nsga.cpp:126-148)
    if (keep >= 0) {
        if (tid == 0) {
            int32_t c = 0;
            while (c < F && off[c + 1] <= keep)
                ++c;
            sCut = c;
        }
        __syncthreads();
        const int32_t c = sCut;
        const int32_t b = c < F ? off[c] : off[F];
        for (int32_t q = tid; q < min(b, keep); q += kSmallThreads)
            select_out[q] = members_out[q];
        __syncthreads(); // crowd_out / members_out visible to the block
        if (c < F) {
            const int32_t e = off[c + 1];
            for (int32_t q = b + tid; q < e; q += kSmallThreads) {
                const int32_t i = members_out[q];
                const double di = crowd_out[i];
                int32_t r = 0;
                for (int32_t u = b; u < e; ++u) {
                    const int32_t j = members_out[u];
                    const double dj = crowd_out[j];
                    r += dj > di || (dj == di && j < i);
                }
                if (b + r < keep)
                    select_out[b + r] = i;
            }
        }
        if (tid == 0)
            meta[kMetaCut] = c;
    }
    if (tid == 0) {
        meta[kMetaFronts] = F;
        meta[kMetaGroups] = meta[kMetaCosts] = meta[kMetaErrors] = 0; // (not computed here)
        meta[kMetaStrategy] = single_group ? 3 : 4; // 4: small-pool single-CTA path
    }
}

int bits_for(int32_t n) {
    int b = 1;
    while ((1ll << b) <= n)
        ++b;
    return b;
}

template <typename T>
T* carve(char*& p, size_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += (count * sizeof(T) + 255) & ~size_t(255);
    return r;
}

} // namespace

void rank_release(RankWorkspace& w) {
    if (w.mem)
        cudaFree(w.mem);
    if (w.cub)
        cudaFree(w.cub);
    w = RankWorkspace{};
}

cudaError_t rank_reserve(RankWorkspace& w, int32_t n) {
    if (n <= static_cast<int32_t>(w.cap) && w.mem)
        return cudaSuccess;
    rank_release(w);
    const size_t N = static_cast<size_t>(std::max(n, 1));
    const size_t bytes = 256 * 40 + N * (3 * 8 + 4 * 8 + 26 * 4) + 16 * 4;
    cudaError_t e = cudaMalloc(&w.mem, bytes);
    if (e != cudaSuccess)
        return e;
    char* p = static_cast<char*>(w.mem);
    // inputs, then every output in one span (one copy each way, see rank_impl)
    w.cost = carve<double>(p, N);
    w.err = carve<double>(p, N);
    w.crowd = carve<double>(p, N);
    w.front = carve<int32_t>(p, N);
    w.members = carve<int32_t>(p, N);
    w.offsets = carve<int32_t>(p, N + 1);
    w.select = carve<int32_t>(p, N);
    w.meta = carve<int32_t>(p, kMetaCount);
    w.kc = carve<uint64_t>(p, N);
    w.ke = carve<uint64_t>(p, N);
    w.k0 = carve<uint64_t>(p, N);
    w.k1 = carve<uint64_t>(p, N);
    w.seg = carve<int32_t>(p, 4);
    w.A = carve<int32_t>(p, N);
    w.B = carve<int32_t>(p, N);
    w.v0 = carve<int32_t>(p, N);
    w.v1 = carve<int32_t>(p, N);
    w.gid = carve<int32_t>(p, N);
    w.cpos = carve<int32_t>(p, N);
    w.epos = carve<int32_t>(p, N);
    w.posA = carve<int32_t>(p, N);
    w.grp_c = carve<int32_t>(p, N);
    w.grp_e = carve<int32_t>(p, N);
    w.gB = carve<int32_t>(p, N);
    w.lvl = carve<int32_t>(p, N + 1);
    w.fg = carve<int32_t>(p, N);
    w.pq = carve<int32_t>(p, N);
    w.uq = carve<int32_t>(p, N);
    w.stair = carve<int32_t>(p, N);
    w.ocost = carve<int32_t>(p, N);
    w.oerr = carve<int32_t>(p, N);
    w.pos_c = carve<int32_t>(p, N);
    w.pos_e = carve<int32_t>(p, N);
    w.cnt = carve<int32_t>(p, N + 1);
    // CUB temporary storage: the largest of the calls launch_rank makes
    const int ni = static_cast<int>(N);
    size_t b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0, b6 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b1, w.k0, w.k1, w.v0, w.v1, ni);
    cub::DeviceRadixSort::SortPairs(nullptr, b2, reinterpret_cast<uint32_t*>(w.k0),
                                    reinterpret_cast<uint32_t*>(w.k1), w.v0, w.v1, ni);
    cub::DeviceScan::InclusiveSum(nullptr, b3, w.gid, w.gid, ni);
    cub::DeviceScan::ExclusiveSum(nullptr, b4, w.cnt, w.offsets, ni + 1);
    cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, b5, w.k0, w.k1, w.members, w.v1, ni, 1,
                                                       w.seg, w.seg + 1);
    b6 = std::max({b1, b2, b3, b4, b5}) + 256;
    e = cudaMalloc(&w.cub, b6);
    if (e != cudaSuccess)
        return e;
    w.cub_bytes = b6;
    w.cap = N;
    return cudaSuccess;
}

cudaError_t launch_rank(RankWorkspace& w, int32_t n, bool single_group, int32_t keep, cudaStream_t s) {
    if (n <= 0) {
        return cudaMemsetAsync(w.meta, 0, kMetaCount * sizeof(int32_t), s);
    }
    if (n <= kSmallN) {
        const size_t smem = static_cast<size_t>(n) * 16 + (static_cast<size_t>(n) * 9 + 1) * 4;
        cudaError_t e = cudaFuncSetAttribute(rank_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess)
            return e;
        rank_small_kernel<<<1, kSmallThreads, smem, s>>>(w.cost, w.err, n, single_group, keep, w.front,
                                                         w.members, w.offsets, w.crowd, w.select, w.meta);
        return cudaGetLastError();
    }
    const int grid = (n + kThreads - 1) / kThreads;
    size_t tb = w.cub_bytes;
    cudaError_t e;
#define GEVO_TRY(x)                                                                                \
    do {                                                                                           \
        e = (x);                                                                                   \
        if (e != cudaSuccess)                                                                      \
            return e;                                                                              \
    } while (0)
    key_kernel<<<grid, kThreads, 0, s>>>(w.cost, w.err, n, w.kc, w.ke, w.v0);
    // A = (cost, error, index): by error, then stably by cost
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.ke, w.k1, w.v0, w.v1, n, 0, 64, s));
    gather_u64<<<grid, kThreads, 0, s>>>(w.kc, w.v1, n, w.k0);
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.v1, w.A, n, 0, 64, s));
    // B = (error, cost, index): A stably by error
    gather_u64<<<grid, kThreads, 0, s>>>(w.ke, w.A, n, w.k0);
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, w.k0, w.k1, w.A, w.B, n, 0, 64, s));
    // groups and dense ranks (pos_c / pos_e / stair double as scratch here)
    int32_t* bflag = w.stair;
    int32_t* posB = w.pos_e;
    flags_kernel<<<grid, kThreads, 0, s>>>(w.kc, w.ke, w.A, w.B, n, w.gid, w.cpos, w.epos, bflag,
                                           w.posA, posB);
    GEVO_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.gid, w.gid, n, s));
    GEVO_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.cpos, w.cpos, n, s));
    GEVO_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, w.epos, w.epos, n, s));
    GEVO_TRY(cub::DeviceScan::InclusiveSum(w.cub, tb, bflag, bflag, n, s));
    group_kernel<<<grid, kThreads, 0, s>>>(w.A, w.B, n, w.gid, w.cpos, w.epos, bflag, w.posA, posB,
                                           w.grp_c, w.grp_e, w.gB, w.meta);
    // fronts of the groups (one CTA)
    const size_t smem = kStairSmem * sizeof(int32_t);
    GEVO_TRY(cudaFuncSetAttribute(front_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    front_kernel<<<1, kFrontThreads, smem, s>>>(w.grp_c, w.grp_e, w.gB, single_group, w.lvl, w.pq,
                                                w.uq, w.stair, w.fg, w.meta);
    GEVO_TRY(cudaMemsetAsync(w.cnt, 0, (static_cast<size_t>(n) + 1) * sizeof(int32_t), s));
    scatter_front_kernel<<<grid, kThreads, 0, s>>>(w.A, w.gid, w.fg, n, w.front, w.cnt);
    GEVO_TRY(cub::DeviceScan::ExclusiveSum(w.cub, tb, w.cnt, w.offsets, n + 1, s));
    // members: indices stably sorted by front (ascending index per front)
    const int fb = bits_for(n);
    uint32_t* u0 = reinterpret_cast<uint32_t*>(w.k0);
    uint32_t* u1 = reinterpret_cast<uint32_t*>(w.k1);
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, reinterpret_cast<const uint32_t*>(w.front), u1,
                                             w.v0, w.members, n, 0, fb, s));
    // per-front cost / error orders: A and B stably sorted by front
    gather_u32<<<grid, kThreads, 0, s>>>(w.front, w.A, n, u0);
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, u0, u1, w.A, w.ocost, n, 0, fb, s));
    gather_u32<<<grid, kThreads, 0, s>>>(w.front, w.B, n, u0);
    GEVO_TRY(cub::DeviceRadixSort::SortPairs(w.cub, tb, u0, u1, w.B, w.oerr, n, 0, fb, s));
    pos_kernel<<<grid, kThreads, 0, s>>>(w.ocost, w.oerr, n, w.pos_c, w.pos_e);
    crowd_kernel<<<grid, kThreads, 0, s>>>(w.cost, w.err, w.front, w.offsets, w.ocost, w.oerr, w.pos_c,
                                           w.pos_e, n, w.crowd);
    if (keep >= 0) {
        cut_kernel<<<1, 1, 0, s>>>(w.offsets, keep, w.meta, w.seg);
        crowd_key_kernel<<<grid, kThreads, 0, s>>>(w.crowd, w.members, n, w.k0);
        GEVO_TRY(cub::DeviceSegmentedRadixSort::SortPairsDescending(
            w.cub, tb, w.k0, w.k1, w.members, w.v1, n, 1, w.seg, w.seg + 1, 0, 64, s));
        if (keep > 0)
            select_kernel<<<(keep + kThreads - 1) / kThreads, kThreads, 0, s>>>(w.members, w.v1, w.seg,
                                                                                 keep, w.select);
    }
#undef GEVO_TRY
    return cudaGetLastError();
}

} // namespace gevo
