// GPU NSGA-II ranking over (cost, error): non-dominated fronts and crowding
// distance, bit-identical to src/nsga.cpp:9-106 of arxiv/paper_2004_08140.
//
// Fronts: with two objectives the peeling rank of a point equals the length of
// its longest dominance chain. After a lexicographic (cost, error, index)
// order, every dominator of a point precedes it, and the per-rank minimum
// error forms a non-decreasing staircase, so rank = upper_bound(staircase, e);
// runs of identical points share a rank (they do not dominate each other).
// The partition is unique, so it equals the reference's O(n^2) peel; members
// are listed in ascending index order like the reference (nsga.cpp:32-43).
//
// Crowding: per front and objective, the reference sorts by (key, other key,
// index), sets both ends to +inf, skips +inf entries and adds
// (key[i+1] - key[i-1]) / (hi - lo), cost objective first (nsga.cpp:48-86).
// Each member's position in both orders is a rank count inside its front, then
// the same double operations are replayed per member.
#include "nsga_rank.cuh"

#include <cuda_runtime.h>

namespace gevo {

namespace {

struct Key {
    double a, b;
    int32_t i;
};

__device__ __forceinline__ bool key_less(double a0, double b0, int32_t i0, double a1, double b1,
                                         int32_t i1) {
    if (a0 != a1)
        return a0 < a1;
    if (b0 != b1)
        return b0 < b1;
    return i0 < i1;
}

// pos[i] = number of j with (cost, err, j) < (cost_i, err_i, i); order[pos] = i.
__global__ void lex_rank_kernel(const double* __restrict__ cost, const double* __restrict__ err,
                                int32_t n, int32_t* __restrict__ order) {
    extern __shared__ double tile[];
    double* tc = tile;
    double* te = tile + blockDim.x;
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const double ci = i < n ? cost[i] : 0.0, ei = i < n ? err[i] : 0.0;
    int32_t pos = 0;
    for (int32_t base = 0; base < n; base += blockDim.x) {
        const int32_t j = base + threadIdx.x;
        tc[threadIdx.x] = j < n ? cost[j] : 0.0;
        te[threadIdx.x] = j < n ? err[j] : 0.0;
        __syncthreads();
        const int32_t m = min(static_cast<int32_t>(blockDim.x), n - base);
        for (int32_t k = 0; k < m; ++k)
            pos += key_less(tc[k], te[k], base + k, ci, ei, i) ? 1 : 0;
        __syncthreads();
    }
    if (i < n)
        order[pos] = i;
}

// Staircase scan over the lexicographic order (one thread; O(n log F)).
__global__ void front_scan_kernel(const double* __restrict__ cost, const double* __restrict__ err,
                                  const int32_t* __restrict__ order, int32_t n,
                                  double* __restrict__ stair, int32_t* __restrict__ front,
                                  int32_t* __restrict__ n_fronts) {
    if (blockIdx.x != 0 || threadIdx.x != 0)
        return;
    int32_t F = 0;
    int32_t g = 0;
    while (g < n) {
        const int32_t first = order[g];
        const double c = cost[first], e = err[first];
        int32_t h = g + 1;
        while (h < n && cost[order[h]] == c && err[order[h]] == e)
            ++h;
        // upper_bound: first level whose minimum error exceeds e
        int32_t lo = 0, hi = F;
        while (lo < hi) {
            const int32_t mid = (lo + hi) >> 1;
            if (stair[mid] <= e)
                lo = mid + 1;
            else
                hi = mid;
        }
        const int32_t r = lo;
        for (int32_t k = g; k < h; ++k)
            front[order[k]] = r;
        if (r == F)
            stair[F++] = e;
        else
            stair[r] = e;
        g = h;
    }
    *n_fronts = F;
}

// Front sizes, offsets and ascending-index member lists (one thread; O(n)).
__global__ void front_lists_kernel(const int32_t* __restrict__ front, int32_t n,
                                   const int32_t* __restrict__ n_fronts,
                                   int32_t* __restrict__ offsets, int32_t* __restrict__ fill,
                                   int32_t* __restrict__ members) {
    if (blockIdx.x != 0 || threadIdx.x != 0)
        return;
    const int32_t F = *n_fronts;
    for (int32_t f = 0; f <= F; ++f)
        offsets[f] = 0;
    for (int32_t i = 0; i < n; ++i)
        offsets[front[i] + 1] += 1;
    for (int32_t f = 0; f < F; ++f) {
        offsets[f + 1] += offsets[f];
        fill[f] = 0;
    }
    for (int32_t i = 0; i < n; ++i) {
        const int32_t f = front[i];
        members[offsets[f] + fill[f]++] = i;
    }
}

// Position of each member in its front's cost-order and error-order.
__global__ void crowd_order_kernel(const double* __restrict__ cost, const double* __restrict__ err,
                                   const int32_t* __restrict__ front,
                                   const int32_t* __restrict__ offsets,
                                   const int32_t* __restrict__ members, int32_t n,
                                   int32_t* __restrict__ ord_cost, int32_t* __restrict__ ord_err) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int32_t f = front[i];
    const int32_t b = offsets[f], e = offsets[f + 1];
    const double ci = cost[i], ei = err[i];
    int32_t p1 = 0, p2 = 0;
    for (int32_t k = b; k < e; ++k) {
        const int32_t j = members[k];
        const double cj = cost[j], ej = err[j];
        // the reference sorts members by their position inside the front,
        // which is ascending index order, so the index tie-break is j < i
        p1 += key_less(cj, ej, j, ci, ei, i) ? 1 : 0;
        p2 += key_less(ej, cj, j, ei, ci, i) ? 1 : 0;
    }
    ord_cost[b + p1] = i;
    ord_err[b + p2] = i;
}

__global__ void crowd_kernel(const double* __restrict__ cost, const double* __restrict__ err,
                             const int32_t* __restrict__ front, const int32_t* __restrict__ offsets,
                             const int32_t* __restrict__ ord_cost,
                             const int32_t* __restrict__ ord_err, int32_t n,
                             double* __restrict__ crowd) {
    const int32_t f_idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (f_idx >= n)
        return;
    // one thread per slot of the cost order; find its member
    const int32_t i = ord_cost[f_idx];
    const int32_t f = front[i];
    const int32_t b = offsets[f], m = offsets[f + 1] - b;
    const double inf = __longlong_as_double(0x7ff0000000000000LL);
    if (m <= 2) {
        crowd[i] = inf;
        return;
    }
    const int32_t p1 = f_idx - b;
    double d = 0.0;
    const double lo1 = cost[ord_cost[b]], hi1 = cost[ord_cost[b + m - 1]];
    if (p1 == 0 || p1 == m - 1)
        d = inf;
    else if (hi1 > lo1)
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(cost[ord_cost[f_idx + 1]], cost[ord_cost[f_idx - 1]]),
                                   __dsub_rn(hi1, lo1)));
    // position in the error order
    int32_t p2 = 0;
    for (int32_t k = 0; k < m; ++k)
        if (ord_err[b + k] == i) {
            p2 = k;
            break;
        }
    const double lo2 = err[ord_err[b]], hi2 = err[ord_err[b + m - 1]];
    if (p2 == 0 || p2 == m - 1)
        d = inf;
    else if (hi2 > lo2 && d != inf)
        d = __dadd_rn(d, __ddiv_rn(__dsub_rn(err[ord_err[b + p2 + 1]], err[ord_err[b + p2 - 1]]),
                                   __dsub_rn(hi2, lo2)));
    crowd[i] = d;
}

__global__ void single_group_kernel(int32_t n, int32_t* front, int32_t* n_fronts) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        front[i] = 0;
    if (i == 0)
        *n_fronts = n > 0 ? 1 : 0;
}

} // namespace

cudaError_t launch_rank(const RankBuffers& B, int32_t n, bool single_group, cudaStream_t s) {
    if (n <= 0)
        return cudaSuccess;
    const int threads = 256;
    const int grid = (n + threads - 1) / threads;
    if (single_group) {
        single_group_kernel<<<grid, threads, 0, s>>>(n, B.front, B.n_fronts);
    } else {
        lex_rank_kernel<<<grid, threads, 2 * threads * sizeof(double), s>>>(B.cost, B.err, n,
                                                                            B.order);
        front_scan_kernel<<<1, 1, 0, s>>>(B.cost, B.err, B.order, n, B.stair, B.front, B.n_fronts);
    }
    front_lists_kernel<<<1, 1, 0, s>>>(B.front, n, B.n_fronts, B.offsets, B.fill, B.members);
    crowd_order_kernel<<<grid, threads, 0, s>>>(B.cost, B.err, B.front, B.offsets, B.members, n,
                                                B.ord_cost, B.ord_err);
    crowd_kernel<<<grid, threads, 0, s>>>(B.cost, B.err, B.front, B.offsets, B.ord_cost, B.ord_err,
                                          n, B.crowd);
    return cudaGetLastError();
}

} // namespace gevo
