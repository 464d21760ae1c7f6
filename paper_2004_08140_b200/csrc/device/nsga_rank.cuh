// GPU rank_population / select_best: workspace and launcher.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace gevo {

// Scalars the ranking leaves on the device (RankWorkspace::meta).
enum RankMeta : int {
    kMetaFronts = 0,   // number of fronts F
    kMetaGroups = 1,   // distinct (cost, error) points g
    kMetaCosts = 2,    // distinct costs C
    kMetaErrors = 3,   // distinct errors D
    kMetaStrategy = 4, // 0 = cost levels, 1 = error levels, 2 = staircase, 3 = single group
    kMetaCut = 5,      // select_best: the front that is cut (F when none is)
    kMetaCount = 8,
};

// Device buffers of one ranking. Grown on demand, owned by the caller's
// device context; every array is [n] unless noted.
struct RankWorkspace {
    size_t cap = 0;         // n the buffers are sized for
    void* mem = nullptr;    // one allocation holding everything below
    void* cub = nullptr;    // CUB temporary storage
    size_t cub_bytes = 0;

    double* cost = nullptr; // inputs (the caller copies them in)
    double* err = nullptr;
    double* crowd = nullptr;      // output: crowding distance per individual
    int32_t* front = nullptr;     // output: front per individual
    int32_t* members = nullptr;   // output: front members, ascending index per front
    int32_t* offsets = nullptr;   // output: [n + 1] front f = members[offsets[f], offsets[f+1])
    int32_t* select = nullptr;    // output: select_best(rank, keep) order
    int32_t* meta = nullptr;      // output: [kMetaCount] scalars

    // scratch
    uint64_t *kc, *ke, *k0, *k1;
    int32_t *A, *B, *v0, *v1, *gid, *cpos, *epos, *posA, *grp_c, *grp_e, *gB, *lvl, *fg, *pq,
        *uq, *stair, *ocost, *oerr, *pos_c, *pos_e, *cnt, *seg;
};

// Reserve buffers for n individuals (cudaMalloc; no-op when large enough).
cudaError_t rank_reserve(RankWorkspace& w, int32_t n);
void rank_release(RankWorkspace& w);

// Ranks ws.cost/ws.err[0..n) on stream s (src/nsga.cpp:88-106): fronts
// (nondominated_sort, nsga.cpp:15-46) and crowding (nsga.cpp:48-86). With
// single_group the whole input is one front (crowding_distance()). With
// keep >= 0 also writes select_best(rank, keep) (nsga.cpp:126-148) to
// ws.select. Everything stays on the device; no host synchronisation.
cudaError_t launch_rank(RankWorkspace& w, int32_t n, bool single_group, int32_t keep,
                        cudaStream_t s);

} // namespace gevo
