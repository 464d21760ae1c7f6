// GPU rank_population buffers and launcher.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace gevo {

struct RankBuffers {
    const double* cost; // [n]
    const double* err;  // [n]
    int32_t* order;     // [n] lexicographic order
    double* stair;      // [n] staircase minima
    int32_t* front;     // [n] front index per individual (output)
    int32_t* n_fronts;  // [1] (output)
    int32_t* offsets;   // [n + 1] front offsets into members (output)
    int32_t* fill;      // [n]
    int32_t* members;   // [n] front members, ascending index per front (output)
    int32_t* ord_cost;  // [n]
    int32_t* ord_err;   // [n]
    double* crowd;      // [n] crowding distance (output)
};

// single_group: treat the whole input as one front (crowding_distance()).
cudaError_t launch_rank(const RankBuffers& B, int32_t n, bool single_group, cudaStream_t s);

} // namespace gevo
