// NSGA-II entry points. Ranking (fronts + crowding) runs on the GPU
// (csrc/device/nsga_rank.cu); the RNG-consuming tournament and the truncation
// order stay on the host with the reference's exact rules
// (src/nsga.cpp:9-13 dominance, 108-124 tournament, 126-148 truncation of
// arxiv/paper_2004_08140).
#include "runtime.hpp"

#include <algorithm>
#include <cassert>

namespace evoir {

bool dominates(const FitnessVector& a, const FitnessVector& b) {
    if (a.cost > b.cost || a.error > b.error)
        return false;
    return a.cost < b.cost || a.error < b.error;
}

ParetoRank rank_population(const std::vector<FitnessVector>& fits) {
    return b200::rank_on_device(b200::Device::default_device(), fits, false);
}

std::vector<std::vector<int>> nondominated_sort(const std::vector<FitnessVector>& fits) {
    return rank_population(fits).fronts;
}

std::vector<double> crowding_distance(const std::vector<FitnessVector>& front) {
    return b200::rank_on_device(b200::Device::default_device(), front, true).crowding;
}

std::vector<int> tournament_select(const ParetoRank& rank, size_t pop_size, size_t k, Rng& rng) {
    std::vector<int> winners;
    winners.reserve(k);
    for (size_t n = 0; n < k; ++n) {
        const int a = static_cast<int>(rng.index(pop_size));
        const int b = static_cast<int>(rng.index(pop_size));
        const size_t ua = static_cast<size_t>(a), ub = static_cast<size_t>(b);
        int w;
        if (rank.front[ua] != rank.front[ub])
            w = rank.front[ua] < rank.front[ub] ? a : b;
        else if (rank.crowding[ua] != rank.crowding[ub])
            w = rank.crowding[ua] > rank.crowding[ub] ? a : b;
        else
            w = rng.index(2) == 0 ? a : b;
        winners.push_back(w);
    }
    return winners;
}

std::vector<int> select_best(const ParetoRank& rank, size_t n) {
    assert(n <= rank.front.size());
    std::vector<int> keep;
    keep.reserve(n);
    for (const std::vector<int>& f : rank.fronts) {
        if (keep.size() + f.size() <= n) {
            keep.insert(keep.end(), f.begin(), f.end());
            if (keep.size() == n)
                break;
            continue;
        }
        std::vector<int> part = f;
        std::sort(part.begin(), part.end(), [&](int x, int y) {
            const double cx = rank.crowding[static_cast<size_t>(x)];
            const double cy = rank.crowding[static_cast<size_t>(y)];
            return cx != cy ? cx > cy : x < y;
        });
        part.resize(n - keep.size());
        keep.insert(keep.end(), part.begin(), part.end());
        break;
    }
    return keep;
}

} // namespace evoir
