// NSGA-II over (cost, error) (reference: include/evoir/nsga.hpp:12-41 of
// arxiv/paper_2004_08140). rank_population runs on the GPU
// (csrc/device/nsga_rank.cu); the RNG-consuming selection stays on the host.
#pragma once

#include "evoir/rng.hpp"
#include "evoir/vm.hpp"

#include <vector>

namespace evoir {

bool dominates(const FitnessVector& a, const FitnessVector& b);
std::vector<std::vector<int>> nondominated_sort(const std::vector<FitnessVector>& fits);
std::vector<double> crowding_distance(const std::vector<FitnessVector>& front);

struct ParetoRank {
    std::vector<int> front;
    std::vector<double> crowding;
    std::vector<std::vector<int>> fronts;
};

ParetoRank rank_population(const std::vector<FitnessVector>& fits);
std::vector<int> tournament_select(const ParetoRank& rank, size_t pop_size, size_t k, Rng& rng);
std::vector<int> select_best(const ParetoRank& rank, size_t n);

} // namespace evoir
