// matchamg/matching.hpp — compatible weighted matching (reference
// matching.hpp:22-65). build_weights and suitor_match run on the B200; the
// exhaustive oracle stays a host routine (a test oracle, n <= 20).
#ifndef MATCHAMG_B200_MATCHING_HPP
#define MATCHAMG_B200_MATCHING_HPP

#include <span>
#include <vector>

#include "matchamg/csr.hpp"

namespace matchamg {

inline constexpr index_t kUnmatched = -1;

// off-diagonal pattern of A with c_ij = 1 - 2 a_ij w_i w_j / (a_ii w_i^2 + a_jj w_j^2)
struct WeightedGraph {
    index_t n = 0;
    std::vector<index_t> xadj{0};
    std::vector<index_t> adjncy;
    std::vector<double> weight;
    long zero_weight_edges = 0;

    index_t degree(index_t v) const { return xadj[v + 1] - xadj[v]; }
};

struct Matching {
    std::vector<index_t> mate; // mate[i] = j or kUnmatched

    index_t matched_vertices() const;
    bool is_valid() const;
};

WeightedGraph build_weights(const CsrMatrix& A, std::span<const double> w);
// Suitor under the strict edge order (weight desc, then smaller endpoint
// pair); equals the greedy matching, hence identical for every schedule.
Matching suitor_match(const WeightedGraph& G);
Matching exact_match_oracle(const WeightedGraph& G);
double matching_weight(const WeightedGraph& G, const Matching& M);

} // namespace matchamg

#endif
