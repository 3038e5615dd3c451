// weights_host.h -- host WeightSet precompute (build_adjacency +
// build_weight_set of the reference), see weights_host.cpp.
#pragma once

#include <cstdint>
#include <vector>

namespace sdgpu {

struct TriWeight {
    int v = 1, e = 1;
    double stored[13] = {};
    double sup = 1.0, inf = 1.0;
};

struct WeightTableHost {
    double A = 1.0, sup = 1.0;
    std::vector<double> edge_a;  // 5 per polynomial
    std::vector<double> edge_sup, edge_inf;
    std::vector<int32_t> edge_val;  // (valence0, valence1) per polynomial
    std::vector<TriWeight> tri;
    std::vector<int32_t> poly_index;
};

// Valence keys in first-occurrence order + per-simplex polynomial ids
// (gpu_weight_assignment in adjacency.cu computes them on the device).
struct WeightAssignment {
    std::vector<int32_t> poly_index;
    std::vector<std::pair<int32_t, int32_t>> edge_keys;  // (valence(v0), valence(v1))
    std::vector<std::pair<int32_t, int32_t>> tri_keys;   // (max vertex valence, max edge valence)
};

// Host reference pass (hash-map adjacency), kept for A/B checks.
WeightTableHost build_weight_table(const std::vector<int32_t>& simplices, const std::vector<uint8_t>& kinds,
                                   int64_t num_vertices);
// The polynomials of an assignment: closed-form edges, triangle LP per
// distinct (v, e) (memoised), A and sup w~ (weights.hpp:589-621).
WeightTableHost weight_table_from_assignment(const WeightAssignment& wa);
// edge polynomial coefficients and extrema (weights.hpp:46-76)
void edge_weight_poly(int n0, int n1, double a[5], double& sup, double& inf);

}  // namespace sdgpu
