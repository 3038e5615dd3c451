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
    std::vector<double> edge_sup;
    std::vector<TriWeight> tri;
    std::vector<int32_t> poly_index;
};

WeightTableHost build_weight_table(const std::vector<int32_t>& simplices, const std::vector<uint8_t>& kinds,
                                   int64_t num_vertices);

}  // namespace sdgpu
