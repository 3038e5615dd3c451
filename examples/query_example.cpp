// examples/query_example.cpp -- the reference-style C++ API on the GPU engine.
// Build (one line):  g++ -std=c++17 -O2 -Iinclude examples/query_example.cpp
//             -Lpaper_2108_10480_b200 -lsdgpu -Wl,-rpath,$PWD/paper_2108_10480_b200 -o query_example
// A unit-cube corner cloud plus one triangle; prints d_hat and grad for a few
// queries, exact and with the Barnes-Hut tree. Exit code 0 on success.
#include <cmath>
#include <cstdio>

#include "smoothdist_gpu.hpp"

using namespace smoothdist_gpu;

int main() {
    try {
        SimplexMesh m;
        for (int i = 0; i < 8; ++i) {
            m.vertices.push_back({double(i & 1), double((i >> 1) & 1), double((i >> 2) & 1)});
            m.simplices.push_back(Simplex::point(i));
        }
        m.vertices.push_back({3, 0, 0});
        m.vertices.push_back({3, 1, 0});
        m.vertices.push_back({3, 0, 1});
        m.simplices.push_back(Simplex::triangle(8, 9, 10));

        Engine eng(0, SD_FP64);
        eng.set_mesh(m);
        const WeightTable w = eng.build_weights();
        eng.build_bvh(SD_BVH_LBVH);
        std::printf("A = %g, %zu triangle polynomial(s), tree of %zu nodes\n", w.A, w.tri_stored.size() / 13,
                    eng.bvh().size());

        std::vector<Vec3> q = {{0.5, 0.5, 2.0}, {4.0, 0.2, 0.3}, {-3.0, -3.0, -3.0}};
        SmoothParams p;
        p.alpha = 50.0;
        p.beta = 0.0;
        const auto exact = eng.smooth_min_dist_flat(q, p);
        p.beta = 0.5;
        const auto tree = eng.smooth_min_dist(q, p);
        for (size_t i = 0; i < q.size(); ++i)
            std::printf("q%zu: exact d_hat %.9f grad (%.6f %.6f %.6f) | tree d_hat %.9f (%lld leaves, %lld far)\n", i,
                        exact[i].d_hat, exact[i].grad.x, exact[i].grad.y, exact[i].grad.z, tree[i].d_hat,
                        (long long)tree[i].leaves, (long long)tree[i].far_field);
        // conservativeness (acceptance [1]): tree field below the exact one
        for (size_t i = 0; i < q.size(); ++i)
            if (!(tree[i].d_hat <= exact[i].d_hat + 1e-9)) return 2;

        // query edges / triangles and a mesh-to-mesh distance
        const std::vector<SimplexGeom> g = {SimplexGeom::edge({0.5, 0.5, 2.0}, {0.5, 0.5, 3.0}),
                                            SimplexGeom::triangle({4, 0, 0}, {4, 1, 0}, {4, 0, 1})};
        const auto gs = eng.smooth_min_dist(g, p);
        for (size_t i = 0; i < g.size(); ++i)
            std::printf("g%zu (dim %d): d_hat %.9f grad (%.6f %.6f %.6f)\n", i, g[i].dim, gs[i].d_hat, gs[i].grad.x,
                        gs[i].grad.y, gs[i].grad.z);
        SimplexMesh qm;
        qm.vertices = {{4, 0, 0}, {4, 1, 0}, {4, 0, 1}, {0.5, 0.5, 2.0}};
        qm.simplices = {Simplex::triangle(0, 1, 2), Simplex::edge(2, 3)};
        p.alpha_q = 20.0;
        const auto md = eng.smooth_mesh_dist(qm, p);
        std::printf("mesh-to-mesh d_hat %.9f, vertex 0 grad (%.6f %.6f %.6f)\n", md.d_hat, md.vertex_grads[0].x,
                    md.vertex_grads[0].y, md.vertex_grads[0].z);
        return std::isfinite(exact[0].d_hat) ? 0 : 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
