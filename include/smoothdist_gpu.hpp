// include/smoothdist_gpu.hpp -- C++ front end of the B200 engine, keeping the
// reference's names and value types (/root/reference/proj/include/smoothdist:
// SimplexMesh/Simplex mesh.hpp:15-50, SmoothParams params.hpp:13-22,
// SmoothResult smooth.hpp:20-27, BvhNode bvh.hpp:14-22) on top of the C ABI
// in sdgpu.h. Header-only; link with libsdgpu.so.
//
//   smoothdist_gpu::Engine eng(/*device*/ 0, SD_FP32);
//   eng.set_mesh(mesh);                 // SimplexMesh
//   eng.build_weights();                // build_weight_set(mesh, build_adjacency(mesh))
//   eng.build_bvh(SD_BVH_LBVH);         // or set_bvh(reference_tree)
//   auto r = eng.smooth_min_dist(queries, params);      // one call per batch
//   auto e = eng.smooth_min_dist_flat(queries, params); // exact (beta ignored)
//   auto g = eng.smooth_min_dist(simplex_geoms, params); // query edges / triangles
//   auto m = eng.smooth_mesh_dist(query_mesh, params);   // mesh-to-mesh
//
// Failures throw std::runtime_error, as the reference's fail() does
// (common.hpp:50); the evaluator semantics are the reference's (+inf and a
// zero gradient on underflow, never an error).
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "sdgpu.h"

namespace smoothdist_gpu {

// Same 24-byte layout as Eigen::Vector3d, so SimplexMesh::vertices.data()
// of the reference converts with a reinterpret_cast.
struct Vec3 {
    double x = 0, y = 0, z = 0;
};
static_assert(sizeof(Vec3) == 24, "Vec3 must be three packed doubles");

enum class SimplexKind : std::uint8_t { Point = 0, Edge = 1, Triangle = 2 };

struct Simplex {
    std::int32_t v[3] = {-1, -1, -1};
    SimplexKind kind = SimplexKind::Point;
    static Simplex point(std::int32_t a) { return {{a, -1, -1}, SimplexKind::Point}; }
    static Simplex edge(std::int32_t a, std::int32_t b) { return {{a, b, -1}, SimplexKind::Edge}; }
    static Simplex triangle(std::int32_t a, std::int32_t b, std::int32_t c) { return {{a, b, c}, SimplexKind::Triangle}; }
};

struct SimplexMesh {
    std::vector<Vec3> vertices;
    std::vector<Simplex> simplices;
};

// A query simplex by its corners (exact.hpp:24-41): dim 0 point, 1 edge,
// 2 triangle; corners past dim are ignored.
struct SimplexGeom {
    Vec3 c[3];
    int dim = 0;
    static SimplexGeom point(Vec3 a) { return {{a, {}, {}}, 0}; }
    static SimplexGeom edge(Vec3 a, Vec3 b) { return {{a, b, {}}, 1}; }
    static SimplexGeom triangle(Vec3 a, Vec3 b, Vec3 c) { return {{a, b, c}, 2}; }
};

struct SmoothParams {
    double alpha = 100.0, alpha_u = 600.0, beta = 0.5, alpha_q = 100.0, epsilon = 1e-300;
    double attenuation() const { return alpha / (alpha > alpha_u ? alpha : alpha_u); }
};

struct SmoothResult {
    double d_hat = std::numeric_limits<double>::infinity();
    Vec3 grad;
    double c = 0.0;
    Vec3 grad_c;
    std::int64_t leaves = 0, far_field = 0;
    std::uint64_t decision_hash = 0;
};

// WeightSet as flat arrays (weights.hpp:565-579).
struct WeightTable {
    double A = 1.0, sup_wtilde = 1.0;
    std::vector<double> edge_a;      // 5 per edge polynomial
    std::vector<double> tri_stored;  // 13 per triangle polynomial
    std::vector<std::int32_t> poly_index;
};

using BvhNode = sd_bvh_node;  // byte-compatible with the reference BvhNode

inline void check(int rc) {
    if (rc != SD_OK) throw std::runtime_error(std::string("sdgpu: ") + sd_last_error());
}

class Engine {
public:
    explicit Engine(int device = 0, int precision = SD_FP32) { check(sd_create(&ctx_, device, precision)); }
    ~Engine() {
        if (ctx_) sd_destroy(ctx_);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    sd_ctx* handle() const { return ctx_; }

    void set_mesh(const SimplexMesh& m) {
        std::vector<std::int32_t> sv(3 * m.simplices.size());
        std::vector<std::uint8_t> kind(m.simplices.size());
        for (size_t i = 0; i < m.simplices.size(); ++i) {
            for (int k = 0; k < 3; ++k) sv[3 * i + k] = m.simplices[i].v[k];
            kind[i] = static_cast<std::uint8_t>(m.simplices[i].kind);
        }
        check(sd_set_geometry(ctx_, reinterpret_cast<const double*>(m.vertices.data()),
                              static_cast<std::int64_t>(m.vertices.size()), sv.data(), kind.data(),
                              static_cast<std::int64_t>(kind.size())));
        n_ = kind.size();
    }

    void set_weights(const WeightTable& w) {
        check(sd_set_weights(ctx_, w.A, w.sup_wtilde, static_cast<std::int32_t>(w.edge_a.size() / 5), w.edge_a.data(),
                             static_cast<std::int32_t>(w.tri_stored.size() / 13), w.tri_stored.data(),
                             w.poly_index.data()));
    }

    WeightTable build_weights() {
        check(sd_build_weights(ctx_));
        return weights();
    }

    WeightTable weights() const {
        WeightTable w;
        std::int32_t ne = 0, nt = 0;
        check(sd_weights_info(ctx_, &w.A, &w.sup_wtilde, &ne, &nt));
        w.edge_a.resize(5 * size_t(ne));
        w.tri_stored.resize(13 * size_t(nt));
        w.poly_index.resize(n_);
        check(sd_export_weights(ctx_, w.edge_a.data(), w.tri_stored.data(), w.poly_index.data()));
        return w;
    }

    // sd_set_exact_pruning: 0 (default) sums every pair like smooth_min_dist_flat
    void set_exact_pruning(double bits) { check(sd_set_exact_pruning(ctx_, bits)); }

    void build_bvh(int method = SD_BVH_LBVH) { check(sd_build_bvh(ctx_, method)); }
    void set_bvh(const std::vector<BvhNode>& nodes) {
        check(sd_set_bvh(ctx_, nodes.data(), static_cast<std::int64_t>(nodes.size())));
    }
    std::vector<BvhNode> bvh() const {
        std::int64_t n = 0;
        check(sd_bvh_size(ctx_, &n));
        std::vector<BvhNode> out(static_cast<size_t>(n));
        check(sd_export_bvh(ctx_, out.data(), n));
        return out;
    }

    // smooth_min_dist (smooth.hpp:166-184) for a batch: tree path when beta > 0.
    std::vector<SmoothResult> smooth_min_dist(const std::vector<Vec3>& q, const SmoothParams& p) {
        return run(q, p, p.beta > 0.0 ? SD_BVH : SD_EXACT);
    }
    // smooth_min_dist (smooth.hpp:166-184) / _flat (:189-198) for a batch of
    // query SIMPLICES (points, edges, triangles); fp64 on the device.
    std::vector<SmoothResult> smooth_min_dist(const std::vector<SimplexGeom>& g, const SmoothParams& p) {
        return run_simplices(g, p, p.beta > 0.0 ? SD_BVH : SD_EXACT);
    }
    std::vector<SmoothResult> smooth_min_dist_flat(const std::vector<SimplexGeom>& g, const SmoothParams& p) {
        return run_simplices(g, p, SD_EXACT);
    }

    // smooth_mesh_dist (smooth.hpp:212-255) for any query mesh.
    struct MeshDistResult {
        double d_hat = std::numeric_limits<double>::infinity();
        std::vector<Vec3> vertex_grads;
        std::vector<double> per_primitive;
    };
    MeshDistResult smooth_mesh_dist(const SimplexMesh& query, const SmoothParams& p) {
        std::vector<std::int32_t> sv(3 * query.simplices.size());
        std::vector<std::uint8_t> kind(query.simplices.size());
        for (size_t j = 0; j < query.simplices.size(); ++j) {
            for (int k = 0; k < 3; ++k) sv[3 * j + k] = query.simplices[j].v[k];
            kind[j] = static_cast<std::uint8_t>(query.simplices[j].kind);
        }
        MeshDistResult r;
        r.vertex_grads.resize(query.vertices.size());
        r.per_primitive.resize(kind.size());
        const sd_params sp{p.alpha, p.alpha_u, p.beta, p.epsilon};
        check(sd_mesh_dist(ctx_, reinterpret_cast<const double*>(query.vertices.data()),
                           static_cast<std::int64_t>(query.vertices.size()), sv.data(), kind.data(),
                           static_cast<std::int64_t>(kind.size()), &sp, p.alpha_q, p.beta > 0 ? SD_BVH : SD_EXACT,
                           &r.d_hat, reinterpret_cast<double*>(r.vertex_grads.data()), r.per_primitive.data()));
        return r;
    }

    // smooth_min_dist_flat (smooth.hpp:189-198) for a batch.
    std::vector<SmoothResult> smooth_min_dist_flat(const std::vector<Vec3>& q, const SmoothParams& p) {
        return run(q, p, SD_EXACT);
    }

private:
    std::vector<SmoothResult> run(const std::vector<Vec3>& q, const SmoothParams& p, int mode) {
        const size_t n = q.size();
        std::vector<double> d(n), c(n), g(3 * n), gc(3 * n);
        std::vector<std::int64_t> leaves(n), far(n);
        std::vector<std::uint64_t> hash(n);
        sd_outputs o{d.data(), g.data(), c.data(), gc.data(), leaves.data(), far.data(), hash.data()};
        const sd_params sp{p.alpha, p.alpha_u, p.beta, p.epsilon};
        check(sd_query_points(ctx_, reinterpret_cast<const double*>(q.data()), static_cast<std::int64_t>(n), &sp, mode,
                              &o));
        std::vector<SmoothResult> out(n);
        for (size_t i = 0; i < n; ++i) {
            out[i].d_hat = d[i];
            out[i].grad = {g[3 * i], g[3 * i + 1], g[3 * i + 2]};
            out[i].c = c[i];
            out[i].grad_c = {gc[3 * i], gc[3 * i + 1], gc[3 * i + 2]};
            out[i].leaves = leaves[i];
            out[i].far_field = far[i];
            out[i].decision_hash = hash[i];
        }
        return out;
    }

    std::vector<SmoothResult> run_simplices(const std::vector<SimplexGeom>& g, const SmoothParams& p, int mode) {
        const size_t n = g.size();
        std::vector<double> corners(9 * n, 0.0), d(n), c(n), gr(3 * n), gc(3 * n);
        std::vector<std::int32_t> dims(n);
        std::vector<std::int64_t> leaves(n), far(n);
        std::vector<std::uint64_t> hash(n);
        for (size_t i = 0; i < n; ++i) {
            dims[i] = g[i].dim;
            for (int k = 0; k < 3; ++k) {
                corners[9 * i + 3 * k] = g[i].c[k].x;
                corners[9 * i + 3 * k + 1] = g[i].c[k].y;
                corners[9 * i + 3 * k + 2] = g[i].c[k].z;
            }
        }
        sd_outputs o{d.data(), gr.data(), c.data(), gc.data(), leaves.data(), far.data(), hash.data()};
        const sd_params sp{p.alpha, p.alpha_u, p.beta, p.epsilon};
        check(sd_query_simplices(ctx_, corners.data(), dims.data(), static_cast<std::int64_t>(n), &sp, mode, &o));
        std::vector<SmoothResult> out(n);
        for (size_t i = 0; i < n; ++i) {
            out[i].d_hat = d[i];
            out[i].grad = {gr[3 * i], gr[3 * i + 1], gr[3 * i + 2]};
            out[i].c = c[i];
            out[i].grad_c = {gc[3 * i], gc[3 * i + 1], gc[3 * i + 2]};
            out[i].leaves = leaves[i];
            out[i].far_field = far[i];
            out[i].decision_hash = hash[i];
        }
        return out;
    }

    sd_ctx* ctx_ = nullptr;
    size_t n_ = 0;
};

}  // namespace smoothdist_gpu
