// include/smoothdist_gpu_backend.hpp -- the drop-in for the REFERENCE'S OWN
// types: include it next to the reference's <smoothdist/smooth.hpp>
// (/root/reference/proj/include) and link libsdgpu.so. Every call takes
// and returns the reference's values -- SimplexMesh (mesh.hpp:31-50), Bvh
// (bvh.hpp:14-32), WeightSet (weights.hpp:565-579), SmoothParams
// (params.hpp:13-22), SimplexGeom (exact.hpp:24-41), SmoothResult
// (smooth.hpp:20-27), MeshDistResult (smooth.hpp:205-210) -- and replaces a
// per-query loop of the reference's evaluator with one batched call:
//
//   smooth_min_dist(mesh, bvh, ws, q, params)      (smooth.hpp:166-184)
//   smooth_min_dist_flat(mesh, ws, g, params)      (smooth.hpp:189-198)
//   smooth_mesh_dist(mesh, bvh, ws, query, params) (smooth.hpp:212-255)
//
//   smoothdist::gpu::Backend gpu(/*device*/ 0, SD_FP64);
//   gpu.upload(mesh, ws, &bvh);            // same node ids -> comparable counters
//   auto r = gpu.smooth_min_dist(points, params);   // std::vector<SmoothResult>
//
// Layout facts it relies on (checked at compile time): Vec3 is 24
// contiguous bytes (Eigen::Vector3d), so SimplexMesh::vertices.data() is
// the C ABI's xyz array; BvhNode is byte-identical to sd_bvh_node (the
// record save_bvh_cache writes, bvh.hpp:193-212). Errors go through the
// reference's fail() (common.hpp:50), i.e. std::runtime_error.
#pragma once

#include <smoothdist/smooth.hpp>

#include <cstdint>
#include <vector>

#include "sdgpu.h"

namespace smoothdist::gpu {

static_assert(sizeof(Vec3) == 3 * sizeof(double), "Vec3 must be three packed doubles");
static_assert(sizeof(BvhNode) == sizeof(sd_bvh_node), "BvhNode must match sd_bvh_node");

class Backend {
  public:
    explicit Backend(int device, int precision = SD_FP32) {
        if (sd_create(&ctx_, device, precision)) fail(sd_last_error());
    }
    ~Backend() { sd_destroy(ctx_); }
    Backend(const Backend&) = delete;
    Backend& operator=(const Backend&) = delete;

    // Geometry + WeightSet (+ the reference's tree; nullptr builds one on
    // the GPU: SD_BVH_AUTO, the median split of build_bvh or the LBVH,
    // whichever has the smaller surface-area cost).
    void upload(const SimplexMesh& m, const WeightSet& ws, const Bvh* tree) {
        const std::size_t n = m.simplices.size();
        std::vector<std::int32_t> sv(3 * n);
        std::vector<std::uint8_t> kind(n);
        for (std::size_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) sv[3 * i + k] = m.simplices[i].v[std::size_t(k)];
            kind[i] = std::uint8_t(m.simplices[i].kind);
        }
        if (sd_set_geometry(ctx_, m.vertices.data()->data(), std::int64_t(m.vertices.size()), sv.data(), kind.data(),
                            std::int64_t(n)))
            fail(sd_last_error());
        std::vector<double> ea, ts;
        for (const auto& p : ws.edge_polys) ea.insert(ea.end(), p.a.begin(), p.a.end());
        for (const auto& p : ws.tri_polys) ts.insert(ts.end(), p.stored.begin(), p.stored.end());
        if (sd_set_weights(ctx_, ws.A, ws.sup_wtilde, std::int32_t(ws.edge_polys.size()), ea.data(),
                           std::int32_t(ws.tri_polys.size()), ts.data(), ws.poly_index.data()))
            fail(sd_last_error());
        if (tree) {
            if (sd_set_bvh(ctx_, reinterpret_cast<const sd_bvh_node*>(tree->nodes.data()),
                           std::int64_t(tree->nodes.size())))
                fail(sd_last_error());
        } else if (sd_build_bvh(ctx_, SD_BVH_AUTO)) {
            fail(sd_last_error());
        }
    }

    // Pruned exact evaluation (sd_set_exact_pruning; 0 = the reference's sum
    // over all pairs, the default): smooth_min_dist_flat skips primitive
    // tiles whose terms are below 2^-bits of a lower bound of the sum.
    void set_exact_pruning(double bits) {
        if (sd_set_exact_pruning(ctx_, bits)) fail(sd_last_error());
    }

    // The tree the engine traverses, as the reference's Bvh.
    Bvh tree() const {
        std::int64_t n = 0;
        if (sd_bvh_size(ctx_, &n)) fail(sd_last_error());
        Bvh b;
        b.nodes.resize(std::size_t(n));
        if (sd_export_bvh(ctx_, reinterpret_cast<sd_bvh_node*>(b.nodes.data()), n)) fail(sd_last_error());
        return b;
    }

    // A batch of smooth_min_dist(mesh, bvh, ws, q, params) (beta > 0: the
    // tree path, as the reference's collect_contributions decides) or of
    // smooth_min_dist_flat (exact = true, or beta == 0).
    std::vector<SmoothResult> smooth_min_dist(const std::vector<Vec3>& q, const SmoothParams& p,
                                              bool exact = false) const {
        const std::size_t n = q.size();
        std::vector<double> d(n), g(3 * n), c(n), gc(3 * n);
        std::vector<std::int64_t> leaves(n), far(n);
        sd_outputs o{d.data(), g.data(), c.data(), gc.data(), leaves.data(), far.data(), nullptr};
        const sd_params sp = params(p);
        const int mode = (exact || !(p.beta > 0.0)) ? SD_EXACT : SD_BVH;
        if (n && sd_query_points(ctx_, q.data()->data(), std::int64_t(n), &sp, mode, &o)) fail(sd_last_error());
        std::vector<SmoothResult> out(n);
        for (std::size_t i = 0; i < n; ++i) {
            out[i].d_hat = d[i];
            out[i].grad = Vec3(g[3 * i], g[3 * i + 1], g[3 * i + 2]);
            out[i].c = c[i];
            out[i].grad_c = Vec3(gc[3 * i], gc[3 * i + 1], gc[3 * i + 2]);
            out[i].leaves = leaves[i];
            out[i].far_field = far[i];
        }
        return out;
    }
    std::vector<SmoothResult> smooth_min_dist_flat(const std::vector<Vec3>& q, const SmoothParams& p) const {
        return smooth_min_dist(q, p, true);
    }

    // Pipelined batches (sd_query_points_async): submit() enqueues the H2D,
    // the evaluation and the D2H of one batch of points and returns at once;
    // d_hat / grad (n and 3 n doubles, pinned memory for real overlap) must
    // stay alive until wait(ticket). Two batches are in flight.
    std::int64_t submit(const std::vector<Vec3>& q, const SmoothParams& p, double* d_hat, double* grad,
                        bool exact = false) const {
        sd_outputs o{d_hat, grad, nullptr, nullptr, nullptr, nullptr, nullptr};
        const sd_params sp = params(p);
        std::int64_t t = -1;
        if (sd_query_points_async(ctx_, q.data()->data(), std::int64_t(q.size()), &sp,
                                  (exact || !(p.beta > 0.0)) ? SD_EXACT : SD_BVH, &o, &t))
            fail(sd_last_error());
        return t;
    }
    void wait(std::int64_t ticket = -1) const {
        if (sd_query_wait(ctx_, ticket)) fail(sd_last_error());
    }

    // A batch of smooth_min_dist(mesh, bvh, ws, SimplexGeom g, params) over
    // query points / edges / triangles (gradient: rigid translation of g).
    std::vector<SmoothResult> smooth_min_dist(const std::vector<SimplexGeom>& g, const SmoothParams& p,
                                              bool exact = false) const {
        const std::size_t n = g.size();
        std::vector<double> corners(9 * n, 0.0), d(n), gr(3 * n), c(n), gc(3 * n);
        std::vector<std::int32_t> dims(n);
        std::vector<std::int64_t> leaves(n), far(n);
        for (std::size_t i = 0; i < n; ++i) {
            dims[i] = g[i].dim;
            for (int k = 0; k <= g[i].dim; ++k)
                for (int a = 0; a < 3; ++a) corners[9 * i + 3 * std::size_t(k) + std::size_t(a)] = g[i].c[std::size_t(k)](a);
        }
        sd_outputs o{d.data(), gr.data(), c.data(), gc.data(), leaves.data(), far.data(), nullptr};
        const sd_params sp = params(p);
        const int mode = (exact || !(p.beta > 0.0)) ? SD_EXACT : SD_BVH;
        if (n && sd_query_simplices(ctx_, corners.data(), dims.data(), std::int64_t(n), &sp, mode, &o))
            fail(sd_last_error());
        std::vector<SmoothResult> out(n);
        for (std::size_t i = 0; i < n; ++i) {
            out[i].d_hat = d[i];
            out[i].grad = Vec3(gr[3 * i], gr[3 * i + 1], gr[3 * i + 2]);
            out[i].c = c[i];
            out[i].grad_c = Vec3(gc[3 * i], gc[3 * i + 1], gc[3 * i + 2]);
            out[i].leaves = leaves[i];
            out[i].far_field = far[i];
        }
        return out;
    }

    // smooth_mesh_dist(mesh, bvh, ws, query, params) for any query mesh.
    MeshDistResult smooth_mesh_dist(const SimplexMesh& query, const SmoothParams& p) const {
        const std::size_t nq = query.simplices.size();
        std::vector<std::int32_t> sv(3 * nq);
        std::vector<std::uint8_t> kind(nq);
        for (std::size_t j = 0; j < nq; ++j) {
            for (int k = 0; k < 3; ++k) sv[3 * j + k] = query.simplices[j].v[std::size_t(k)];
            kind[j] = std::uint8_t(query.simplices[j].kind);
        }
        MeshDistResult r;
        r.vertex_grads.assign(query.vertices.size(), Vec3::Zero());
        r.per_primitive.assign(nq, 0.0);
        const sd_params sp = params(p);
        if (sd_mesh_dist(ctx_, query.vertices.data()->data(), std::int64_t(query.vertices.size()), sv.data(),
                         kind.data(), std::int64_t(nq), &sp, p.alpha_q, p.beta > 0.0 ? SD_BVH : SD_EXACT, &r.d_hat,
                         r.vertex_grads.data()->data(), r.per_primitive.data()))
            fail(sd_last_error());
        return r;
    }

    sd_ctx* handle() const { return ctx_; }

  private:
    static sd_params params(const SmoothParams& p) { return sd_params{p.alpha, p.alpha_u, p.beta, p.epsilon}; }
    sd_ctx* ctx_ = nullptr;
};

}  // namespace smoothdist::gpu
