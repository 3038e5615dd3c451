// oracle/sdoracle_callers.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference's batched CALLERS of the evaluator
// (SURVEY 8f #3): the wavefront-free per-pixel sphere tracer render()
// (render.hpp:17-134), write_ppm (:139-146), and the voxel-grid benchmark
// grid_benchmark / write_grid_csv (bench.hpp:13-88). Plain fp64,
// -ffp-contract=off, Eigen expressions restated component-wise.
#pragma once

#include <chrono>
#include <cstdio>
#include <fstream>

#include "sdoracle_simplex.hpp"

namespace sdo {

struct RenderConfig {  // render.hpp:17-25
    V3 origin{1.5, 1.5, 1.5};
    V3 target{0.5, 0.5, 0.5};
    V3 up{0, 1, 0};
    double fov_deg = 45.0;
    int width = 256, height = 256;
    double threshold = 0.0;
    int max_steps = 128;
};

struct RenderOut {  // render.hpp:27-45
    std::vector<std::uint8_t> rgb;
    std::vector<double> hit_t;
    double seconds = 0.0;
    std::int64_t leaves = 0, far_field = 0, rays = 0, hits = 0;
};

// Eigen normalized(): v / sqrt(squaredNorm()) (unchanged when zero)
inline V3 normalized_eigen(V3 v) {
    const double n = sqnorm(v);
    if (n > 0.0) {
        const double s = std::sqrt(n);
        return V3(v.x / s, v.y / s, v.z / s);
    }
    return v;
}

struct CameraFrame {  // render.hpp:50-67
    V3 origin, forward, right, up;
    double half_w, half_h;
};
inline CameraFrame make_camera(const RenderConfig& cfg) {
    CameraFrame cam;
    cam.origin = cfg.origin;
    cam.forward = normalized_eigen(cfg.target - cfg.origin);
    cam.right = normalized_eigen(cross(cam.forward, cfg.up));
    cam.up = cross(cam.right, cam.forward);
    cam.half_h = std::tan(cfg.fov_deg * M_PI / 360.0);
    cam.half_w = cam.half_h * double(cfg.width) / double(cfg.height);
    return cam;
}
inline V3 pixel_ray(const CameraFrame& cam, const RenderConfig& cfg, int x, int y) {  // :69-73
    const double u = (2.0 * (x + 0.5) / cfg.width - 1.0) * cam.half_w;
    const double v = (1.0 - 2.0 * (y + 0.5) / cfg.height) * cam.half_h;
    return normalized_eigen(cam.forward + u * cam.right + v * cam.up);
}

// render.hpp:77-134 -- per pixel: step by d_hat (at least 0.1 threshold),
// hit when d_hat < threshold, gray shade |n . dir| from the gradient.
inline RenderOut render(const Mesh& m, const Bvh& bvh, const WeightSet& ws, const Params& prm,
                        const RenderConfig& cfg, int threads) {
    RenderOut out;
    out.rgb.assign(std::size_t(cfg.width) * cfg.height * 3, 0);
    out.hit_t.assign(std::size_t(cfg.width) * cfg.height, -1.0);
    out.rays = std::int64_t(cfg.width) * cfg.height;
    const Aabb box = bounding_box(m);
    const double diag = box.diagonal();
    const double threshold = cfg.threshold > 0.0 ? cfg.threshold : 1e-3 * std::max(diag, 1e-12);
    const double min_step = 0.1 * threshold;
    const CameraFrame cam = make_camera(cfg);
    const double t_far = norm(box.center() - cfg.origin) + std::max(diag, 1e-12) * 1.5 + threshold;
    std::vector<std::int64_t> leaves(std::size_t(std::max(threads, 1)), 0), far(leaves.size(), 0),
        hits(leaves.size(), 0);
    const auto start = std::chrono::steady_clock::now();
    parallel_for(std::int64_t(cfg.height), threads, [&](std::int64_t y0, std::int64_t y1, int worker) {
        Scratch scratch;
        for (std::int64_t y = y0; y < y1; ++y) {
            for (int x = 0; x < cfg.width; ++x) {
                const V3 dir = pixel_ray(cam, cfg, x, int(y));
                double t = 0.0;
                for (int step = 0; step < cfg.max_steps && t <= t_far; ++step) {
                    const V3 q = cam.origin + t * dir;
                    const Result r = smooth_min_dist(m, bvh, ws, q, prm, scratch);
                    leaves[worker] += r.leaves;
                    far[worker] += r.far_field;
                    if (r.d_hat < threshold) {
                        out.hit_t[std::size_t(y) * cfg.width + x] = t;
                        ++hits[worker];
                        const double gn = norm(r.grad);
                        const V3 n = gn > 0.0 ? r.grad / gn : -dir;
                        const double shade = std::abs(dot(n, dir));
                        const auto gray = std::uint8_t(16.5 + 239.0 * std::min(1.0, shade));
                        std::uint8_t* px = out.rgb.data() + 3 * (std::size_t(y) * cfg.width + x);
                        px[0] = px[1] = px[2] = gray;
                        break;
                    }
                    t += std::max(std::isfinite(r.d_hat) ? r.d_hat : t_far, min_step);
                }
            }
        }
    });
    out.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    for (std::size_t i = 0; i < leaves.size(); ++i) {
        out.leaves += leaves[i];
        out.far_field += far[i];
        out.hits += hits[i];
    }
    return out;
}

// render.hpp:139-146 -- P6, rows top to bottom
inline void write_ppm(const std::vector<std::uint8_t>& rgb, int w, int h, const std::string& path) {
    std::ofstream out(path, std::ios::binary);
    if (!out) fail("cannot open " + path + " for writing");
    // the header of render.hpp:142 ("P6\n" << w << " " << h << "\n255\n"),
    // formatted with snprintf (stream integer formatting is unreliable when
    // this library is loaded into the Python test process)
    char head[64];
    const int len = std::snprintf(head, sizeof head, "P6\n%d %d\n255\n", w, h);
    out.write(head, len);
    out.write(reinterpret_cast<const char*>(rgb.data()), std::streamsize(rgb.size()));
    if (!out) fail("write failed: " + path);
}

// bench.hpp:29-70 -- d_hat at the N^3 voxel centres of [0,1]^3, x fastest
struct GridOut {
    std::vector<double> d_hat;
    std::vector<std::int64_t> leaves, far_field;
};
inline GridOut grid_benchmark(const Mesh& m, const Bvh& bvh, const WeightSet& ws, const Params& prm, int n,
                              int threads) {
    GridOut out;
    const std::size_t n3 = std::size_t(n) * n * n;
    out.d_hat.assign(n3, 0.0);
    out.leaves.assign(n3, 0);
    out.far_field.assign(n3, 0);
    parallel_for(std::int64_t(n), threads, [&](std::int64_t k0, std::int64_t k1, int) {
        Scratch s;
        for (std::int64_t k = k0; k < k1; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    const V3 q((i + 0.5) / n, (j + 0.5) / n, (k + 0.5) / n);
                    const Result r = smooth_min_dist(m, bvh, ws, q, prm, s);
                    const std::size_t idx = std::size_t(i) + n * (std::size_t(j) + n * k);
                    out.d_hat[idx] = r.d_hat;
                    out.leaves[idx] = r.leaves;
                    out.far_field[idx] = r.far_field;
                }
    });
    return out;
}

// bench.hpp:75-88 -- "%zu,%.17g,%lld,%lld,%.6g"
inline void write_grid_csv(const GridOut& r, int n, const std::vector<double>& slab_seconds,
                           const std::string& path) {
    std::ofstream out(path);
    if (!out) fail("cannot open " + path + " for writing");
    out << "voxel_index,d_hat,leaves_visited,far_field,slab_time_s\n";
    char buf[160];
    for (std::size_t idx = 0; idx < r.d_hat.size(); ++idx) {
        const int k = int(idx / (std::size_t(n) * n));
        std::snprintf(buf, sizeof buf, "%zu,%.17g,%lld,%lld,%.6g\n", idx, r.d_hat[idx],
                      static_cast<long long>(r.leaves[idx]), static_cast<long long>(r.far_field[idx]),
                      slab_seconds[std::size_t(k)]);
        out << buf;
    }
    if (!out) fail("write failed: " + path);
}

}  // namespace sdo
