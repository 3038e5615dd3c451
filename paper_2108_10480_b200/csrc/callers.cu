// callers.cu -- the reference's batched callers of the evaluator (SURVEY
// 8f #3), re-designed as device-resident wavefronts over the batched query
// path:
//   sd_render          <- render (render.hpp:77-134): sphere tracing of the
//                         d_hat = 0 isosurface, one wavefront iteration per
//                         marching step over the still-active rays
//   sd_grid_benchmark  <- grid_benchmark (bench.hpp:29-70): d_hat at the N^3
//                         voxel centres of [0,1]^3 as one batch
// Per ray the iteration is the reference's (step by max(d_hat, 0.1 thr),
// hit when d_hat < thr, gray shade |n . dir| from the gradient); rays are
// independent, so marching them in lockstep changes nothing but the order
// of work. Camera, ray directions and point updates are fp64 with no FMA
// contraction (this file is compiled with -fmad=false), in the reference's
// operation order; d_hat comes from the context's query path (fp32 or fp64).
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "context.h"

namespace sdgpu {

namespace {

struct Cam {
    double ox, oy, oz, fx, fy, fz, rx, ry, rz, ux, uy, uz, half_w, half_h;
};

// render.hpp:69-73 and Eigen normalized() (v / sqrt(squaredNorm))
__global__ void ray_dirs(Cam cam, int W, int H, double* dirs) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= int64_t(W) * H) return;
    const int x = int(i % W), y = int(i / W);
    const double u = (2.0 * (x + 0.5) / W - 1.0) * cam.half_w;
    const double v = (1.0 - 2.0 * (y + 0.5) / H) * cam.half_h;
    double dx = cam.fx + u * cam.rx + v * cam.ux;
    double dy = cam.fy + u * cam.ry + v * cam.uy;
    double dz = cam.fz + u * cam.rz + v * cam.uz;
    const double n = dx * dx + dy * dy + dz * dz;
    if (n > 0.0) {
        const double s = sqrt(n);
        dx = dx / s;
        dy = dy / s;
        dz = dz / s;
    }
    dirs[3 * i] = dx;
    dirs[3 * i + 1] = dy;
    dirs[3 * i + 2] = dz;
}

// query point of every active ray: origin + t dir
__global__ void ray_points(const int32_t* __restrict__ act, int n, Cam cam, const double* __restrict__ dirs,
                           const double* __restrict__ t, double* q) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t r = act[k];
    const double tr = t[r];
    q[3 * k] = cam.ox + tr * dirs[3 * r];
    q[3 * k + 1] = cam.oy + tr * dirs[3 * r + 1];
    q[3 * k + 2] = cam.oz + tr * dirs[3 * r + 2];
}

// one marching step for every active ray (render.hpp:105-121)
__global__ void ray_update(const int32_t* __restrict__ act, int n, const double* __restrict__ d_hat,
                           const double* __restrict__ grad, const int64_t* __restrict__ lv,
                           const int64_t* __restrict__ fr, const double* __restrict__ dirs, double* t, double* hit_t,
                           uint8_t* rgb, int64_t* leaves, int64_t* far, uint8_t* alive, double threshold,
                           double min_step, double t_far) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t r = act[k];
    leaves[r] += lv[k];
    far[r] += fr[k];
    const double d = d_hat[k];
    if (d < threshold) {
        hit_t[r] = t[r];
        const double gx = grad[3 * k], gy = grad[3 * k + 1], gz = grad[3 * k + 2];
        const double gn = sqrt(gx * gx + gy * gy + gz * gz);
        const double dx = dirs[3 * r], dy = dirs[3 * r + 1], dz = dirs[3 * r + 2];
        double nx, ny, nz;
        if (gn > 0.0) {
            nx = gx / gn;
            ny = gy / gn;
            nz = gz / gn;
        } else {
            nx = -dx;
            ny = -dy;
            nz = -dz;
        }
        const double shade = fabs(nx * dx + ny * dy + nz * dz);
        const uint8_t gray = uint8_t(16.5 + 239.0 * (shade < 1.0 ? shade : 1.0));
        rgb[3 * size_t(r)] = rgb[3 * size_t(r) + 1] = rgb[3 * size_t(r) + 2] = gray;
        alive[k] = 0;
        return;
    }
    const double step = isfinite(d) ? d : t_far;
    const double tn = t[r] + (step < min_step ? min_step : step);
    t[r] = tn;
    alive[k] = tn <= t_far ? 1 : 0;
}

__global__ void iota32(int32_t* a, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) a[k] = k;
}

// bench.hpp:45-50: voxel centres, x fastest
__global__ void grid_points(int n, double* q) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n3 = int64_t(n) * n * n;
    if (idx >= n3) return;
    const int i = int(idx % n), j = int((idx / n) % n), k = int(idx / (int64_t(n) * n));
    q[3 * idx] = (i + 0.5) / n;
    q[3 * idx + 1] = (j + 0.5) / n;
    q[3 * idx + 2] = (k + 0.5) / n;
}

}  // namespace

}  // namespace sdgpu

using namespace sdgpu;

namespace {

// Eigen normalized() / cross (host, fp64)
void normalize3(double v[3]) {
    const double n = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
    if (n > 0.0) {
        const double s = std::sqrt(n);
        v[0] = v[0] / s;
        v[1] = v[1] / s;
        v[2] = v[2] / s;
    }
}
void cross3(const double a[3], const double b[3], double out[3]) {
    out[0] = a[1] * b[2] - a[2] * b[1];
    out[1] = a[2] * b[0] - a[0] * b[2];
    out[2] = a[0] * b[1] - a[1] * b[0];
}

}  // namespace

namespace sdgpu {

void render_impl(Ctx& c, const sd_params& p, int mode, const sd_render_config& cfg, uint8_t* rgb_out,
                 double* hit_out, int64_t* stats, double* seconds) {
    cudaStream_t st = c.stream;
    const int W = cfg.width, H = cfg.height;
    const int64_t N = int64_t(W) * H;
    // bounding_box(mesh) over all vertices (mesh.hpp:89-93)
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t v = 0; v < c.V; ++v)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], c.xyz[3 * v + a]);
            hi[a] = std::max(hi[a], c.xyz[3 * v + a]);
        }
    const bool valid = lo[0] <= hi[0] && lo[1] <= hi[1] && lo[2] <= hi[2];
    double e[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    const double diag = valid ? std::sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]) : 0.0;
    const double threshold = cfg.threshold > 0.0 ? cfg.threshold : 1e-3 * std::max(diag, 1e-12);
    const double min_step = 0.1 * threshold;
    // make_camera (render.hpp:55-67)
    double fwd[3] = {cfg.target[0] - cfg.origin[0], cfg.target[1] - cfg.origin[1], cfg.target[2] - cfg.origin[2]};
    normalize3(fwd);
    double right[3], up[3];
    cross3(fwd, cfg.up, right);
    normalize3(right);
    cross3(right, fwd, up);
    const double half_h = std::tan(cfg.fov_deg * M_PI / 360.0);
    const double half_w = half_h * double(W) / double(H);
    Cam cam{cfg.origin[0], cfg.origin[1], cfg.origin[2], fwd[0], fwd[1], fwd[2], right[0], right[1], right[2],
            up[0], up[1], up[2], half_w, half_h};
    const double cen[3] = {0.5 * (lo[0] + hi[0]), 0.5 * (lo[1] + hi[1]), 0.5 * (lo[2] + hi[2])};
    const double oc[3] = {cen[0] - cfg.origin[0], cen[1] - cfg.origin[1], cen[2] - cfg.origin[2]};
    const double t_far = std::sqrt(oc[0] * oc[0] + oc[1] * oc[1] + oc[2] * oc[2]) + std::max(diag, 1e-12) * 1.5 +
                         threshold;

    DevBuf b_dirs, b_t, b_hit, b_rgb, b_lv, b_fr, b_act, b_act2, b_alive, b_q, b_d, b_g, b_ql, b_qf, b_n, b_tmp;
    double* dirs = static_cast<double*>(b_dirs.ensure(size_t(N) * 3 * sizeof(double)));
    double* t = static_cast<double*>(b_t.ensure(size_t(N) * sizeof(double)));
    double* hit = static_cast<double*>(b_hit.ensure(size_t(N) * sizeof(double)));
    uint8_t* rgb = static_cast<uint8_t*>(b_rgb.ensure(size_t(N) * 3));
    int64_t* lv = static_cast<int64_t*>(b_lv.ensure(size_t(N) * sizeof(int64_t)));
    int64_t* fr = static_cast<int64_t*>(b_fr.ensure(size_t(N) * sizeof(int64_t)));
    int32_t* act = static_cast<int32_t*>(b_act.ensure(size_t(N) * sizeof(int32_t)));
    int32_t* act2 = static_cast<int32_t*>(b_act2.ensure(size_t(N) * sizeof(int32_t)));
    uint8_t* alive = static_cast<uint8_t*>(b_alive.ensure(size_t(N)));
    double* q = static_cast<double*>(b_q.ensure(size_t(N) * 3 * sizeof(double)));
    FinalizeOut out;
    out.d_hat = static_cast<double*>(b_d.ensure(size_t(N) * sizeof(double)));
    out.grad = static_cast<double*>(b_g.ensure(size_t(N) * 3 * sizeof(double)));
    out.leaves = static_cast<int64_t*>(b_ql.ensure(size_t(N) * sizeof(int64_t)));
    out.far_field = static_cast<int64_t*>(b_qf.ensure(size_t(N) * sizeof(int64_t)));
    int* nsel = static_cast<int*>(b_n.ensure(sizeof(int)));

    ScopedEvent e0, e1;
    check_cuda(cudaEventRecord(e0, st), "event");
    const unsigned B = 256;
    ray_dirs<<<unsigned((N + B - 1) / B), B, 0, st>>>(cam, W, H, dirs);
    check_cuda(cudaMemsetAsync(t, 0, size_t(N) * sizeof(double), st), "memset");
    check_cuda(cudaMemsetAsync(rgb, 0, size_t(N) * 3, st), "memset");
    check_cuda(cudaMemsetAsync(lv, 0, size_t(N) * sizeof(int64_t), st), "memset");
    check_cuda(cudaMemsetAsync(fr, 0, size_t(N) * sizeof(int64_t), st), "memset");
    {
        std::vector<double> minus1(size_t(N), -1.0);
        check_cuda(cudaMemcpyAsync(hit, minus1.data(), size_t(N) * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
        check_cuda(cudaStreamSynchronize(st), "render init");
    }
    iota32<<<unsigned((N + B - 1) / B), B, 0, st>>>(act, int(N));
    int n = int(N);  // t = 0 <= t_far for every ray
    int64_t launches = 2;
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, act, alive, act2, nsel, int(N), st);
    void* tmp = b_tmp.ensure(tb);
    for (int step = 0; step < cfg.max_steps && n > 0; ++step) {
        ray_points<<<unsigned((n + B - 1) / B), B, 0, st>>>(act, n, cam, dirs, t, q);
        query_batch_f64(c, q, n, p, mode, out, st);
        launches += 1 + c.last_launches;
        ray_update<<<unsigned((n + B - 1) / B), B, 0, st>>>(act, n, out.d_hat, out.grad, out.leaves, out.far_field,
                                                             dirs, t, hit, rgb, lv, fr, alive, threshold, min_step,
                                                             t_far);
        check_cuda(cudaGetLastError(), "ray update");
        // stable compaction keeps the batch order (and so every result) deterministic
        check_cuda(cub::DeviceSelect::Flagged(tmp, tb, act, alive, act2, nsel, n, st), "compact rays");
        launches += 2;
        check_cuda(cudaMemcpyAsync(&n, nsel, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "render step");
        std::swap(act, act2);
    }
    check_cuda(cudaEventRecord(e1, st), "event");
    std::vector<int64_t> hl(static_cast<size_t>(N)), hf(static_cast<size_t>(N));
    check_cuda(cudaMemcpyAsync(rgb_out, rgb, size_t(N) * 3, cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaMemcpyAsync(hit_out, hit, size_t(N) * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaMemcpyAsync(hl.data(), lv, size_t(N) * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaMemcpyAsync(hf.data(), fr, size_t(N) * sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "render");
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "event");
    int64_t L = 0, F = 0, hits = 0;
    for (int64_t i = 0; i < N; ++i) {
        L += hl[i];
        F += hf[i];
        hits += hit_out[i] >= 0.0;
    }
    if (stats) {
        stats[0] = L;
        stats[1] = F;
        stats[2] = N;
        stats[3] = hits;
    }
    if (seconds) *seconds = ms * 1e-3;
    c.last_launches = launches;
}

void grid_impl(Ctx& c, const sd_params& p, int mode, int n, double* d_out, int64_t* leaves_out, int64_t* far_out,
               double* seconds) {
    cudaStream_t st = c.stream;
    const int64_t n3 = int64_t(n) * n * n;
    DevBuf b_q, b_d, b_l, b_f;
    double* q = static_cast<double*>(b_q.ensure(size_t(n3) * 3 * sizeof(double)));
    FinalizeOut out;
    out.d_hat = static_cast<double*>(b_d.ensure(size_t(n3) * sizeof(double)));
    if (leaves_out) out.leaves = static_cast<int64_t*>(b_l.ensure(size_t(n3) * sizeof(int64_t)));
    if (far_out) out.far_field = static_cast<int64_t*>(b_f.ensure(size_t(n3) * sizeof(int64_t)));
    ScopedEvent e0, e1;
    check_cuda(cudaEventRecord(e0, st), "event");
    grid_points<<<unsigned((n3 + 255) / 256), 256, 0, st>>>(n, q);
    query_batch_f64(c, q, n3, p, mode, out, st);
    check_cuda(cudaEventRecord(e1, st), "event");
    check_cuda(cudaMemcpyAsync(d_out, out.d_hat, size_t(n3) * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    if (leaves_out)
        check_cuda(cudaMemcpyAsync(leaves_out, out.leaves, size_t(n3) * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                   "D2H");
    if (far_out)
        check_cuda(cudaMemcpyAsync(far_out, out.far_field, size_t(n3) * sizeof(int64_t), cudaMemcpyDeviceToHost, st),
                   "D2H");
    check_cuda(cudaStreamSynchronize(st), "grid benchmark");
    float ms = 0;
    check_cuda(cudaEventElapsedTime(&ms, e0, e1), "event");
    if (seconds) *seconds = ms * 1e-3;
    c.last_launches += 2;
}

}  // namespace sdgpu
