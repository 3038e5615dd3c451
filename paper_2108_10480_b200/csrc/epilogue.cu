// epilogue.cu -- K4: de-shift the per-query partial state into the
// reference's unshifted fp64 domain and finalise exactly as
// detail::result_from_accum does (smooth.hpp:147-159):
//   c = sum_k s_k 2^{m_k},  grad_c = sum_k g_k 2^{m_k}
//   c <= 0  ->  d_hat = +inf, grad = 0
//   else        d_hat = -log(c) / alpha, grad = grad_c / (c + epsilon)
// The -708 underflow mask of smooth.hpp:85-88 was applied per term in the
// producing kernels, so the fp64 sums here have the reference semantics.
#include "exact.h"

#include <algorithm>
#include <cmath>

#include <cub/cub.cuh>

namespace sdgpu {

__device__ __forceinline__ void finalize_write(double M, double s, double gx, double gy, double gz, int64_t i,
                                               double alpha, double eps, int64_t const_leaves,
                                               const int64_t* __restrict__ leaves_in, const int64_t* __restrict__ far_in,
                                               const uint64_t* __restrict__ hash_in, const int64_t* __restrict__ perm,
                                               const FinalizeOut& o) {
    double c, cx, cy, cz;
    if (M < -1000.0 && M > -INFINITY) {
        // The anchor can sit below fp64's exponent range while the sum does
        // not: the first tile with a nonzero sum anchors the totals at its
        // shift (a far tile just inside the -708 mask: ~ -1021 - 96), and
        // nearer tiles within 2^512 of it add to s without re-anchoring, so
        // s 2^M is representable (2^-760, say) although 2^M alone is 0.
        // Scale in two steps.
        const double h = exp2(0.5 * M), h2 = exp2(M - 0.5 * M);
        c = (s * h) * h2;
        cx = (gx * h) * h2, cy = (gy * h) * h2, cz = (gz * h) * h2;
    } else {
        const double scale = M > -INFINITY ? exp2(M) : 0.0;
        c = s * scale;
        cx = gx * scale, cy = gy * scale, cz = gz * scale;
    }
    const int64_t j = perm ? perm[i] : i;  // tree path: undo the query sort
    if (o.nan_keys) {
        if (o.nan_keys[i] == 0xffffffffu) c = cx = cy = cz = NAN;
    } else if (o.qf || o.qd) {
        const double x = o.qf ? double(o.qf[3 * j]) : o.qd[3 * j];
        const double y = o.qf ? double(o.qf[3 * j + 1]) : o.qd[3 * j + 1];
        const double z = o.qf ? double(o.qf[3 * j + 2]) : o.qd[3 * j + 2];
        if (isnan(x) || isnan(y) || isnan(z)) c = cx = cy = cz = NAN;
    }
    if (o.peers) {  // fused exchange: NVLink stores into the owner's buffer
        const int64_t ow = j / o.peer_qown, k = j - ow * o.peer_qown;
        double* dst = o.peers[ow] + size_t(o.peer_rank) * 4 * o.peer_qown + k;
        dst[0] = c;
        dst[o.peer_qown] = cx;
        dst[2 * o.peer_qown] = cy;
        dst[3 * o.peer_qown] = cz;
        if (o.leaves) o.leaves[j] = leaves_in ? leaves_in[i] : const_leaves;
        if (o.far_field) o.far_field[j] = far_in ? far_in[i] : 0;
        if (o.hash) o.hash[j] = hash_in ? hash_in[i] : 0;
        return;
    }
    double d = INFINITY, ax = 0, ay = 0, az = 0;
    if (!(c <= 0.0)) {  // c > 0, or NaN (propagates like the reference's -log(NaN))
        d = -log(c) / alpha;
        const double den = c + eps;
        ax = cx / den;
        ay = cy / den;
        az = cz / den;
    }
    if (o.aos) {  // one full sector; split_aos writes d_hat / grad
        double4* dst = reinterpret_cast<double4*>(o.aos) + j;
        *dst = make_double4(d, ax, ay, az);
    } else {
        o.d_hat[j] = d;
    }
    if (o.grad && !o.aos) {
        o.grad[3 * j] = ax;
        o.grad[3 * j + 1] = ay;
        o.grad[3 * j + 2] = az;
    }
    if (o.c) o.c[j] = c;
    if (o.grad_c) {
        o.grad_c[3 * j] = cx;
        o.grad_c[3 * j + 1] = cy;
        o.grad_c[3 * j + 2] = cz;
    }
    if (o.leaves) o.leaves[j] = leaves_in ? leaves_in[i] : const_leaves;
    if (o.far_field) o.far_field[j] = far_in ? far_in[i] : 0;
    if (o.hash) o.hash[j] = hash_in ? hash_in[i] : 0;
}

__global__ void finalize_kernel(const double* __restrict__ part, int splits, int64_t Q, double alpha, double eps,
                                int64_t const_leaves, const int64_t* __restrict__ leaves_in,
                                const int64_t* __restrict__ far_in, const uint64_t* __restrict__ hash_in,
                                const int64_t* __restrict__ perm, FinalizeOut o) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i = o.pk_world > 1 ? shard_packet(t >> 5, o.pk_world, o.pk_rank, o.pk_chunk) * 32 + (t & 31) : t;
    if (i >= Q) return;
    double M = -INFINITY;
    for (int k = 0; k < splits; ++k) M = fmax(M, double(part[size_t(k) * 5 * Q + i]));
    double s = 0, gx = 0, gy = 0, gz = 0;
    for (int k = 0; k < splits && M > -INFINITY; ++k) {
        const double* p = part + size_t(k) * 5 * Q;
        const double f = exp2(double(p[i]) - M);
        s = fma(double(p[Q + i]), f, s);
        gx = fma(double(p[2 * Q + i]), f, gx);
        gy = fma(double(p[3 * Q + i]), f, gy);
        gz = fma(double(p[4 * Q + i]), f, gz);
    }
    finalize_write(M, s, gx, gy, gz, i, alpha, eps, const_leaves, leaves_in, far_in, hash_in, perm, o);
}

// Many splits (the few-query split traversal): one warp per query, lanes
// over the splits, shuffle merge.
__global__ void finalize_warp_kernel(const double* __restrict__ part, int splits, int64_t Q, double alpha, double eps,
                                     int64_t const_leaves, const int64_t* __restrict__ leaves_in,
                                     const int64_t* __restrict__ far_in, const uint64_t* __restrict__ hash_in,
                                     const int64_t* __restrict__ perm, FinalizeOut o) {
    const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= Q) return;
    double M = -INFINITY;
    for (int k = lane; k < splits; k += 32) M = fmax(M, part[size_t(k) * 5 * Q + i]);
    for (int off = 16; off; off >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, off));
    double s = 0, gx = 0, gy = 0, gz = 0;
    if (M > -INFINITY) {
        for (int k = lane; k < splits; k += 32) {
            const double* p = part + size_t(k) * 5 * Q;
            const double f = exp2(p[i] - M);
            s = fma(p[Q + i], f, s);
            gx = fma(p[2 * Q + i], f, gx);
            gy = fma(p[3 * Q + i], f, gy);
            gz = fma(p[4 * Q + i], f, gz);
        }
        for (int off = 16; off; off >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, off);
            gx += __shfl_xor_sync(0xffffffffu, gx, off);
            gy += __shfl_xor_sync(0xffffffffu, gy, off);
            gz += __shfl_xor_sync(0xffffffffu, gz, off);
        }
    }
    if (lane == 0) finalize_write(M, s, gx, gy, gz, i, alpha, eps, const_leaves, leaves_in, far_in, hash_in, perm, o);
}

// (d_hat, grad) of the queries in original order from the AoS scratch
__global__ void split_aos(const double4* __restrict__ aos, int64_t Q, double* __restrict__ d_hat,
                          double* __restrict__ grad) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= Q) return;
    const double4 v = aos[j];
    d_hat[j] = v.x;
    grad[3 * j] = v.y;
    grad[3 * j + 1] = v.z;
    grad[3 * j + 2] = v.w;
}

cudaError_t launch_finalize(const double* part, int splits, int64_t Q, double alpha, double epsilon,
                            int64_t const_leaves, const int64_t* leaves_in, const int64_t* far_in,
                            const uint64_t* hash_in, const int64_t* perm, const FinalizeOut& out, cudaStream_t st) {
    if (Q <= 0) return cudaSuccess;
    if (out.aos && (!out.grad || out.peers || out.pk_world > 1)) {  // the AoS route only for whole batches
        FinalizeOut o = out;
        o.aos = nullptr;
        return launch_finalize(part, splits, Q, alpha, epsilon, const_leaves, leaves_in, far_in, hash_in, perm, o, st);
    }
    const int threads = 256;
    if (splits >= 32) {
        finalize_warp_kernel<<<unsigned((Q * 32 + threads - 1) / threads), threads, 0, st>>>(
            part, splits, Q, alpha, epsilon, const_leaves, leaves_in, far_in, hash_in, perm, out);
    } else {
        int64_t n = Q;  // positions covered
        if (out.pk_world > 1) {
            n = shard_count((Q + 31) / 32, out.pk_world, out.pk_rank, out.pk_chunk) * 32;
            if (n == 0) return cudaSuccess;
        }
        const unsigned blocks = unsigned((n + threads - 1) / threads);
        finalize_kernel<<<blocks, threads, 0, st>>>(part, splits, Q, alpha, epsilon, const_leaves, leaves_in, far_in,
                                                       hash_in, perm, out);
    }
    if (out.aos) {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        split_aos<<<unsigned((Q + threads - 1) / threads), threads, 0, st>>>(reinterpret_cast<const double4*>(out.aos),
                                                                             Q, out.d_hat, out.grad);
    }
    return cudaGetLastError();
}
__global__ void finalize_sums_kernel(const double* __restrict__ c, const double* __restrict__ gc, int64_t Q,
                                     double alpha, double eps, double* d_hat, double* grad) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    const double ci = c[i];
    double d = INFINITY, ax = 0, ay = 0, az = 0;
    if (ci > 0.0) {
        d = -log(ci) / alpha;
        const double den = ci + eps;
        ax = gc[3 * i] / den;
        ay = gc[3 * i + 1] / den;
        az = gc[3 * i + 2] / den;
    }
    d_hat[i] = d;
    if (grad) {
        grad[3 * i] = ax;
        grad[3 * i + 1] = ay;
        grad[3 * i + 2] = az;
    }
}

cudaError_t launch_finalize_sums(const double* c, const double* grad_c, int64_t Q, double alpha, double epsilon,
                                 double* d_hat, double* grad, cudaStream_t st) {
    if (Q <= 0) return cudaSuccess;
    const unsigned blocks = unsigned((Q + 255) / 256);
    finalize_sums_kernel<<<blocks, 256, 0, st>>>(c, grad_c, Q, alpha, epsilon, d_hat, grad);
    return cudaGetLastError();
}

__global__ void empty_kernel(int64_t Q, FinalizeOut o) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    if (o.peers) {  // an empty shard contributes zero partials
        const int64_t ow = i / o.peer_qown, k = i - ow * o.peer_qown;
        double* dst = o.peers[ow] + size_t(o.peer_rank) * 4 * o.peer_qown + k;
        dst[0] = dst[o.peer_qown] = dst[2 * o.peer_qown] = dst[3 * o.peer_qown] = 0.0;
        if (o.leaves) o.leaves[i] = 0;
        if (o.far_field) o.far_field[i] = 0;
        return;
    }
    o.d_hat[i] = INFINITY;
    if (o.grad) o.grad[3 * i] = o.grad[3 * i + 1] = o.grad[3 * i + 2] = 0.0;
    if (o.c) o.c[i] = 0.0;
    if (o.grad_c) o.grad_c[3 * i] = o.grad_c[3 * i + 1] = o.grad_c[3 * i + 2] = 0.0;
    if (o.leaves) o.leaves[i] = 0;
    if (o.far_field) o.far_field[i] = 0;
    if (o.hash) o.hash[i] = 0;
}

cudaError_t launch_empty_result(int64_t Q, const FinalizeOut& out, cudaStream_t st) {
    if (Q <= 0) return cudaSuccess;
    empty_kernel<<<unsigned((Q + 255) / 256), 256, 0, st>>>(Q, out);
    return cudaGetLastError();
}

// --------------------------------- primitive-sharded exchange
// Instead of an all-reduce of the per-query partial sums, rank r stores its
// unshifted partials (c, grad_c) of query i straight into the symmetric
// buffer of the query's owner o = i / qown (NVLink stores through the
// peer pointer table; layout [world][4][qown] SoA), and each owner then sums
// the world contributions of its queries in rank order and finalises them
// (result_from_accum, smooth.hpp:147-159): a reduce-scatter done by the
// producing ranks' own stores, half the traffic of an all-reduce.
// sd_query_points_scatter fuses the stores into K4 (finalize_write above:
// FinalizeOut::peers), so the partials never round-trip through local
// memory; this standalone kernel serves partials computed elsewhere.
__global__ void scatter_partials_kernel(const double* __restrict__ c, const double* __restrict__ gc, int64_t Q,
                                        double* const* __restrict__ peers, int rank, int64_t qown) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    const int64_t o = i / qown, j = i - o * qown;
    double* dst = peers[o] + size_t(rank) * 4 * qown + j;
    dst[0] = c[i];
    dst[qown] = gc[3 * i];
    dst[2 * qown] = gc[3 * i + 1];
    dst[3 * qown] = gc[3 * i + 2];
}

__global__ void reduce_owned_kernel(const double* __restrict__ sbuf, int64_t qown, int64_t n, int world, double alpha,
                                    double eps, double* d_hat, double* grad) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double c = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
    for (int r = 0; r < world; ++r) {
        const double* p = sbuf + size_t(r) * 4 * qown + j;
        c += p[0];
        gx += p[qown];
        gy += p[2 * qown];
        gz += p[3 * qown];
    }
    double d = INFINITY, ax = 0, ay = 0, az = 0;
    if (c > 0.0) {
        d = -log(c) / alpha;
        const double den = c + eps;
        ax = gx / den;
        ay = gy / den;
        az = gz / den;
    }
    d_hat[j] = d;
    if (grad) {
        grad[3 * j] = ax;
        grad[3 * j + 1] = ay;
        grad[3 * j + 2] = az;
    }
}

cudaError_t launch_scatter_partials(const double* c, const double* grad_c, int64_t Q, double* const* peers, int rank,
                                    int64_t qown, cudaStream_t st) {
    if (Q <= 0) return cudaSuccess;
    scatter_partials_kernel<<<unsigned((Q + 255) / 256), 256, 0, st>>>(c, grad_c, Q, peers, rank, qown);
    return cudaGetLastError();
}

cudaError_t launch_reduce_owned(const double* sbuf, int64_t qown, int64_t n, int world, double alpha, double epsilon,
                                double* d_hat, double* grad, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    reduce_owned_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(sbuf, qown, n, world, alpha, epsilon, d_hat, grad);
    return cudaGetLastError();
}

// ------------------------------------------ mesh-to-mesh outer LogSumExp
// smooth.hpp:237-254: mass_j = exp(-alpha_q d_j); denom = sum_j mass_j;
// vertex gradient = sum over the simplices at the vertex of mass_j / n_j
// times the inner gradient, divided by denom + epsilon; denom <= 0 ->
// d_hat = +inf and zero gradients. Point simplices: n_j = 1.
__global__ void mass_kernel(const double* __restrict__ d, int64_t n, double alpha_q, double* mass) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) mass[j] = exp(-alpha_q * d[j]);
}
// vidx: vertex of each point simplex (stride 1; NULL = identity), or the
// corners of each simplex (stride 3, -1 past the last corner): the mass is
// split evenly over the corners (smooth.hpp:243-245).
__global__ void scatter_kernel(const double* __restrict__ mass, const double* __restrict__ grad, int64_t n,
                               const int32_t* __restrict__ vidx, int stride, double* vg) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n) return;
    if (stride == 1) {
        const int64_t v = vidx ? vidx[j] : j;
        const double m = mass[j];
        atomicAdd(vg + 3 * v, m * grad[3 * j]);
        atomicAdd(vg + 3 * v + 1, m * grad[3 * j + 1]);
        atomicAdd(vg + 3 * v + 2, m * grad[3 * j + 2]);
        return;
    }
    const int32_t* s = vidx + size_t(stride) * j;
    const int nv = 1 + (s[1] >= 0) + (s[1] >= 0 && s[2] >= 0);
    const double split = mass[j] / nv;
    for (int k = 0; k < nv; ++k) {
        const int64_t v = s[k];
        atomicAdd(vg + 3 * v, split * grad[3 * j]);
        atomicAdd(vg + 3 * v + 1, split * grad[3 * j + 1]);
        atomicAdd(vg + 3 * v + 2, split * grad[3 * j + 2]);
    }
}
__global__ void mesh_finish_kernel(double* vg, int64_t nv, const double* __restrict__ denom, double alpha_q, double eps,
                                   double* d_out) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const double den = denom[0];
    if (k == 0) d_out[0] = den > 0.0 ? -log(den) / alpha_q : INFINITY;
    if (k >= nv) return;
    const double f = den > 0.0 ? 1.0 / (den + eps) : 0.0;
    vg[3 * k] = den > 0.0 ? vg[3 * k] / (den + eps) : 0.0;
    vg[3 * k + 1] = den > 0.0 ? vg[3 * k + 1] / (den + eps) : 0.0;
    vg[3 * k + 2] = den > 0.0 ? vg[3 * k + 2] / (den + eps) : 0.0;
    (void)f;
}

cudaError_t launch_mesh_reduce(const double* d, const double* grad, int64_t n, const int32_t* vidx, int stride,
                               int64_t nv, double alpha_q, double eps, double* work, size_t work_bytes, double* vg,
                               double* d_out, int64_t& launches, cudaStream_t st) {
    // work: [mass n][denom 1][cub temp]
    double* mass = work;
    double* denom = work + n;
    void* tmp = work + n + 2;
    size_t tb = work_bytes > (size_t(n) + 2) * sizeof(double) ? work_bytes - (size_t(n) + 2) * sizeof(double) : 0;
    const unsigned B = 256;
    cudaError_t e = cudaMemsetAsync(vg, 0, size_t(nv) * 3 * sizeof(double), st);
    if (e != cudaSuccess) return e;
    if (n > 0) {
        mass_kernel<<<unsigned((n + B - 1) / B), B, 0, st>>>(d, n, alpha_q, mass);
        size_t need = 0;
        cub::DeviceReduce::Sum(nullptr, need, mass, denom, int(n), st);
        if (need > tb) return cudaErrorMemoryAllocation;
        e = cub::DeviceReduce::Sum(tmp, tb, mass, denom, int(n), st);
        if (e != cudaSuccess) return e;
        scatter_kernel<<<unsigned((n + B - 1) / B), B, 0, st>>>(mass, grad, n, vidx, stride, vg);
        launches += 4;
    } else {
        e = cudaMemsetAsync(denom, 0, sizeof(double), st);
        if (e != cudaSuccess) return e;
    }
    mesh_finish_kernel<<<unsigned((std::max<int64_t>(nv, 1) + B - 1) / B), B, 0, st>>>(vg, nv, denom, alpha_q, eps,
                                                                                        d_out);
    ++launches;
    return cudaGetLastError();
}

size_t mesh_reduce_work_bytes(int64_t n) {
    size_t need = 0;
    cub::DeviceReduce::Sum(nullptr, need, static_cast<double*>(nullptr), static_cast<double*>(nullptr),
                           int(std::max<int64_t>(n, 1)));
    return (size_t(n) + 2) * sizeof(double) + need + 256;
}

}  // namespace sdgpu
