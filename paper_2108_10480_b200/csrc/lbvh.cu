// lbvh.cu -- K2: GPU-built linear BVH (Karras 2012 radix tree over
// 63-bit Morton codes of primitive bbox centres), refitted bottom-up in
// fp64 and emitted directly in the reference tree layout (bvh.hpp:14-32:
// pre-order ids, root 0, left child = parent + 1, one primitive per leaf,
// count = n_B, diameter = box diagonal) so the CPU evaluator can run on the
// very same tree. Replaces build_bvh (bvh.hpp:34-91) as the builder; the
// median-split tree it produces remains available as SD_BVH_MEDIAN.
//
// Stages (all on the device, CUB for the sort):
//   1 leaf boxes + Morton keys   (fp64 min/max of the corners, exact)
//   2 radix sort (key, primitive)
//   3 hierarchy: each internal node finds its range and split by binary
//     search on common-prefix length (ties broken by sorted index)
//   4 refit: bottom-up with per-node arrival counters, union boxes, counts
//   5 pre-order numbering: pre(left) = pre(p) + 1, pre(right) = pre(p) +
//     2 count(left); computed top-down level by level from the root
//   6 scatter into sd_bvh_node records
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "context.h"

namespace sdgpu {

namespace {

__device__ __forceinline__ uint64_t spread21(uint64_t v) {
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

struct Box {
    double lo[3], hi[3];
};

__global__ void leaf_boxes(const double* __restrict__ xyz, const int32_t* __restrict__ sv,
                           const uint8_t* __restrict__ kind, int64_t n, double3 slo, double3 sinv, Box* boxes,
                           uint64_t* keys, int32_t* ids) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Box b;
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = INFINITY;
        b.hi[a] = -INFINITY;
    }
    for (int k = 0; k <= kind[i]; ++k) {
        const int64_t v = sv[3 * i + k];
        for (int a = 0; a < 3; ++a) {
            b.lo[a] = fmin(b.lo[a], xyz[3 * v + a]);
            b.hi[a] = fmax(b.hi[a], xyz[3 * v + a]);
        }
    }
    boxes[i] = b;
    const double cs[3] = {slo.x, slo.y, slo.z}, ci[3] = {sinv.x, sinv.y, sinv.z};
    uint64_t key = 0;
    for (int a = 0; a < 3; ++a) {
        const double c = 0.5 * (b.lo[a] + b.hi[a]);  // bbox centre, as bvh.hpp:45
        const double f = fmin(fmax((c - cs[a]) * ci[a], 0.0), 2097151.0);
        key |= spread21(uint64_t(f)) << (2 - a);
    }
    keys[i] = key;
    ids[i] = int32_t(i);
}

// common prefix length of sorted keys i, j (index tie-break); -1 outside
__device__ __forceinline__ int delta(const uint64_t* k, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    const uint64_t a = k[i], b = k[j];
    if (a != b) return __clzll(a ^ b);
    return 64 + __clzll(uint64_t(i) ^ uint64_t(j));
}

// internal nodes 0..n-2, leaves encoded as n - 1 + sorted index
__global__ void hierarchy(const uint64_t* __restrict__ k, int64_t n, int32_t* left, int32_t* right,
                          int32_t* parent) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = delta(k, n, i, i + 1) - delta(k, n, i, i - 1) >= 0 ? 1 : -1;
    const int dmin = delta(k, n, i, i - d);
    int64_t lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    const int64_t j = i + l * d;
    const int dnode = delta(k, n, i, j);
    int64_t s = 0;
    for (int64_t div = 2;; div *= 2) {
        const int64_t t = (l + div - 1) / div;
        if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
        if (t <= 1) break;
    }
    const int64_t g = i + s * d + min(d, 0);
    const int64_t lo = min(i, j), hi = max(i, j);
    const int32_t lc = int32_t(lo == g ? (n - 1) + g : g);
    const int32_t rc = int32_t(hi == g + 1 ? (n - 1) + g + 1 : g + 1);
    left[i] = lc;
    right[i] = rc;
    parent[lc] = int32_t(i);
    parent[rc] = int32_t(i);
}

__device__ __forceinline__ double diag_rn(const Box& b) {
    if (!(b.lo[0] <= b.hi[0] && b.lo[1] <= b.hi[1] && b.lo[2] <= b.hi[2])) return 0.0;
    const double dx = __dsub_rn(b.hi[0], b.lo[0]), dy = __dsub_rn(b.hi[1], b.lo[1]),
                 dz = __dsub_rn(b.hi[2], b.lo[2]);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

// node arrays are indexed [0, n-1) internal, [n-1, 2n-1) leaves
__global__ void refit(int64_t n, const int32_t* __restrict__ ids, const Box* __restrict__ pbox,
                      const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                      const int32_t* __restrict__ parent, Box* nbox, int32_t* count, int32_t* arrive) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t leaf = (n - 1) + i;
    nbox[leaf] = pbox[ids[i]];
    count[leaf] = 1;
    int32_t node = n > 1 ? parent[leaf] : -1;
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&arrive[node], 1) == 0) return;  // first arrival: sibling not done
        __threadfence();
        // L2 reads (__ldcg): the sibling's box was written by another SM
        const double* a = reinterpret_cast<const double*>(nbox + left[node]);
        const double* b = reinterpret_cast<const double*>(nbox + right[node]);
        Box u;
        for (int ax = 0; ax < 3; ++ax) {
            u.lo[ax] = fmin(__ldcg(a + ax), __ldcg(b + ax));
            u.hi[ax] = fmax(__ldcg(a + 3 + ax), __ldcg(b + 3 + ax));
        }
        nbox[node] = u;
        count[node] = __ldcg(count + left[node]) + __ldcg(count + right[node]);
        node = node == 0 ? -1 : parent[node];
    }
}

// top-down pre-order numbering, one tree level per launch (frontier lists)
__global__ void preorder_level(const int32_t* __restrict__ front, int32_t nf, const int32_t* __restrict__ left,
                               const int32_t* __restrict__ right, const int32_t* __restrict__ count, int64_t n,
                               int32_t* pre, int32_t* next, int32_t* nnext) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nf) return;
    const int32_t node = front[i];
    if (node >= n - 1) return;  // leaf
    const int32_t l = left[node], r = right[node];
    pre[l] = pre[node] + 1;
    pre[r] = pre[node] + 2 * count[l];
    const int32_t slot = atomicAdd(nnext, 2);
    next[slot] = l;
    next[slot + 1] = r;
}

__global__ void emit(int64_t n, const int32_t* __restrict__ ids, const Box* __restrict__ nbox,
                     const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                     const int32_t* __restrict__ count, const int32_t* __restrict__ pre, sd_bvh_node* out) {
    const int64_t node = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (node >= 2 * n - 1) return;
    sd_bvh_node r;
    const Box b = nbox[node];
    for (int a = 0; a < 3; ++a) {
        r.lo[a] = b.lo[a];
        r.hi[a] = b.hi[a];
    }
    r.count = count[node];
    r.diameter = diag_rn(b);
    if (node >= n - 1) {
        r.left = r.right = -1;
        r.primitive = ids[node - (n - 1)];
    } else {
        r.left = pre[left[node]];
        r.right = pre[right[node]];
        r.primitive = -1;
    }
    out[pre[node]] = r;
}

}  // namespace

void tree_build_lbvh(Ctx& c) {
    const int64_t n = c.N;
    c.tree.clear();
    c.dtree_ready = false;
    c.sx_tree_ready = c.sx_prim_ready = false;
    if (n == 0) return;
    cudaStream_t st = c.stream;
    // scene box of the primitive corners (host: O(V), exact)
    double slo[3] = {INFINITY, INFINITY, INFINITY}, shi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k <= c.kind[i]; ++k)
            for (int a = 0; a < 3; ++a) {
                const double x = c.xyz[3 * size_t(c.sv[3 * i + k]) + a];
                slo[a] = std::min(slo[a], x);
                shi[a] = std::max(shi[a], x);
            }
    auto inv = [](double l, double h) { return h > l ? 2097152.0 / (h - l) : 0.0; };
    const double3 dlo = make_double3(slo[0], slo[1], slo[2]);
    const double3 dinv = make_double3(inv(slo[0], shi[0]), inv(slo[1], shi[1]), inv(slo[2], shi[2]));

    DevBuf xyz, sv, kind, boxes, keys, ids, nbox, lr, parent, count, arrive, pre, front, out, tmp;
    double* d_xyz = static_cast<double*>(xyz.ensure(c.xyz.size() * sizeof(double)));
    int32_t* d_sv = static_cast<int32_t*>(sv.ensure(c.sv.size() * sizeof(int32_t)));
    uint8_t* d_kind = static_cast<uint8_t*>(kind.ensure(c.kind.size()));
    check_cuda(cudaMemcpyAsync(d_xyz, c.xyz.data(), c.xyz.size() * sizeof(double), cudaMemcpyHostToDevice, st), "lbvh upload");
    check_cuda(cudaMemcpyAsync(d_sv, c.sv.data(), c.sv.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st), "lbvh upload");
    check_cuda(cudaMemcpyAsync(d_kind, c.kind.data(), c.kind.size(), cudaMemcpyHostToDevice, st), "lbvh upload");

    Box* d_pbox = static_cast<Box*>(boxes.ensure(size_t(n) * sizeof(Box)));
    uint64_t* d_keys = static_cast<uint64_t*>(keys.ensure(size_t(n) * 2 * sizeof(uint64_t)));
    int32_t* d_ids = static_cast<int32_t*>(ids.ensure(size_t(n) * 2 * sizeof(int32_t)));
    const unsigned B = 256;
    leaf_boxes<<<unsigned((n + B - 1) / B), B, 0, st>>>(d_xyz, d_sv, d_kind, n, dlo, dinv, d_pbox, d_keys, d_ids);
    check_cuda(cudaGetLastError(), "lbvh leaf boxes");

    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, d_keys, d_keys + n, d_ids, d_ids + n, int(n), 0, 63, st);
    void* d_tmp = tmp.ensure(tb);
    check_cuda(cub::DeviceRadixSort::SortPairs(d_tmp, tb, d_keys, d_keys + n, d_ids, d_ids + n, int(n), 0, 63, st),
               "lbvh sort");
    const uint64_t* skeys = d_keys + n;
    const int32_t* sids = d_ids + n;

    const int64_t nn = 2 * n - 1;
    int32_t* d_lr = static_cast<int32_t*>(lr.ensure(size_t(std::max<int64_t>(1, n - 1)) * 2 * sizeof(int32_t)));
    int32_t* d_left = d_lr;
    int32_t* d_right = d_lr + std::max<int64_t>(1, n - 1);
    int32_t* d_parent = static_cast<int32_t*>(parent.ensure(size_t(nn) * sizeof(int32_t)));
    Box* d_nbox = static_cast<Box*>(nbox.ensure(size_t(nn) * sizeof(Box)));
    int32_t* d_count = static_cast<int32_t*>(count.ensure(size_t(nn) * sizeof(int32_t)));
    int32_t* d_arrive = static_cast<int32_t*>(arrive.ensure(size_t(nn) * sizeof(int32_t)));
    check_cuda(cudaMemsetAsync(d_arrive, 0, size_t(nn) * sizeof(int32_t), st), "memset");
    if (n > 1) {
        hierarchy<<<unsigned((n - 1 + B - 1) / B), B, 0, st>>>(skeys, n, d_left, d_right, d_parent);
        check_cuda(cudaGetLastError(), "lbvh hierarchy");
    }
    refit<<<unsigned((n + B - 1) / B), B, 0, st>>>(n, sids, d_pbox, d_left, d_right, d_parent, d_nbox, d_count,
                                                    d_arrive);
    check_cuda(cudaGetLastError(), "lbvh refit");

    // pre-order numbering: frontier sweep from the root (node 0, or the
    // single leaf when n == 1)
    int32_t* d_pre = static_cast<int32_t*>(pre.ensure(size_t(nn) * sizeof(int32_t)));
    int32_t* d_front = static_cast<int32_t*>(front.ensure(size_t(nn + 1) * 2 * sizeof(int32_t) + 16));
    int32_t* fa = d_front;
    int32_t* fb = d_front + nn + 1;
    int32_t* d_cnt = fb + nn + 1;
    const int32_t root = 0;  // internal node 0, or the only leaf (index n - 1 = 0) when n == 1
    const int32_t zero = 0;
    check_cuda(cudaMemcpyAsync(d_pre + root, &zero, sizeof(int32_t), cudaMemcpyHostToDevice, st), "pre root");
    check_cuda(cudaMemcpyAsync(fa, &root, sizeof(int32_t), cudaMemcpyHostToDevice, st), "front root");
    int32_t nf = 1;
    int depth = 0;
    while (nf > 0 && n > 1) {
        check_cuda(cudaMemsetAsync(d_cnt, 0, sizeof(int32_t), st), "memset");
        preorder_level<<<unsigned((nf + B - 1) / B), B, 0, st>>>(fa, nf, d_left, d_right, d_count, n, d_pre, fb,
                                                                 d_cnt);
        check_cuda(cudaGetLastError(), "lbvh preorder");
        check_cuda(cudaMemcpyAsync(&nf, d_cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "frontier size");
        check_cuda(cudaStreamSynchronize(st), "lbvh preorder");
        std::swap(fa, fb);
        if (nf > 0) ++depth;
    }
    sd_bvh_node* d_out = static_cast<sd_bvh_node*>(out.ensure(size_t(nn) * sizeof(sd_bvh_node)));
    emit<<<unsigned((nn + B - 1) / B), B, 0, st>>>(n, sids, d_nbox, d_left, d_right, d_count, d_pre, d_out);
    check_cuda(cudaGetLastError(), "lbvh emit");
    c.tree.resize(size_t(nn));
    c.tree_trusted = true;
    check_cuda(cudaMemcpyAsync(c.tree.data(), d_out, size_t(nn) * sizeof(sd_bvh_node), cudaMemcpyDeviceToHost, st),
               "lbvh download");
    check_cuda(cudaStreamSynchronize(st), "lbvh build");
}

}  // namespace sdgpu
