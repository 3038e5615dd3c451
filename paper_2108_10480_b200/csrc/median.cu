// median.cu -- the reference's median-split tree (build_bvh, bvh.hpp:34-91)
// built on the device, level by level, bit-identical to the host restatement
// (SD_BVH_MEDIAN):
//   leaf box = corner bbox, centroid = bbox centre (bvh.hpp:40-46)
//   per node: union box of its primitives' boxes, split axis = longest
//   extent (ties -> x, then y), left = the first n/2 primitives in
//   (centroid[axis], index) order (nth_element's unique partition sets),
//   pre-order ids: left = id + 1, right = id + 2 (n/2)
// Every level works on all nodes at once: a segmented reduction gives the
// node boxes, two stable segmented sorts (by index, then by the centroid
// coordinate on the node's axis) order each node's primitives, and each node
// splits its sorted segment in the middle. Node records are emitted in the
// reference layout as they are decided.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "context.h"

namespace sdgpu {

namespace {

struct MBox {
    double lo[3], hi[3];
};

struct BoxUnion {
    __device__ __forceinline__ MBox operator()(const MBox& a, const MBox& b) const {
        MBox r;
        for (int k = 0; k < 3; ++k) {
            r.lo[k] = fmin(a.lo[k], b.lo[k]);
            r.hi[k] = fmax(a.hi[k], b.hi[k]);
        }
        return r;
    }
};

struct BoxOf {
    const MBox* pbox;
    const int32_t* order;
    __device__ __forceinline__ MBox operator()(int64_t k) const { return pbox[order[k]]; }
};

struct Seg {
    int32_t begin, end, id, pad;
};
struct BeginOf {
    const int32_t* p;
    __host__ __device__ int operator()(int s) const { return p[4 * s]; }
};
struct EndOf {
    const int32_t* p;
    __host__ __device__ int operator()(int s) const { return p[4 * s + 1]; }
};

__global__ void prim_boxes(const double* __restrict__ xyz, const int32_t* __restrict__ sv,
                           const uint8_t* __restrict__ kind, int64_t n, MBox* boxes, double* ce, int32_t* order) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    MBox b;
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
    for (int a = 0; a < 3; ++a) ce[3 * i + a] = __dmul_rn(0.5, __dadd_rn(b.lo[a], b.hi[a]));
    order[i] = int32_t(i);
}

__device__ __forceinline__ double diag_rn(const MBox& b) {
    if (!(b.lo[0] <= b.hi[0] && b.lo[1] <= b.hi[1] && b.lo[2] <= b.hi[2])) return 0.0;
    const double dx = __dsub_rn(b.hi[0], b.lo[0]), dy = __dsub_rn(b.hi[1], b.lo[1]),
                 dz = __dsub_rn(b.hi[2], b.lo[2]);
    return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
}

__device__ __forceinline__ void put_node(sd_bvh_node* out, int32_t id, const MBox& b, int32_t left, int32_t right,
                                         int32_t prim, int32_t count) {
    sd_bvh_node r;
    for (int a = 0; a < 3; ++a) {
        r.lo[a] = b.lo[a];
        r.hi[a] = b.hi[a];
    }
    r.left = left;
    r.right = right;
    r.primitive = prim;
    r.count = count;
    r.diameter = diag_rn(b);
    out[id] = r;
}

// internal node records, split axes
__global__ void split_nodes(const Seg* __restrict__ segs, int S, const MBox* __restrict__ sbox, int8_t* axis,
                            sd_bvh_node* out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const Seg g = segs[s];
    const MBox b = sbox[s];
    int ax = 0;  // longest extent, ties -> x, then y (bvh.hpp:66-69)
    if (__dsub_rn(b.hi[1], b.lo[1]) > __dsub_rn(b.hi[0], b.lo[0])) ax = 1;
    if (__dsub_rn(b.hi[2], b.lo[2]) > __dsub_rn(b.hi[ax], b.lo[ax])) ax = 2;
    axis[s] = int8_t(ax);
    const int32_t n = g.end - g.begin, half = n / 2;
    put_node(out, g.id, b, g.id + 1, g.id + 2 * half, -1, n);
}

// centroid coordinate on the node's axis, for every element of an active
// segment (segments sorted by begin; elements outside keep a dummy key)
__global__ void axis_keys(const int32_t* __restrict__ order, int64_t n, const Seg* __restrict__ segs, int S,
                          const int8_t* __restrict__ axis, const double* __restrict__ ce, double* key) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    int lo = 0, hi = S;  // first segment with begin > k
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (segs[mid].begin <= k) lo = mid + 1;
        else hi = mid;
    }
    const int s = lo - 1;
    // + 0.0 folds -0.0 into +0.0: the radix order of the keys is then the
    // comparator's (equal coordinates tie on the index, pass 1)
    key[k] = (s >= 0 && k < segs[s].end) ? __dadd_rn(ce[3 * int64_t(order[k]) + axis[s]], 0.0) : 0.0;
}

// children: leaves are emitted, larger children go to the next level
__global__ void children(const Seg* __restrict__ segs, int S, const int32_t* __restrict__ order,
                         const MBox* __restrict__ pbox, sd_bvh_node* out, Seg* next, uint8_t* flag) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    const Seg g = segs[s];
    const int32_t half = (g.end - g.begin) / 2, mid = g.begin + half;
    const Seg c[2] = {{g.begin, mid, g.id + 1, 0}, {mid, g.end, g.id + 2 * half, 0}};
    for (int k = 0; k < 2; ++k) {
        next[2 * s + k] = c[k];
        const bool leaf = c[k].end - c[k].begin == 1;
        flag[2 * s + k] = leaf ? 0 : 1;
        if (leaf) {
            const int32_t p = order[c[k].begin];
            put_node(out, c[k].id, pbox[p], -1, -1, p, 1);
        }
    }
}

}  // namespace

void tree_build_median_gpu(Ctx& c) {
    const int64_t n = c.N;
    c.tree.clear();
    c.dtree_ready = false;
    c.sx_tree_ready = c.sx_prim_ready = false;
    if (n == 0) return;
    if (n >= (int64_t(1) << 30)) throw std::runtime_error("too many primitives for the median build");
    cudaStream_t st = c.stream;
    const unsigned B = 256;
    DevBuf b_xyz, b_sv, b_kind, b_pbox, b_ce, b_ord, b_ord2, b_key, b_key2, b_segs, b_next, b_flag, b_sbox, b_axis,
        b_out, b_tmp, b_ns;
    double* xyz = static_cast<double*>(b_xyz.ensure(c.xyz.size() * sizeof(double)));
    int32_t* sv = static_cast<int32_t*>(b_sv.ensure(c.sv.size() * sizeof(int32_t)));
    uint8_t* kind = static_cast<uint8_t*>(b_kind.ensure(c.kind.size()));
    check_cuda(cudaMemcpyAsync(xyz, c.xyz.data(), c.xyz.size() * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemcpyAsync(sv, c.sv.data(), c.sv.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
    check_cuda(cudaMemcpyAsync(kind, c.kind.data(), c.kind.size(), cudaMemcpyHostToDevice, st), "H2D");
    MBox* pbox = static_cast<MBox*>(b_pbox.ensure(size_t(n) * sizeof(MBox)));
    double* ce = static_cast<double*>(b_ce.ensure(size_t(n) * 3 * sizeof(double)));
    int32_t* order = static_cast<int32_t*>(b_ord.ensure(size_t(n) * sizeof(int32_t)));
    int32_t* order2 = static_cast<int32_t*>(b_ord2.ensure(size_t(n) * sizeof(int32_t)));
    double* key = static_cast<double*>(b_key.ensure(size_t(n) * sizeof(double)));
    double* key2 = static_cast<double*>(b_key2.ensure(size_t(n) * sizeof(double)));
    sd_bvh_node* out = static_cast<sd_bvh_node*>(b_out.ensure(size_t(2 * n - 1) * sizeof(sd_bvh_node)));
    prim_boxes<<<unsigned((n + B - 1) / B), B, 0, st>>>(xyz, sv, kind, n, pbox, ce, order);
    check_cuda(cudaGetLastError(), "median prim boxes");

    Seg* segs = static_cast<Seg*>(b_segs.ensure(size_t(std::max<int64_t>(n, 2)) * sizeof(Seg)));
    Seg* next = static_cast<Seg*>(b_next.ensure(size_t(std::max<int64_t>(n, 2)) * sizeof(Seg)));
    uint8_t* flag = static_cast<uint8_t*>(b_flag.ensure(size_t(std::max<int64_t>(n, 2))));
    MBox* sbox = static_cast<MBox*>(b_sbox.ensure(size_t(std::max<int64_t>(n / 2, 1)) * sizeof(MBox)));
    int8_t* axis = static_cast<int8_t*>(b_axis.ensure(size_t(std::max<int64_t>(n / 2, 1))));
    int* nsel = static_cast<int*>(b_ns.ensure(sizeof(int)));
    if (n == 1) {  // a single leaf root
        MBox b;
        check_cuda(cudaMemcpyAsync(&b, pbox, sizeof(MBox), cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "median");
        sd_bvh_node r;
        for (int a = 0; a < 3; ++a) {
            r.lo[a] = b.lo[a];
            r.hi[a] = b.hi[a];
        }
        r.left = r.right = -1;
        r.primitive = 0;
        r.count = 1;
        const double dx = b.hi[0] - b.lo[0], dy = b.hi[1] - b.lo[1], dz = b.hi[2] - b.lo[2];
        r.diameter = (b.lo[0] <= b.hi[0] && b.lo[1] <= b.hi[1] && b.lo[2] <= b.hi[2])
                         ? std::sqrt(dx * dx + dy * dy + dz * dz)
                         : 0.0;
        c.tree.assign(1, r);
        return;
    }
    const Seg root{0, int32_t(n), 0, 0};
    check_cuda(cudaMemcpyAsync(segs, &root, sizeof(Seg), cudaMemcpyHostToDevice, st), "H2D");
    int S = 1;
    while (S > 0) {
        // node boxes: union of the primitive boxes of each segment
        const int32_t* seg_i32 = reinterpret_cast<const int32_t*>(segs);
        cub::CountingInputIterator<int64_t> cnt(0);
        cub::TransformInputIterator<MBox, BoxOf, cub::CountingInputIterator<int64_t>> boxes_in(cnt, BoxOf{pbox, order});
        MBox empty;
        for (int a = 0; a < 3; ++a) {
            empty.lo[a] = INFINITY;
            empty.hi[a] = -INFINITY;
        }
        // begin / end offsets with stride 4 (Seg layout)
        cub::CountingInputIterator<int> sidx(0);
        cub::TransformInputIterator<int, BeginOf, cub::CountingInputIterator<int>> bo(sidx, BeginOf{seg_i32});
        cub::TransformInputIterator<int, EndOf, cub::CountingInputIterator<int>> eo(sidx, EndOf{seg_i32});
        size_t tb = 0;
        cub::DeviceSegmentedReduce::Reduce(nullptr, tb, boxes_in, sbox, S, bo, eo, BoxUnion{}, empty, st);
        check_cuda(cub::DeviceSegmentedReduce::Reduce(b_tmp.ensure(tb), tb, boxes_in, sbox, S, bo, eo, BoxUnion{}, empty,
                                                      st),
                   "median node boxes");
        split_nodes<<<unsigned((S + B - 1) / B), B, 0, st>>>(segs, S, sbox, axis, out);
        check_cuda(cudaGetLastError(), "median split");
        // pass 1: primitives of each segment by index (stable sort of the ids)
        check_cuda(cudaMemcpyAsync(order2, order, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st), "copy");
        tb = 0;
        cub::DeviceSegmentedSort::StableSortKeys(nullptr, tb, order, order2, int(n), S, bo, eo, st);
        check_cuda(cub::DeviceSegmentedSort::StableSortKeys(b_tmp.ensure(tb), tb, order, order2, int(n), S, bo, eo, st),
                   "median sort ids");
        // pass 2: stable by the centroid coordinate on the node's axis
        axis_keys<<<unsigned((n + B - 1) / B), B, 0, st>>>(order2, n, segs, S, axis, ce, key);
        check_cuda(cudaGetLastError(), "median keys");
        check_cuda(cudaMemcpyAsync(order, order2, size_t(n) * sizeof(int32_t), cudaMemcpyDeviceToDevice, st), "copy");
        tb = 0;
        cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, key, key2, order2, order, int(n), S, bo, eo, st);
        check_cuda(cub::DeviceSegmentedSort::StableSortPairs(b_tmp.ensure(tb), tb, key, key2, order2, order, int(n), S,
                                                              bo, eo, st),
                   "median sort centroids");
        // split in the middle; leaves out, the rest to the next level
        children<<<unsigned((S + B - 1) / B), B, 0, st>>>(segs, S, order, pbox, out, next, flag);
        check_cuda(cudaGetLastError(), "median children");
        tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, next, flag, segs, nsel, 2 * S, st);
        check_cuda(cub::DeviceSelect::Flagged(b_tmp.ensure(tb), tb, next, flag, segs, nsel, 2 * S, st),
                   "median next level");
        check_cuda(cudaMemcpyAsync(&S, nsel, sizeof(int), cudaMemcpyDeviceToHost, st), "D2H");
        check_cuda(cudaStreamSynchronize(st), "median level");
    }
    c.tree.resize(size_t(2 * n - 1));
    check_cuda(cudaMemcpyAsync(c.tree.data(), out, size_t(2 * n - 1) * sizeof(sd_bvh_node), cudaMemcpyDeviceToHost, st),
               "D2H tree");
    check_cuda(cudaStreamSynchronize(st), "median build");
}

}  // namespace sdgpu
