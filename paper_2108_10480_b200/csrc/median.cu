// median.cu -- the reference's median-split tree (build_bvh, bvh.hpp:34-91)
// built on the device, level by level, bit-identical to the host restatement
// (SD_BVH_MEDIAN):
//   leaf box = corner bbox, centroid = bbox centre (bvh.hpp:40-46)
//   per node: union box of its primitives' boxes, split axis = longest
//   extent (ties -> x, then y), left = the first n/2 primitives in
//   (centroid[axis], index) order (nth_element's unique partition sets),
//   pre-order ids: left = id + 1, right = id + 2 (n/2)
// Every level works on all nodes at once, with device-wide primitives whose
// parallelism does not depend on the segment sizes (the top levels have one
// huge segment): a reduce-by-key over the positions gives the node boxes, and
// ONE radix sort of 2 ceil(log2 n)-bit keys (segment start, rank of the
// primitive on the node's axis) orders every node's primitives, where the
// per-axis ranks -- positions in (centroid coordinate, index) order -- are
// computed once up front. Each node splits its sorted segment in the middle. Node
// records are emitted in the reference layout as they are decided.
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

// segment of position k: the first segment with begin > k, minus one
__device__ __forceinline__ int seg_of(const Seg* __restrict__ segs, int S, int64_t k) {
    int lo = 0, hi = S;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (segs[mid].begin <= k) lo = mid + 1;
        else hi = mid;
    }
    const int s = lo - 1;
    return (s >= 0 && k < segs[s].end) ? s : -1;
}

// reduce-by-key keys: the segment of an active position, a value >= S that
// differs from both neighbours' for a finished one (its own run)
__global__ void seg_keys(int64_t n, const Seg* __restrict__ segs, int S, int32_t* key) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = seg_of(segs, S, k);
    key[k] = s >= 0 ? s : int32_t(S + k);
}

__global__ void scatter_boxes(const int32_t* __restrict__ ukey, const MBox* __restrict__ agg,
                              const int* __restrict__ nruns, int S, MBox* sbox) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= *nruns) return;
    const int32_t s = ukey[r];
    if (s < S) sbox[s] = agg[r];
}

// sort keys of a level: (segment start << rb) | rank on the segment's axis
// for an active position, (k << rb) for a finished one (it stays in place);
// rb = ceil(log2 n) bits hold any position or rank
__global__ void sort_keys(const int32_t* __restrict__ order, int64_t n, const Seg* __restrict__ segs, int S,
                          const int8_t* __restrict__ axis, const int32_t* __restrict__ rank, int rb, uint64_t* key) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int s = seg_of(segs, S, k);
    key[k] = s >= 0 ? (uint64_t(segs[s].begin) << rb) | uint64_t(rank[int64_t(axis[s]) * n + order[k]])
                    : uint64_t(k) << rb;
}

// order-preserving bits of a centroid coordinate (+ 0.0 folds -0.0 into
// +0.0: equal coordinates then tie on the index, as in the comparator)
__global__ void coord_keys(const double* __restrict__ ce, int64_t n, int a, uint64_t* key, int32_t* ids) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double x = __dadd_rn(ce[3 * i + a], 0.0);
    const uint64_t b = uint64_t(__double_as_longlong(x));
    key[i] = (b >> 63) ? ~b : (b | (uint64_t(1) << 63));
    ids[i] = int32_t(i);
}

__global__ void scatter_rank(const int32_t* __restrict__ sorted_ids, int64_t n, int32_t* rank) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j < n) rank[sorted_ids[j]] = int32_t(j);
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
        b_out, b_tmp, b_ns, b_rank, b_skey, b_ukey, b_agg, b_nruns;
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
    uint64_t* key = static_cast<uint64_t*>(b_key.ensure(size_t(n) * sizeof(uint64_t)));
    uint64_t* key2 = static_cast<uint64_t*>(b_key2.ensure(size_t(n) * sizeof(uint64_t)));
    int32_t* rank = static_cast<int32_t*>(b_rank.ensure(size_t(3 * n) * sizeof(int32_t)));
    int32_t* skey = static_cast<int32_t*>(b_skey.ensure(size_t(n) * sizeof(int32_t)));
    int32_t* ukey = static_cast<int32_t*>(b_ukey.ensure(size_t(n) * sizeof(int32_t)));
    MBox* agg = static_cast<MBox*>(b_agg.ensure(size_t(n) * sizeof(MBox)));
    int* nruns = static_cast<int*>(b_nruns.ensure(sizeof(int)));
    sd_bvh_node* out = static_cast<sd_bvh_node*>(b_out.ensure(size_t(2 * n - 1) * sizeof(sd_bvh_node)));
    prim_boxes<<<unsigned((n + B - 1) / B), B, 0, st>>>(xyz, sv, kind, n, pbox, ce, order);
    check_cuda(cudaGetLastError(), "median prim boxes");
    const unsigned G = unsigned((n + B - 1) / B);
    // per-axis ranks: positions in (centroid coordinate, index) order (the
    // radix sort is stable and its input is in index order)
    for (int a = 0; a < 3; ++a) {
        coord_keys<<<G, B, 0, st>>>(ce, n, a, key, order2);
        check_cuda(cudaGetLastError(), "median coord keys");
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, order2, skey, int(n), 0, 64, st);
        check_cuda(cub::DeviceRadixSort::SortPairs(b_tmp.ensure(tb), tb, key, key2, order2, skey, int(n), 0, 64, st),
                   "median axis ranks");
        scatter_rank<<<G, B, 0, st>>>(skey, n, rank + size_t(a) * n);
        check_cuda(cudaGetLastError(), "median ranks");
    }
    int rb = 1;  // ceil(log2 n): bits of a position or a rank
    while ((int64_t(1) << rb) < n) ++rb;
    const int key_bits = 2 * rb;

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
        c.tree_trusted = true;
        return;
    }
    const Seg root{0, int32_t(n), 0, 0};
    check_cuda(cudaMemcpyAsync(segs, &root, sizeof(Seg), cudaMemcpyHostToDevice, st), "H2D");
    int S = 1;
    while (S > 0) {
        // node boxes: union of the primitive boxes of each segment
        // (reduce-by-key over the positions; finished positions are own runs)
        cub::CountingInputIterator<int64_t> cnt(0);
        cub::TransformInputIterator<MBox, BoxOf, cub::CountingInputIterator<int64_t>> boxes_in(cnt, BoxOf{pbox, order});
        seg_keys<<<G, B, 0, st>>>(n, segs, S, skey);
        check_cuda(cudaGetLastError(), "median segment keys");
        size_t tb = 0;
        cub::DeviceReduce::ReduceByKey(nullptr, tb, skey, ukey, boxes_in, agg, nruns, BoxUnion{}, n, st);
        check_cuda(cub::DeviceReduce::ReduceByKey(b_tmp.ensure(tb), tb, skey, ukey, boxes_in, agg, nruns, BoxUnion{}, n,
                                                  st),
                   "median node boxes");
        scatter_boxes<<<G, B, 0, st>>>(ukey, agg, nruns, S, sbox);
        check_cuda(cudaGetLastError(), "median node boxes scatter");
        split_nodes<<<unsigned((S + B - 1) / B), B, 0, st>>>(segs, S, sbox, axis, out);
        check_cuda(cudaGetLastError(), "median split");
        // every segment's primitives in (centroid[axis], index) order, in place
        sort_keys<<<G, B, 0, st>>>(order, n, segs, S, axis, rank, rb, key);
        check_cuda(cudaGetLastError(), "median sort keys");
        tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, order, order2, int(n), 0, key_bits, st);
        check_cuda(cub::DeviceRadixSort::SortPairs(b_tmp.ensure(tb), tb, key, key2, order, order2, int(n), 0, key_bits,
                                                   st),
                   "median sort");
        std::swap(order, order2);
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
    c.tree_trusted = true;
    check_cuda(cudaMemcpyAsync(c.tree.data(), out, size_t(2 * n - 1) * sizeof(sd_bvh_node), cudaMemcpyDeviceToHost, st),
               "D2H tree");
    check_cuda(cudaStreamSynchronize(st), "median build");
}

}  // namespace sdgpu
