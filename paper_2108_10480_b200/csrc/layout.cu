// layout.cu -- the traversal layout of a tree (DeviceTree, context.h) built
// on the device from the reference node array (bvh.hpp:14-32): per node the
// T box rounded outward, the link (right child, or -(leaf slot + 1)), n_B,
// log2 n_B and the fp64 diameter; per internal node the child-pair record;
// per leaf slot (leaves in pre-order) the primitive record and its meta.
// Replaces a single-threaded host pass that took ~2 s at 5.2M triangles.
// The primitive records are the host build_record's (api.cu) bit for bit:
// the same fp64 operations, each rounded separately (no contraction).
#include <cub/cub.cuh>

#include "context.h"
#include "traverse.cuh"

namespace sdgpu {

namespace {

struct R3 {
    double x, y, z;
};
__device__ __forceinline__ R3 ld3(const double* xyz, int32_t i) {
    return R3{xyz[3 * int64_t(i)], xyz[3 * int64_t(i) + 1], xyz[3 * int64_t(i) + 2]};
}
__device__ __forceinline__ R3 sub(R3 a, R3 b) { return R3{__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z)}; }
__device__ __forceinline__ double dot(R3 a, R3 b) {
    return __dadd_rn(__dadd_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dmul_rn(a.z, b.z));
}
__device__ __forceinline__ R3 cross(R3 a, R3 b) {
    return R3{__dsub_rn(__dmul_rn(a.y, b.z), __dmul_rn(a.z, b.y)), __dsub_rn(__dmul_rn(a.z, b.x), __dmul_rn(a.x, b.z)),
              __dsub_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ R3 scale(R3 a, double s) { return R3{__dmul_rn(a.x, s), __dmul_rn(a.y, s), __dmul_rn(a.z, s)}; }
__device__ __forceinline__ double rcp(double x) { return __ddiv_rn(1.0, x); }

template <class T>
__device__ __forceinline__ T to(double x) {
    if constexpr (sizeof(T) == 4) return __double2float_rn(x);
    else return x;
}

// device twin of build_record (api.cu): rec_size(kind) values, rest zero
template <class T>
__device__ void record_dev(const double* __restrict__ xyz, const int32_t* __restrict__ sv, int k, int64_t p,
                           T* out) {
    for (int i = 0; i < kRecTri; ++i) out[i] = T(0);
    const int32_t* s = sv + 3 * p;
    const R3 a = ld3(xyz, s[0]);
    out[0] = to<T>(a.x);
    out[1] = to<T>(a.y);
    out[2] = to<T>(a.z);
    if (k == SD_EDGE) {
        const R3 e = sub(ld3(xyz, s[1]), a);
        const double e2 = dot(e, e);
        const double inv = e2 > 0 ? rcp(e2) : 0.0;  // exact.hpp:71
        out[3] = to<T>(e.x);
        out[4] = to<T>(e.y);
        out[5] = to<T>(e.z);
        out[6] = to<T>(inv);
        out[7] = to<T>(__dmul_rn(e.x, inv));
        out[8] = to<T>(__dmul_rn(e.y, inv));
        out[9] = to<T>(__dmul_rn(e.z, inv));
    } else if (k == SD_TRIANGLE) {
        const R3 b = ld3(xyz, s[1]), c = ld3(xyz, s[2]);
        const R3 ab = sub(b, a), ac = sub(c, a), bc = sub(c, b);
        const double A = dot(ab, ab), B = dot(ab, ac), C = dot(ac, ac), BC = dot(bc, bc);
        const double det = __dsub_rn(__dmul_rn(A, C), __dmul_rn(B, B));
        out[3] = to<T>(ab.x);
        out[4] = to<T>(ab.y);
        out[5] = to<T>(ab.z);
        out[6] = to<T>(ac.x);
        out[7] = to<T>(ac.y);
        out[8] = to<T>(ac.z);
        out[9] = to<T>(A);
        out[10] = to<T>(B);
        out[11] = to<T>(C);
        out[12] = to<T>(rcp(A));
        out[13] = to<T>(rcp(C));
        out[14] = to<T>(rcp(BC));
        out[15] = to<T>(rcp(det));
        const R3 n = cross(ab, ac);
        const double nn = dot(n, n);
        const double inv = nn > 0 ? rcp(nn) : 0.0;
        const R3 g1 = scale(cross(n, sub(a, c)), inv), g2 = scale(cross(n, ab), inv);
        out[16] = to<T>(g1.x);
        out[17] = to<T>(g1.y);
        out[18] = to<T>(g1.z);
        out[19] = to<T>(g2.x);
        out[20] = to<T>(g2.y);
        out[21] = to<T>(g2.z);
    }
}

__global__ void leaf_flags(const sd_bvh_node* __restrict__ nodes, int64_t n, int32_t* flag) {
    const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id < n) flag[id] = nodes[id].left < 0 ? 1 : 0;
}

// err bit 0: an internal node whose left child is not id + 1
template <class T>
__global__ void node_records(const sd_bvh_node* __restrict__ nodes, int64_t n, const int32_t* __restrict__ slot,
                             const double* __restrict__ xyz, const int32_t* __restrict__ sv,
                             const uint8_t* __restrict__ kind, const int32_t* __restrict__ poly_index,
                             NodeT<T>* box, int32_t* count, T* lgc, double* d64, T* leafrec, int32_t* leafmeta,
                             int* inexact, int* err) {
    const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const sd_bvh_node nd = nodes[id];
    NodeT<T> b;
    bool exact = true;
    for (int a = 0; a < 3; ++a) {
        // outward rounding keeps the T box a superset (exact when the
        // geometry was quantized to float, as SD_FP32 does)
        T l = to<T>(nd.lo[a]), h = to<T>(nd.hi[a]);
        if (double(l) > nd.lo[a]) l = sizeof(T) == 4 ? T(nextafterf(float(l), -INFINITY)) : T(nextafter(double(l), -INFINITY));
        if (double(h) < nd.hi[a]) h = sizeof(T) == 4 ? T(nextafterf(float(h), INFINITY)) : T(nextafter(double(h), INFINITY));
        exact = exact && double(l) == nd.lo[a] && double(h) == nd.hi[a];
        b.v[a] = l;
        b.v[4 + a] = h;
    }
    b.v[3] = to<T>(nd.diameter);
    int32_t link;
    if (nd.left < 0) {
        const int32_t s = slot[id];
        link = -(s + 1);
        const int32_t p = nd.primitive;
        const int k = kind[p];
        T rec[kRecTri];
        record_dev<T>(xyz, sv, k, p, rec);
        for (int i = 0; i < kRecTri; ++i) leafrec[int64_t(s) * kRecTri + i] = rec[i];
        const int poly = k == SD_POINT ? -1 : poly_index[p];
        leafmeta[s] = k | ((poly + 1) << 2);
    } else {
        if (nd.left != id + 1) atomicOr(err, 1);
        link = nd.right;
    }
    T lv = T(0);
    memcpy(&b.v[7], &link, sizeof(int32_t));
    if (sizeof(T) == 8) memcpy(reinterpret_cast<char*>(&b.v[7]) + 4, &lv, 4);
    box[id] = b;
    count[id] = nd.count;
    lgc[id] = to<T>(log2(double(nd.count)));
    d64[id] = nd.diameter;
    if (!exact) atomicOr(inexact, 1);
}

template <class T>
__global__ void pair_records(const sd_bvh_node* __restrict__ nodes, int64_t n, const NodeT<T>* __restrict__ box,
                             const T* __restrict__ lgc, PairT<T>* pairs) {
    const int64_t id = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (id >= n) return;
    const sd_bvh_node& nd = nodes[id];
    PairT<T> pr;
    if (nd.left >= 0) {
        pr.set(box[id + 1], box[nd.right]);
        pr.lgc[0] = lgc[id + 1];
        pr.lgc[1] = lgc[nd.right];
    } else {
        for (int i = 0; i < 16; ++i) pr.w[i] = T(0);
        pr.lgc[0] = pr.lgc[1] = T(0);
    }
    pr.lgc[2] = pr.lgc[3] = T(0);
    pairs[id] = pr;
}

}  // namespace

template <class T>
void upload_tree_device(Ctx& c, DeviceTree& t, int depth) {
    const int64_t n = int64_t(c.tree.size());
    const int64_t N = c.N;
    cudaStream_t st = c.stream;
    const unsigned B = 256, G = unsigned((n + B - 1) / B);
    DevBuf b_nodes, b_xyz, b_sv, b_kind, b_poly, b_flag, b_slot, b_tmp, b_err;
    auto h2d = [&](DevBuf& buf, const void* src, size_t bytes) {
        void* d = buf.ensure(bytes);
        if (bytes) check_cuda(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, st), "upload tree");
        return d;
    };
    auto* nodes = static_cast<sd_bvh_node*>(h2d(b_nodes, c.tree.data(), size_t(n) * sizeof(sd_bvh_node)));
    auto* xyz = static_cast<double*>(h2d(b_xyz, c.xyz.data(), c.xyz.size() * sizeof(double)));
    auto* sv = static_cast<int32_t*>(h2d(b_sv, c.sv.data(), c.sv.size() * sizeof(int32_t)));
    auto* kind = static_cast<uint8_t*>(h2d(b_kind, c.kind.data(), c.kind.size()));
    std::vector<int32_t> poly(c.poly_index);
    if (poly.size() != size_t(N)) poly.assign(size_t(N), -1);
    auto* pidx = static_cast<int32_t*>(h2d(b_poly, poly.data(), poly.size() * sizeof(int32_t)));
    // leaf slots: leaves numbered in pre-order
    int32_t* flag = static_cast<int32_t*>(b_flag.ensure(size_t(n) * sizeof(int32_t)));
    int32_t* slot = static_cast<int32_t*>(b_slot.ensure(size_t(n) * sizeof(int32_t)));
    leaf_flags<<<G, B, 0, st>>>(nodes, n, flag);
    check_cuda(cudaGetLastError(), "tree leaf flags");
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, slot, n, st);
    check_cuda(cub::DeviceScan::ExclusiveSum(b_tmp.ensure(tb), tb, flag, slot, n, st), "tree leaf slots");
    auto* box = static_cast<NodeT<T>*>(t.box.ensure(size_t(n) * sizeof(NodeT<T>)));
    auto* cnt = static_cast<int32_t*>(t.count.ensure(size_t(n) * sizeof(int32_t)));
    auto* lgc = static_cast<T*>(t.lgcount.ensure(size_t(n) * sizeof(T)));
    auto* d64 = static_cast<double*>(t.diam64.ensure(size_t(n) * sizeof(double)));
    auto* leafrec = static_cast<T*>(t.leafrec.ensure(size_t(N) * kRecTri * sizeof(T)));
    auto* leafmeta = static_cast<int32_t*>(t.leafmeta.ensure(size_t(N) * sizeof(int32_t)));
    int* flags = static_cast<int*>(b_err.ensure(2 * sizeof(int)));
    check_cuda(cudaMemsetAsync(flags, 0, 2 * sizeof(int), st), "memset");
    node_records<T><<<G, B, 0, st>>>(nodes, n, slot, xyz, sv, kind, pidx, box, cnt, lgc, d64, leafrec, leafmeta,
                                     flags, flags + 1);
    check_cuda(cudaGetLastError(), "tree node records");
    auto* pairs = static_cast<PairT<T>*>(t.pairs.ensure(size_t(n) * sizeof(PairT<T>)));
    pair_records<T><<<G, B, 0, st>>>(nodes, n, box, lgc, pairs);
    check_cuda(cudaGetLastError(), "tree pair records");
    int hf[2] = {0, 0};
    check_cuda(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, st), "D2H");
    check_cuda(cudaStreamSynchronize(st), "tree layout");
    if (hf[1]) throw std::runtime_error("tree: left child must follow its parent");
    t.nodes = n;
    t.split_k = -1;
    t.leaves = N;
    t.depth = depth;
    t.exact_boxes = hf[0] == 0;
}
template void upload_tree_device<float>(Ctx&, DeviceTree&, int);
template void upload_tree_device<double>(Ctx&, DeviceTree&, int);

}  // namespace sdgpu
