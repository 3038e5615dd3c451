// bvh.cu -- Barnes-Hut tree path: tree construction (reference median
// split on the host; the GPU LBVH lives in lbvh.cu), upload into the
// traversal layout, query Morton sort, and K3, the stack traversal that
// replaces collect_contributions (smooth.hpp:101-131) for a query batch.
//
// Decision semantics (checked invariant): at every popped node, leaves
// included, when beta > 0: admissible iff d_B > 0 and diameter < beta d_B
// (bvh.hpp:185-187) with d_B the point-box distance (bvh.hpp:105-111).
// The fp32 path decides in fp32 when |diameter - beta d_B| is clearly
// outside a 1e-5 relative band and otherwise re-decides in fp64 with the
// reference's operation order (no FMA contraction), which is bit-identical
// to the oracle compiled with -ffp-contract=off. The fp64 path always
// decides that way.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdlib>
#include <numeric>
#include <string>

#include <cub/cub.cuh>

#include "pair2.cuh"
#include "traverse.cuh"

namespace sdgpu {

// ------------------------------------------------------------ host tree
// Restates build_bvh (bvh.hpp:34-91): leaf box = corner bbox, centroid =
// bbox centre, split axis = longest extent (ties -> x, then y), median by
// (centroid[axis], index); one primitive per leaf; pre-order ids.
static void median_build_host(const Ctx& c, std::vector<sd_bvh_node>& out) {
    const int64_t n = c.N;
    out.clear();
    if (n == 0) return;
    std::vector<double> lo(3 * n), hi(3 * n), ce(3 * n);
    for (int64_t i = 0; i < n; ++i) {
        for (int a = 0; a < 3; ++a) {
            lo[3 * i + a] = INFINITY;
            hi[3 * i + a] = -INFINITY;
        }
        for (int k = 0; k <= c.kind[i]; ++k) {
            const int32_t v = c.sv[3 * i + k];
            for (int a = 0; a < 3; ++a) {
                lo[3 * i + a] = std::min(lo[3 * i + a], c.xyz[3 * size_t(v) + a]);
                hi[3 * i + a] = std::max(hi[3 * i + a], c.xyz[3 * size_t(v) + a]);
            }
        }
        for (int a = 0; a < 3; ++a) ce[3 * i + a] = 0.5 * (lo[3 * i + a] + hi[3 * i + a]);
    }
    std::vector<int32_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    out.resize(size_t(2 * n - 1));
    auto diag = [](const double* l, const double* h) {
        if (!(l[0] <= h[0] && l[1] <= h[1] && l[2] <= h[2])) return 0.0;
        const double dx = h[0] - l[0], dy = h[1] - l[1], dz = h[2] - l[2];
        return std::sqrt(dx * dx + dy * dy + dz * dz);
    };
    int32_t next = 0;
    // explicit-stack version of the reference recursion (same id order)
    struct Job {
        int64_t first, last;
        int32_t id;
        int stage;
    };
    std::vector<Job> stack;
    stack.push_back({0, n, next++, 0});
    while (!stack.empty()) {
        Job& j = stack.back();
        sd_bvh_node& node = out[j.id];
        if (j.last - j.first == 1) {
            const int32_t p = order[j.first];
            node.left = node.right = -1;
            node.primitive = p;
            node.count = 1;
            for (int a = 0; a < 3; ++a) {
                node.lo[a] = lo[3 * p + a];
                node.hi[a] = hi[3 * p + a];
            }
            node.diameter = diag(node.lo, node.hi);
            stack.pop_back();
            continue;
        }
        const int64_t mid = j.first + (j.last - j.first) / 2;
        if (j.stage == 0) {
            double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int64_t i = j.first; i < j.last; ++i)
                for (int a = 0; a < 3; ++a) {
                    bl[a] = std::min(bl[a], lo[3 * size_t(order[i]) + a]);
                    bh[a] = std::max(bh[a], hi[3 * size_t(order[i]) + a]);
                }
            int axis = 0;
            if (bh[1] - bl[1] > bh[0] - bl[0]) axis = 1;
            if (bh[2] - bl[2] > bh[axis] - bl[axis]) axis = 2;
            std::nth_element(order.begin() + j.first, order.begin() + mid, order.begin() + j.last,
                             [&](int32_t x, int32_t y) {
                                 const double cx = ce[3 * size_t(x) + axis], cy = ce[3 * size_t(y) + axis];
                                 return cx != cy ? cx < cy : x < y;
                             });
            j.stage = 1;
            node.left = next++;
            stack.push_back({j.first, mid, node.left, 0});
        } else if (j.stage == 1) {
            j.stage = 2;
            node.right = next++;
            stack.push_back({mid, j.last, node.right, 0});
        } else {
            const sd_bvh_node& l = out[node.left];
            const sd_bvh_node& r = out[node.right];
            node.primitive = -1;
            node.count = l.count + r.count;
            for (int a = 0; a < 3; ++a) {
                node.lo[a] = std::min(l.lo[a], r.lo[a]);
                node.hi[a] = std::max(l.hi[a], r.hi[a]);
            }
            node.diameter = diag(node.lo, node.hi);
            stack.pop_back();
        }
    }
}

void tree_build_median_host(Ctx& c) {
    median_build_host(c, c.tree);
    c.tree_trusted = true;
    c.dtree_ready = false;
    c.sx_tree_ready = c.sx_prim_ready = false;
}

// ---------------------------------------------------------------- upload
template <class T>
void upload_tree_device(Ctx& c, DeviceTree& t, int depth);  // layout.cu

// Checks an externally supplied tree (sd_set_bvh, SDBV0001 cache) and returns
// its depth; trees from this library's builders skip the check.
static int validate_tree(const Ctx& c) {
    const int64_t n = int64_t(c.tree.size());
    const int64_t N = c.N;
    if (n != 2 * N - 1) throw std::runtime_error("tree must have 2N - 1 nodes");
    std::vector<int32_t> dep(size_t(n), 0);
    int depth = 0;
    if (c.tree_trusted) {  // pre-order: parents precede children
        for (int64_t id = 0; id < n; ++id) {
            const sd_bvh_node& nd = c.tree[id];
            depth = std::max(depth, dep[id]);
            if (nd.left >= 0) dep[nd.left] = dep[nd.right] = dep[id] + 1;
        }
        return depth;
    }
    // validate and compute the pre-order numbering of the given tree
    std::vector<int32_t> pre(n, -1), stack;
    int64_t visited = 0;
    stack.push_back(0);
    std::vector<char> seen_prim(N, 0);
    while (!stack.empty()) {
        const int32_t id = stack.back();
        stack.pop_back();
        if (id < 0 || id >= n || pre[id] >= 0) throw std::runtime_error("tree: bad or repeated child index");
        pre[id] = int32_t(visited++);
        const sd_bvh_node& nd = c.tree[id];
        depth = std::max(depth, dep[id]);
        if (nd.left < 0) {
            if (nd.primitive < 0 || nd.primitive >= N || seen_prim[nd.primitive])
                throw std::runtime_error("tree: bad or repeated leaf primitive");
            seen_prim[nd.primitive] = 1;
        } else {
            if (nd.right < 0 || nd.right >= n || nd.left >= n) throw std::runtime_error("tree: bad child index");
            dep[nd.left] = dep[nd.right] = dep[id] + 1;
            stack.push_back(nd.right);
            stack.push_back(nd.left);
        }
    }
    if (visited != n) throw std::runtime_error("tree: unreachable nodes");
    for (int64_t i = 0; i < n; ++i)
        if (pre[i] != i) throw std::runtime_error("tree must be in pre-order layout (left child = parent + 1, root 0)");
    return depth;
}

template <class T>
static void upload_tree_T(Ctx& c, DeviceTree& t) {
    upload_tree_device<T>(c, t, validate_tree(c));
}

// Split slots at depth k (see pair_kernel): nodes at depth k and leaves
// above it, in pre-order; per slot its ancestors (root first) and the bits
// of those ancestors whose first slot (in pre-order) it is. Cached per k.
void split_tables(Ctx& c, DeviceTree& t, int k) {
    if (t.split_k == k) return;
    const int64_t n = int64_t(c.tree.size());
    std::vector<int32_t> parent(size_t(n), -1), dep(size_t(n), 0);
    for (int64_t id = 0; id < n; ++id) {  // pre-order: parents precede children
        const sd_bvh_node& nd = c.tree[id];
        if (nd.left >= 0) {
            dep[nd.left] = dep[nd.right] = dep[id] + 1;
            parent[nd.left] = parent[nd.right] = int32_t(id);
        }
    }
    std::vector<char> has_first(size_t(n), 0);
    std::vector<int2> meta;
    std::vector<int32_t> path;
    std::vector<int32_t> anc;
    for (int64_t id = 0; id < n; ++id) {
        const bool leaf = c.tree[id].left < 0;
        if (!(dep[id] == k || (leaf && dep[id] < k))) continue;
        anc.clear();
        for (int32_t p = parent[id]; p >= 0; p = parent[p]) anc.push_back(p);
        std::reverse(anc.begin(), anc.end());  // root first
        unsigned first = 0;
        for (size_t j = 0; j < anc.size(); ++j)
            if (!has_first[anc[j]]) {
                has_first[anc[j]] = 1;
                first |= 1u << j;
            }
        meta.push_back(make_int2(int(id), int(anc.size()) | int(first << 8)));
        for (int j = 0; j < k; ++j) path.push_back(j < int(anc.size()) ? anc[j] : 0);
    }
    t.split_count = int64_t(meta.size());
    auto up = [](DevBuf& buf, const void* src, size_t bytes) {
        void* d = buf.ensure(bytes);
        if (bytes) check_cuda(cudaMemcpy(d, src, bytes, cudaMemcpyHostToDevice), "upload split tables");
    };
    up(t.split_meta, meta.data(), meta.size() * sizeof(int2));
    up(t.split_path, path.data(), path.size() * sizeof(int32_t));
    t.split_k = k;
}

void tree_upload(Ctx& c) {
    c.dtree.contact_rc2 = -1.f;
    if (c.precision == SD_FP32) upload_tree_T<float>(c, c.dtree);
    else upload_tree_T<double>(c, c.dtree);
    c.dtree_ready = true;
}

void tree_upload64(Ctx& c, DeviceTree& t) { upload_tree_T<double>(c, t); }

// ---------------------------------------------------------- query order
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

template <class T, class I>
__global__ void query_morton(const T* __restrict__ q, int64_t Q, double3 lo, double3 inv, uint32_t* keys,
                             I* idx) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    auto cell = [](double x, double l, double s) {
        const double f = (x - l) * s;
        return uint32_t(fmin(fmax(f, 0.0), 1023.0));
    };
    const uint32_t x = cell(double(q[3 * i]), lo.x, inv.x);
    const uint32_t y = cell(double(q[3 * i + 1]), lo.y, inv.y);
    const uint32_t z = cell(double(q[3 * i + 2]), lo.z, inv.z);
    const T a = q[3 * i], b = q[3 * i + 1], d = q[3 * i + 2];
    keys[i] = (a == a && b == b && d == d) ? (spread10(x) << 2) | (spread10(y) << 1) | spread10(z) : 0xffffffffu;
    idx[i] = I(i);
}

// ------------------------------------------------------------ traversal
// Unit-weight edge / triangle leaf (poly_index < 0): w = A^S.
template <class T, int KIND, bool FIX>
__device__ __forceinline__ void unit_term(const Phys<T>& ph, const Poly<T>& pc, T qx, T qy, T qz, const T* rec,
                                          Acc<T>& acc, bool* contact) {
    acc.m -= ph.lw_unit;
    if constexpr (KIND == 1) edge_term<T, false, false>(ph, pc, qx, qy, qz, rec, acc);
    else tri_term<T, false, false, FIX>(ph, pc, qx, qy, qz, rec, acc, contact);
    acc.m += ph.lw_unit;
}

// Reference-rounded fp64 decision (bvh.hpp:105-111,185-187).
template <class T>
__device__ __forceinline__ bool decide64(const NodeT<T>& b, double d64, double qx, double qy, double qz,
                                         double beta) {
    const double yx = fmin(fmax(qx, double(b.v[0])), double(b.v[4]));
    const double yy = fmin(fmax(qy, double(b.v[1])), double(b.v[5]));
    const double yz = fmin(fmax(qz, double(b.v[2])), double(b.v[6]));
    const double dx = __dsub_rn(qx, yx), dy = __dsub_rn(qy, yy), dz = __dsub_rn(qz, yz);
    const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const double d = __dsqrt_rn(s);
    return d > 0.0 && d64 < __dmul_rn(beta, d);
}

// Exact leaf term (smooth.hpp:51-61) of the primitive in leaf slot `slot`
// for query q, added to acc.
// FIX / contact: see tri_contact (pair.cuh). K3 and K3F add the exact-
// normal form inline (FIX); K3Q's cooperative flush adds the term as is
// (FIX off) and K3C (contact_search) corrects it after the walk.
template <class T, bool FIX = true>
__device__ __forceinline__ void leaf_term(const TraverseArgs<T>& a, const Poly<T>* polys, int slot, T qx, T qy, T qz,
                                          Acc<T>& acc, bool* contact = nullptr) {
    const int meta = a.leafmeta[slot];
    const int kind = meta & 3, poly = (meta >> 2) - 1;
    T rec[kRecTri];
    using V = typename Vec4<T>::type;
    const V* src = reinterpret_cast<const V*>(a.leafrec + size_t(slot) * kRecTri);
    if (kind == 0) {
        for (int j = 0; j < kRecPoint * int(sizeof(T)) / int(sizeof(V)); ++j) reinterpret_cast<V*>(rec)[j] = src[j];
        acc.m -= a.ph.lw_unit;
        point_term(a.ph, qx, qy, qz, rec[0], rec[1], rec[2], acc);
        acc.m += a.ph.lw_unit;
    } else if (kind == 1) {
#pragma unroll
        for (int j = 0; j < kRecEdge * int(sizeof(T)) / int(sizeof(V)); ++j) reinterpret_cast<V*>(rec)[j] = src[j];
        if (poly >= 0) edge_term<T, true, false>(a.ph, polys[poly], qx, qy, qz, rec, acc);
        else unit_term<T, 1, FIX>(a.ph, polys[0], qx, qy, qz, rec, acc, contact);
    } else {
#pragma unroll
        for (int j = 0; j < kRecTri * int(sizeof(T)) / int(sizeof(V)); ++j) reinterpret_cast<V*>(rec)[j] = src[j];
        if (poly >= 0) tri_term<T, true, false, FIX>(a.ph, polys[a.ne + poly], qx, qy, qz, rec, acc, contact);
        else unit_term<T, 2, FIX>(a.ph, polys[0], qx, qy, qz, rec, acc, contact);
    }
}

// Exact leaf visit of one lane; the record is the same for every lane of
// the warp.
template <class T, bool HASH, class CNT>
__device__ __forceinline__ void leaf_visit(const TraverseArgs<T>& a, const Poly<T>* polys, int32_t id, int32_t link,
                                           T qx, T qy, T qz, Acc<T>& acc, CNT& nleaf, uint64_t& h) {
    leaf_term<T>(a, polys, -link - 1, qx, qy, qz, acc);
    ++nleaf;
    if constexpr (HASH) h += decision_mix(uint64_t(id), 2);
}

// Adds a partial (m, s, g) -- sums relative to 2^m -- into acc.
template <class T>
__device__ __forceinline__ void merge_partial(Acc<T>& acc, T m, T s, T gx, T gy, T gz) {
    if (m > acc.m) {
        acc.scale(Math<T>::ex2(acc.m - m));
        acc.m = m;
    }
    const T f = m == acc.m ? T(1) : Math<T>::ex2(m - acc.m);
    acc.s = fma(s, f, acc.s);
    acc.gx = fma(gx, f, acc.gx);
    acc.gy = fma(gy, f, acc.gy);
    acc.gz = fma(gz, f, acc.gz);
}


// Barnes-Hut admissibility of box b for query point q (bvh.hpp:105-111,
// 185-187): fp32 decides outside a 1e-5 relative band, fp64 re-decides in
// the reference rounding inside it. On "far" also returns d_B, 1/d_B and
// q - y_B for the far-field term.
template <class T>
__device__ __forceinline__ bool point_far(const TraverseArgs<T>& a, const NodeT<T>& b, int32_t id, T qx, T qy, T qz,
                                          T& d, T& r, T& dx, T& dy, T& dz, unsigned long long& nre) {
    const T yx = fmin(fmax(qx, b.v[0]), b.v[4]);
    const T yy = fmin(fmax(qy, b.v[1]), b.v[5]);
    const T yz = fmin(fmax(qz, b.v[2]), b.v[6]);
    dx = qx - yx;
    dy = qy - yy;
    dz = qz - yz;
    const T s = fma(dx, dx, fma(dy, dy, dz * dz));
    bool far;
    if constexpr (sizeof(T) == 4) {
        // squared: diam^2 against beta^2 s with a 2e-5 relative band (the
        // reciprocal square root only for far-field nodes)
        const T dd = b.v[3] * b.v[3], rhs2 = (a.ph.beta * a.ph.beta) * s;
        const T gap = dd - rhs2;  // exact sign outside the band (|gap| >> its rounding)
        if (fabs(gap) > T(2e-5) * rhs2) far = gap < T(0);
        else if (s == T(0) && a.exact_boxes) far = false;
        else {
            far = decide64(b, a.diam64[id], double(qx), double(qy), double(qz), a.beta64);
            ++nre;
        }
        if (far) {  // s = 0 only for an fp64-confirmed box that the fp32 box contains; then dx = dy = dz = 0
            r = Math<T>::rsqrt(fmax(s, T(1e-30)));
            d = s * r;
        }
    } else {
        // squared test with FMA-contracted s and a 1e-12 relative band; the
        // reference-rounded decision (sqrt and all) only inside the band
        const double diam = b.v[3];  // the fp64 diameter itself (T = double)
        const double dd = diam * diam, rhs2 = a.beta64 * a.beta64 * s;
        if (s == 0.0) far = false;  // d_B = 0 exactly: fp64 boxes are the reference's
        else if (dd < rhs2 * (1.0 - 1e-12)) far = true;
        else if (dd > rhs2 * (1.0 + 1e-12)) far = false;
        else {
            far = decide64(b, a.diam64[id], double(qx), double(qy), double(qz), a.beta64);
            ++nre;
        }
        if (far) {
            r = Math<double>::rsqrt(s);
            d = s * r;
        }
    }
    return far;
}

// One node test of the packet traversal for one lane (decision + term),
// shared by the single-node and child-pair kernels. Returns "descend".
template <class T, bool HASH, class CNT>
__device__ __forceinline__ bool visit(const TraverseArgs<T>& a, const Poly<T>* polys, const NodeT<T>& b,
                                      int32_t id, T lgc, T qx, T qy, T qz, Acc<T>& acc, CNT& nleaf,
                                      CNT& nfar, uint64_t& h, unsigned long long& nre) {
    int32_t link;
    memcpy(&link, &b.v[7], sizeof(int32_t));
    {  // no Barnes-Hut (beta <= 0): tree_query passes beta = 0, which is never admissible
        T d, r, dx, dy, dz;
        if (point_far(a, b, id, qx, qy, qz, d, r, dx, dy, dz, nre)) {
            far_term(a.ph, lgc + a.lw_ff, d, r, dx, dy, dz, acc);
            ++nfar;
            if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
            return false;
        }
    }
    if (link >= 0) return true;
    leaf_visit<T, HASH, CNT>(a, polys, id, link, qx, qy, qz, acc, nleaf, h);
    return false;
}

// The fp32 K3Q walk keeps each lane's shift relative to log2 w_ff (the
// far-field weight), so that a far-field term's exponent is kappa d +
// log2 n_B - m without adding log2 w_ff per term; leaf terms convert.
template <class T>
constexpr bool kFarFrame = sizeof(T) == 4;

// The point query of one lane (K3's VIS for bvh.cu).
template <class T>
struct PointVisit {
    static constexpr bool kLeafQueue = true;
    template <class U>
    static constexpr bool kFrame = kFarFrame<U>;
    T qx, qy, qz;
    __device__ __forceinline__ void load(const TraverseArgs<T>& a, int64_t qi, bool valid) {
        qx = valid ? a.q[3 * qi] : T(0);
        qy = valid ? a.q[3 * qi + 1] : T(0);
        qz = valid ? a.q[3 * qi + 2] : T(0);
    }
    template <bool HASH, class CNT>
    __device__ __forceinline__ bool visit(const TraverseArgs<T>& a, const Poly<T>* polys, const NodeT<T>& b,
                                          int32_t id, T lgc, Acc<T>& acc, CNT& nleaf, CNT& nfar, uint64_t& h,
                                          unsigned long long& nre) const {
        return sdgpu::visit<T, HASH, CNT>(a, polys, b, id, lgc, qx, qy, qz, acc, nleaf, nfar, h, nre);
    }
    // K3Q node test: far field inline; an exact leaf is counted, hashed and
    // appended to this lane's leaf queue (its term comes in leaf_round).
    template <bool HASH, class CNT>
    __device__ __forceinline__ bool visit_q(const TraverseArgs<T>& a, const NodeT<T>& b, int32_t id, T lgc,
                                            Acc<T>& acc, CNT& nleaf, CNT& nfar, uint64_t& h,
                                            unsigned long long& nre, uint32_t lq0, int& nq) const {
        int32_t link;
        memcpy(&link, &b.v[7], sizeof(int32_t));
        {  // beta = 0 when there is no Barnes-Hut (see visit)
            T d, r, dx, dy, dz;
            if (point_far(a, b, id, qx, qy, qz, d, r, dx, dy, dz, nre)) {
                far_term(a.ph, lgc + a.lw_ff, d, r, dx, dy, dz, acc);
                ++nfar;
                if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
                return false;
            }
        }
        if (link >= 0) return true;
        asm volatile("st.shared.s32 [%0], %1;" ::"r"(lq0 + uint32_t(nq) * kLeafStride), "r"(link) : "memory");
        ++nq;
        ++nleaf;
        if constexpr (HASH) h += decision_mix(uint64_t(id), 2);
        return false;
    }
    // K3Q step: both children of a node. fp32: the box tests of the two
    // children run as one packed fp32x2 sequence on the interleaved pair
    // record (clamps and the decisions per child; each child's decision is
    // point_far's, bit for bit -- the fp64 re-check band included); fp64:
    // two visit_q calls. active = this lane reached the node.
    template <bool HASH, class CNT>
    __device__ __forceinline__ void visit_pair_q(const TraverseArgs<T>& a, const PairT<T>& pr, int32_t lid,
                                                 int32_t rid, bool active, Acc<T>& acc, CNT& nleaf, CNT& nfar,
                                                 uint64_t& h, unsigned long long& nre, uint32_t lq0, int& nq,
                                                 bool& dl, bool& dr, int32_t& llink, int32_t& rlink) const {
        if constexpr (sizeof(T) == 8) {
            const NodeT<T> bl = pr.l(), br = pr.r();
            memcpy(&llink, &bl.v[7], sizeof(int32_t));
            memcpy(&rlink, &br.v[7], sizeof(int32_t));
            if (active) {
                dl = visit_q<HASH>(a, bl, lid, pr.lgc[0], acc, nleaf, nfar, h, nre, lq0, nq);
                dr = visit_q<HASH>(a, br, rid, pr.lgc[1], acc, nleaf, nfar, h, nre, lq0, nq);
            }
        } else {
            const float4* p4 = reinterpret_cast<const float4*>(pr.w);
            // (lo.x, lo.y | lo.z, diam | hi.x, hi.y | hi.z, link) of (left, right)
            const float4 w0 = p4[0], w1 = p4[1], w2 = p4[2], w3 = p4[3];
            const float2 lg = *reinterpret_cast<const float2*>(pr.lgc);
            memcpy(&llink, &w3.z, sizeof(int32_t));
            memcpy(&rlink, &w3.w, sizeof(int32_t));
            if (!active) return;
            const f2 dx = sub2(bcast(qx), pack(fminf(fmaxf(qx, w0.x), w2.x), fminf(fmaxf(qx, w0.y), w2.y)));
            const f2 dy = sub2(bcast(qy), pack(fminf(fmaxf(qy, w0.z), w2.z), fminf(fmaxf(qy, w0.w), w2.w)));
            const f2 dz = sub2(bcast(qz), pack(fminf(fmaxf(qz, w1.x), w3.x), fminf(fmaxf(qz, w1.y), w3.y)));
            const f2 s2 = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
            const float b2 = a.ph.beta * a.ph.beta;
            const f2 diam = pack(w1.z, w1.w);
            const f2 gap = fma2(diam, diam, mul2(bcast(-b2), s2));  // diam^2 - beta^2 s
            const f2 band = mul2(bcast(2e-5f * b2), s2);
            auto child = [&](int hh, int32_t id, int32_t link, float lgc) -> bool {
                const float g = hh ? hi(gap) : lo(gap), bd = hh ? hi(band) : lo(band), s = hh ? hi(s2) : lo(s2);
                bool far;
                if (fabsf(g) > bd) far = g < 0.f;
                else if (s == 0.f && a.exact_boxes) far = false;
                else {
                    const NodeT<float> b = hh ? pr.r() : pr.l();
                    far = decide64(b, a.diam64[id], double(qx), double(qy), double(qz), a.beta64);
                    ++nre;
                }
                if (far) {
                    const float r = Math<float>::rsqrt(fmaxf(s, 1e-30f));
                    far_term(a.ph, lgc, s * r, r, hh ? hi(dx) : lo(dx), hh ? hi(dy) : lo(dy),
                             hh ? hi(dz) : lo(dz), acc);
                    ++nfar;
                    if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
                    return false;
                }
                if (link >= 0) return true;
                asm volatile("st.shared.s32 [%0], %1;" ::"r"(lq0 + uint32_t(nq) * kLeafStride), "r"(link)
                             : "memory");
                ++nq;
                ++nleaf;
                if constexpr (HASH) h += decision_mix(uint64_t(id), 2);
                return false;
            };
            dl = child(0, lid, llink, lg.x);
            dr = child(1, rid, rlink, lg.y);
        }
    }
    // All pending leaf entries of the warp at once (called by the whole
    // warp): item t (in the lanes' queue order) belongs to the owner lane o
    // with excl[o] <= t < excl[o] + nq[o]; 32 items per round are spread
    // over the 32 lanes, each evaluated for its owner's query (coordinates
    // and shift by shuffle) into a partial relative to the owner's shift
    // (raised only by a term above it). The items of one owner are
    // contiguous, so a segmented max / sum over the lanes (starts known from
    // excl) gives each owner one partial per round, merged into its
    // accumulator. Per lane the terms are exactly the queued leaves'; only
    // the summation order changes. lqw: the warp's lane-0 queue address.
    __device__ __forceinline__ void leaf_flush_coop(const TraverseArgs<T>& a, const Poly<T>* polys, Acc<T>& acc,
                                                    uint32_t lqw, int& nq, unsigned lane) const {
        constexpr unsigned FULL = 0xffffffffu;
        const T frame = kFarFrame<T> ? a.lw_ff : T(0);  // acc.m is kept relative to log2 w_ff (fp32 walk)
        int incl = nq;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL, incl, o);
            if (int(lane) >= o) incl += y;
        }
        const int excl = incl - nq;
        const int total = __shfl_sync(FULL, incl, 31);
        for (int base = 0; base < total; base += 32) {
            const int t = base + int(lane);
            int o = 0;  // owner: the first lane whose inclusive count exceeds t
#pragma unroll
            for (int step = 16; step; step >>= 1)
                if (__shfl_sync(FULL, incl, o + step - 1) <= t) o += step;
            o &= 31;
            const int oex = __shfl_sync(FULL, excl, o);
            const T ox = __shfl_sync(FULL, qx, o), oy = __shfl_sync(FULL, qy, o), oz = __shfl_sync(FULL, qz, o);
            Acc<T> it;
            it.m = __shfl_sync(FULL, acc.m, o) + frame;
            it.s = it.gx = it.gy = it.gz = T(0);
            if (t < total) {
                int slot;
                asm volatile("ld.shared.s32 %0, [%1];"
                             : "=r"(slot)
                             : "r"(lqw + uint32_t(o) * 4u + uint32_t(t - oex) * kLeafStride));
                // (FIX off: near-contact face terms are corrected after the
                // walk by K3C, contact_search, to keep this loop's registers)
                leaf_term<T, false>(a, polys, -slot - 1, ox, oy, oz, it);  // the leaf link -(slot + 1)
            }
            // segmented max of the shifts, then segmented sums, over the
            // lanes of each owner's run in this round
            const int s0 = max(oex - base, 0);  // this run's first lane
            T m = it.m;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const T y = __shfl_up_sync(FULL, m, off);
                if (int(lane) - off >= s0) m = fmax(m, y);
            }
            const int oend = min(__shfl_sync(FULL, incl, o), base + 32) - 1 - base;  // run's last lane
            m = __shfl_sync(FULL, m, oend);
            const T f = t >= total ? T(0) : (it.m == m ? T(1) : Math<T>::ex2(it.m - m));
            T v0 = it.s * f, v1 = it.gx * f, v2 = it.gy * f, v3 = it.gz * f;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const T y0 = __shfl_up_sync(FULL, v0, off), y1 = __shfl_up_sync(FULL, v1, off),
                        y2 = __shfl_up_sync(FULL, v2, off), y3 = __shfl_up_sync(FULL, v3, off);
                if (int(lane) - off >= s0) {
                    v0 += y0;
                    v1 += y1;
                    v2 += y2;
                    v3 += y3;
                }
            }
            // each owner collects its run's total from the run's last lane
            const int my_lo = excl - base, my_hi = min(incl, base + 32) - 1 - base;
            const bool mine = nq > 0 && my_lo < 32 && my_hi >= 0 && my_hi >= my_lo;
            const int src = mine ? my_hi : 0;
            const T rm = __shfl_sync(FULL, m, src), r0 = __shfl_sync(FULL, v0, src), r1 = __shfl_sync(FULL, v1, src),
                    r2 = __shfl_sync(FULL, v2, src), r3 = __shfl_sync(FULL, v3, src);
            if (mine && r0 != T(0)) merge_partial(acc, rm - frame, r0, r1, r2, r3);
        }
        nq = 0;
    }
    __device__ __forceinline__ void leaf_round(const TraverseArgs<T>& a, const Poly<T>* polys, int link,
                                               Acc<T>& acc) const {
        if constexpr (kFarFrame<T>) acc.m += a.lw_ff;
        leaf_term<T>(a, polys, -link - 1, qx, qy, qz, acc);  // queued: the leaf link -(slot + 1)
        if constexpr (kFarFrame<T>) acc.m -= a.lw_ff;
    }
    template <bool HASH, class CNT>
    __device__ __forceinline__ bool far_test(const TraverseArgs<T>& a, const NodeT<T>& b, int32_t id, T lgc, bool emit,
                                             Acc<T>& acc, CNT& nfar, uint64_t& h, unsigned long long& nre) const {
        if (!a.use_bh) return false;
        T d, r, dx, dy, dz;
        if (!point_far(a, b, id, qx, qy, qz, d, r, dx, dy, dz, nre)) return false;
        if (emit) {
            far_term(a.ph, lgc + a.lw_ff, d, r, dx, dy, dz, acc);
            ++nfar;
            if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
        }
        return true;
    }

    // Both children of a node (K3's child-pair step in the split walk): two
    // scalar tests.
    template <bool HASH, class CNT>
    __device__ __forceinline__ void visit_pair(const TraverseArgs<T>& a, const Poly<T>* polys, const NodeT<T>& bl,
                                               const NodeT<T>& br, int32_t lid, int32_t rid, T lgl, T lgr,
                                               Acc<T>& acc, CNT& nleaf, CNT& nfar, uint64_t& h,
                                               unsigned long long& nre, bool& dl, bool& dr) const {
        dl = visit<HASH>(a, polys, bl, lid, lgl, acc, nleaf, nfar, h, nre);
        dr = visit<HASH>(a, polys, br, rid, lgr, acc, nleaf, nfar, h, nre);
    }
};

// The queries' bounding box as order-preserving uint32 images of the
// fp32 coordinates (min in [0..2], max in [3..5]): one pass, a warp / block
// reduction and one atomic per block and component (was a CUB reduce over
// a 24-byte struct: 25 us at cfg4, now a few).
__device__ __forceinline__ uint32_t ord_f32(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}
__global__ void qbox_init(uint32_t* ob) {
    if (threadIdx.x < 6) ob[threadIdx.x] = threadIdx.x < 3 ? 0xffffffffu : 0u;
}
template <class T>
__global__ void __launch_bounds__(256) qbox_reduce(const T* __restrict__ q, int64_t Q, uint32_t* ob) {
    uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < Q; i += int64_t(gridDim.x) * blockDim.x)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float f = float(q[3 * i + k]);
            if (f == f) {  // (NaN coordinates do not widen the box)
                const uint32_t o = ord_f32(f);
                lo[k] = min(lo[k], o);
                hi[k] = max(hi[k], o);
            }
        }
    __shared__ uint32_t red[6][8];
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int off = 16; off; off >>= 1) {
            lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], off));
            hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], off));
        }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
        for (int k = 0; k < 3; ++k) {
            red[k][w] = lo[k];
            red[3 + k][w] = hi[k];
        }
    __syncthreads();
    if (threadIdx.x < 3) {
        uint32_t a = red[threadIdx.x][0], b = red[3 + threadIdx.x][0];
        for (int j = 1; j < int(blockDim.x >> 5); ++j) {
            a = min(a, red[threadIdx.x][j]);
            b = max(b, red[3 + threadIdx.x][j]);
        }
        atomicMin(ob + threadIdx.x, a);
        atomicMax(ob + 3 + threadIdx.x, b);
    }
}

// Hilbert (or Morton) keys over the union of [lo, hi] (the root box) and
// the queries' own box, read from device memory (no host round trip):
// queries outside the scene keep distinct cells instead of piling up on its
// faces. Cells in fp32 (the order only shapes the packets, not the results).
template <class T, class I>
__global__ void query_morton_union(const T* __restrict__ q, int64_t Q, float3 lo, float3 hi,
                                   const uint32_t* __restrict__ ob, int hilbert, uint32_t* keys, I* idx) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    const float l[3] = {fminf(lo.x, unord_f32(ob[0])), fminf(lo.y, unord_f32(ob[1])), fminf(lo.z, unord_f32(ob[2]))};
    const float h[3] = {fmaxf(hi.x, unord_f32(ob[3])), fmaxf(hi.y, unord_f32(ob[4])), fmaxf(hi.z, unord_f32(ob[5]))};
    uint32_t cell[3];
    for (int a = 0; a < 3; ++a) {
        const float s = h[a] > l[a] ? 1024.0f / (h[a] - l[a]) : 0.0f;
        cell[a] = uint32_t(fminf(fmaxf((float(q[3 * i + a]) - l[a]) * s, 0.0f), 1023.0f));
    }
    uint32_t key = 0;
    if (hilbert) {
        // Skilling's transpose-to-Hilbert (10 bits per axis), then interleave
        uint32_t X[3] = {cell[0], cell[1], cell[2]};
        for (uint32_t Qb = 1u << 9; Qb > 1; Qb >>= 1) {
            const uint32_t P = Qb - 1;
            for (int k = 0; k < 3; ++k) {
                if (X[k] & Qb) X[0] ^= P;
                else {
                    const uint32_t t = (X[0] ^ X[k]) & P;
                    X[0] ^= t;
                    X[k] ^= t;
                }
            }
        }
        X[1] ^= X[0];
        X[2] ^= X[1];
        uint32_t t = 0;
        for (uint32_t Qb = 1u << 9; Qb > 1; Qb >>= 1)
            if (X[2] & Qb) t ^= Qb - 1;
        for (int k = 0; k < 3; ++k) X[k] ^= t;
        key = (spread10(X[0]) << 2) | (spread10(X[1]) << 1) | spread10(X[2]);
    } else {
        for (int a = 0; a < 3; ++a) key |= spread10(cell[a]) << (2 - a);
    }
    const T x = q[3 * i], y = q[3 * i + 1], z = q[3 * i + 2];
    keys[i] = (x == x && y == y && z == z) ? key : 0xffffffffu;  // NaN: last, and flagged for K4
    idx[i] = I(i);
}

// Morton codes (10 bits per axis over [lo, hi] joined with the queries'
// box) + CUB radix sort: the returned permutation lists query indices in
// spatial order (device memory owned by the context).
// sorted 32-bit query indices -> the int64 perm (grid-stride, coalesced)
__global__ void widen_perm(const uint32_t* __restrict__ in, int64_t n, int64_t* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

template <class T>
const int64_t* sort_queries(Ctx& c, const T* q, int64_t Q, const double lo[3], const double hi[3], cudaStream_t st,
                            int64_t& launches, bool union_hilbert) {
    uint32_t* keys = static_cast<uint32_t*>(c.keys.ensure(size_t(Q) * 2 * sizeof(uint32_t)));
    int64_t* idx = static_cast<int64_t*>(c.perm.ensure(size_t(Q) * 2 * sizeof(int64_t)));
    // batches below 2^31 queries sort 32-bit indices (8 instead of 12 bytes
    // per element and radix pass; the same stable order) in the first half
    // of the perm buffer and widen them into the int64 perm (second half)
    static const bool idx64 = [] {  // SDGPU_SORT_IDX64=1: sort the int64 indices (A/B)
        const char* e = std::getenv("SDGPU_SORT_IDX64");
        return e && *e == '1';
    }();
    const bool narrow = !idx64 && Q < (int64_t(1) << 31);
    uint32_t* idx32 = reinterpret_cast<uint32_t*>(idx);  // [0, Q) in, [Q, 2Q) sorted
    const unsigned blocks = unsigned((Q + 255) / 256);
    static const bool union_box = [] {
        const char* e = std::getenv("SDGPU_QBOX");
        return !(e && *e == '0');
    }();
    if (union_box && union_hilbert) {
        uint32_t* ob = static_cast<uint32_t*>(c.qbox.ensure(6 * sizeof(uint32_t)));
        qbox_init<<<1, 32, 0, st>>>(ob);
        qbox_reduce<T><<<unsigned(std::min<int64_t>(148 * 8, std::max<int64_t>(1, (Q + 255) / 256))), 256, 0, st>>>(
            q, Q, ob);
        // Hilbert order by default (SDGPU_HILBERT=0: Morton): no long jumps
        // inside a 32-query packet (cfg4 26.9 -> 26.2 ms)
        static const int hilbert = [] {
            const char* e = std::getenv("SDGPU_HILBERT");
            return e && *e == '0' ? 0 : 1;
        }();
        // (the root box rounded outward to fp32)
        auto dn = [](double x) { return std::nextafter(float(x), -INFINITY); };
        auto up = [](double x) { return std::nextafter(float(x), INFINITY); };
        const float3 flo = make_float3(dn(lo[0]), dn(lo[1]), dn(lo[2]));
        const float3 fhi = make_float3(up(hi[0]), up(hi[1]), up(hi[2]));
        if (narrow) query_morton_union<T, uint32_t><<<blocks, 256, 0, st>>>(q, Q, flo, fhi, ob, hilbert, keys, idx32);
        else query_morton_union<T, int64_t><<<blocks, 256, 0, st>>>(q, Q, flo, fhi, ob, hilbert, keys, idx);
        launches += 3;
    } else {
        auto inv = [](double l, double h) { return h > l ? 1024.0 / (h - l) : 0.0; };
        const double3 dlo = make_double3(lo[0], lo[1], lo[2]);
        const double3 iv = make_double3(inv(lo[0], hi[0]), inv(lo[1], hi[1]), inv(lo[2], hi[2]));
        if (narrow) query_morton<T, uint32_t><<<blocks, 256, 0, st>>>(q, Q, dlo, iv, keys, idx32);
        else query_morton<T, int64_t><<<blocks, 256, 0, st>>>(q, Q, dlo, iv, keys, idx);
        ++launches;
    }
    check_cuda(cudaGetLastError(), "query morton");
    // SDGPU_SORT_BITS = b: order by the top b bits of the 30-bit key only
    // (a coarser curve, fewer radix passes; A/B)
    static const int lo_bit = [] {
        const char* e = std::getenv("SDGPU_SORT_BITS");
        const int b = e && *e ? std::atoi(e) : 30;
        return 30 - std::min(30, std::max(6, b));
    }();
    size_t tmp_bytes = 0;
    if (narrow) {
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys + Q, idx32, idx32 + Q, int(Q), lo_bit, 30, st);
        void* tmp = c.tmp.ensure(tmp_bytes);
        check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys + Q, idx32, idx32 + Q, int(Q), lo_bit,
                                                   30, st),
                   "radix sort queries");
        widen_perm<<<unsigned(std::min<int64_t>(148 * 16, (Q + 255) / 256)), 256, 0, st>>>(idx32 + Q, Q, idx + Q);
        check_cuda(cudaGetLastError(), "widen perm");
        ++launches;
    } else {
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys + Q, idx, idx + Q, int(Q), lo_bit, 30, st);
        void* tmp = c.tmp.ensure(tmp_bytes);
        check_cuda(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys + Q, idx, idx + Q, int(Q), lo_bit, 30,
                                                   st),
                   "radix sort queries");
    }
    launches += 4;  // onesweep histogram + passes (approximate count of CUB kernels)
    return idx + Q;
}
template const int64_t* sort_queries<float>(Ctx&, const float*, int64_t, const double*, const double*, cudaStream_t,
                                            int64_t&, bool);
template const int64_t* sort_queries<double>(Ctx&, const double*, int64_t, const double*, const double*,
                                             cudaStream_t, int64_t&, bool);

static bool variant_is_frontier(int64_t Q) { return use_frontier(Q, 65536); }

// K3C (fp32, with K3Q): the near-contact face terms. K3Q's cooperative
// leaf flush adds every exact leaf term as evaluated (tri_term with FIX off,
// pair.cuh: for a query within |ab| / 128 of a face's interior the fp32
// offset ap - u ab - v ac is rounding noise in direction); adding the
// exact-normal form inline costs the walk its register budget (56 -> 64+
// registers, 5 % at cfg4), so K3C finds those terms on the side:
//   contact_search -- on a second stream, concurrently with the walk: per
//     query (the same sorted packets and shard) a depth-first walk over the
//     boxes within r_c of the query (r_c = the largest |ab| / 128 of the
//     mesh, x sqrt 2); at each triangle leaf tri_contact's own test
//     (tri_near_contact); hits go to a list (sorted position, leaf slot);
//   contact_apply -- after the walk: each hit's term evaluated as the walk
//     did and in the exact-normal form, the difference added to the
//     query's fp64 partial.
// A face within |ab| / 128 of the query is always an exact leaf of the
// walk (its box and every ancestor's is at distance <= d, never admissible
// for beta < 128), so the corrected terms are exactly the walk's
// near-contact terms.
__global__ void __launch_bounds__(kTravThreads) contact_search(const __grid_constant__ TraverseArgs<float> a,
                                                               float rc2, uint64_t* hits, unsigned* nhits,
                                                               unsigned cap) {
    extern __shared__ __align__(16) int32_t cstk[];  // per thread: entry k at [k * kTravThreads + tid]
    const int64_t packet =
        shard_packet((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, a.pk_world, a.pk_rank, a.pk_chunk);
    const int64_t i = packet * 32 + (threadIdx.x & 31u);
    if (i >= a.Q) return;
    const int64_t qi = a.perm ? a.perm[i] : i;
    const float qx = a.q[3 * qi], qy = a.q[3 * qi + 1], qz = a.q[3 * qi + 2];
    auto near = [&](int32_t id) {
        const NodeT<float> b = a.box[id];
        const float dx = fmaxf(fmaxf(b.v[0] - qx, qx - b.v[4]), 0.f);
        const float dy = fmaxf(fmaxf(b.v[1] - qy, qy - b.v[5]), 0.f);
        const float dz = fmaxf(fmaxf(b.v[2] - qz, qz - b.v[6]), 0.f);
        return fmaf(dx, dx, fmaf(dy, dy, dz * dz)) <= rc2;
    };
    // (per lane: each lane its own few root-to-leaf paths, far cheaper here
    // than a packet walk over the union of 32 neighbourhoods)
    int32_t* stk = cstk + threadIdx.x;
    int sp = 0;
    if (near(0)) stk[sp++ * kTravThreads] = 0;
    while (sp > 0) {
        const int32_t id = stk[--sp * kTravThreads];
        int32_t link;
        memcpy(&link, &a.box[id].v[7], sizeof(int32_t));
        if (link >= 0) {  // internal: push the children within r_c (left on top)
            if (near(link)) stk[sp++ * kTravThreads] = link;
            if (near(id + 1)) stk[sp++ * kTravThreads] = id + 1;
            continue;
        }
        const int slot = -link - 1;
        if ((a.leafmeta[slot] & 3) != SD_TRIANGLE) continue;
        float rec[16];
        const float4* src = reinterpret_cast<const float4*>(a.leafrec + size_t(slot) * kRecTri);
#pragma unroll
        for (int j = 0; j < 4; ++j) reinterpret_cast<float4*>(rec)[j] = src[j];  // a, ab, ac, A B C, 1/A 1/C 1/|bc|^2 1/det
        if (!tri_near_contact(rec, qx, qy, qz)) continue;
        const unsigned k = atomicAdd(nhits, 1u);
        if (k < cap) hits[k] = (uint64_t(i) << 32) | uint32_t(slot);
    }
}

__global__ void contact_apply(const __grid_constant__ TraverseArgs<float> a, const uint64_t* hits,
                              const unsigned* nhits, unsigned cap) {
    const unsigned n = min(*nhits, cap);
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        const int64_t i = int64_t(hits[k] >> 32);
        const int slot = int(hits[k] & 0xffffffffu);
        const int64_t qi = a.perm ? a.perm[i] : i;
        const float qx = a.q[3 * qi], qy = a.q[3 * qi + 1], qz = a.q[3 * qi + 2];
        Acc<float> was, fix;
        was.init();
        fix.init();
        bool contact = false;
        leaf_term<float, false>(a, a.polys, slot, qx, qy, qz, was, &contact);
        if (!contact) continue;
        leaf_term<float, true>(a, a.polys, slot, qx, qy, qz, fix);
        const double M = a.part[i];  // the walk's anchor (finite: the term itself is in the sum)
        const double fw = was.s != 0.f ? exp2(double(was.m) - M) : 0.0;
        const double ff = fix.s != 0.f ? exp2(double(fix.m) - M) : 0.0;
        atomicAdd(a.part + a.Q + i, double(fix.s) * ff - double(was.s) * fw);
        atomicAdd(a.part + 2 * a.Q + i, double(fix.gx) * ff - double(was.gx) * fw);
        atomicAdd(a.part + 3 * a.Q + i, double(fix.gy) * ff - double(was.gy) * fw);
        atomicAdd(a.part + 4 * a.Q + i, double(fix.gz) * ff - double(was.gz) * fw);
    }
}

// K3C search radius (2 x the largest |ab|^2 / 16384 of the mesh's
// triangles: tri_contact's threshold with margin for the fp32 distance),
// cached per tree upload; 0: no triangles.
static float contact_radius2(Ctx& c) {
    DeviceTree& t = c.dtree;
    if (t.contact_rc2 < 0.f) {
        double m = 0.0;
        for (int64_t p = 0; p < c.N; ++p) {
            if (c.kind[p] != SD_TRIANGLE) continue;
            const double* x0 = &c.xyz[3 * size_t(c.sv[3 * p])];
            const double* x1 = &c.xyz[3 * size_t(c.sv[3 * p + 1])];
            const double dx = x1[0] - x0[0], dy = x1[1] - x0[1], dz = x1[2] - x0[2];
            m = std::max(m, dx * dx + dy * dy + dz * dz);
        }
        t.contact_rc2 = float(2.0 * m / 16384.0);
    }
    return t.contact_rc2;
}

// Fork: contact_search on c.aux_stream once the sorted order exists on st
// (call right before the walk's launch). Returns false if nothing to do.
static bool contact_fork(Ctx& c, TraverseArgs<float>& a, cudaStream_t st, int64_t& launches) {
    const float rc2 = contact_radius2(c);
    if (rc2 == 0.f || a.Q == 0) return false;
    const int64_t npackets = (a.Q + 31) / 32;
    const int64_t warps = a.pk_world > 1 ? shard_count(npackets, a.pk_world, a.pk_rank, a.pk_chunk) : npackets;
    if (warps == 0) return false;
    if (!c.aux_stream) {
        check_cuda(cudaStreamCreateWithFlags(&c.aux_stream, cudaStreamNonBlocking), "stream");
        check_cuda(cudaEventCreateWithFlags(&c.aux_fork, cudaEventDisableTiming), "event");
        check_cuda(cudaEventCreateWithFlags(&c.aux_join, cudaEventDisableTiming), "event");
    }
    c.contact_cap = unsigned(std::min<int64_t>(std::max<int64_t>(65536, a.Q / 64), int64_t(1) << 30));
    uint64_t* hits = static_cast<uint64_t*>(c.contact_hits.ensure(size_t(c.contact_cap) * sizeof(uint64_t) + 64));
    unsigned* nhits = reinterpret_cast<unsigned*>(hits + c.contact_cap);
    check_cuda(cudaMemsetAsync(nhits, 0, sizeof(unsigned), st), "memset");
    check_cuda(cudaEventRecord(c.aux_fork, st), "event");
    check_cuda(cudaStreamWaitEvent(c.aux_stream, c.aux_fork, 0), "wait");
    const size_t smem = size_t(a.stack_depth + 1) * kTravThreads * sizeof(int32_t);
    contact_search<<<unsigned((warps * 32 + kTravThreads - 1) / kTravThreads), kTravThreads, smem, c.aux_stream>>>(
        a, rc2, hits, nhits, c.contact_cap);
    check_cuda(cudaGetLastError(), "contact search");
    check_cuda(cudaEventRecord(c.aux_join, c.aux_stream), "event");
    ++launches;
    return true;
}

// Join: after the walk, st waits for the search and applies the hits.
static void contact_join(Ctx& c, TraverseArgs<float>& a, cudaStream_t st, int64_t& launches) {
    uint64_t* hits = c.contact_hits.as<uint64_t>();
    unsigned* nhits = reinterpret_cast<unsigned*>(hits + c.contact_cap);
    check_cuda(cudaStreamWaitEvent(st, c.aux_join, 0), "wait");
    contact_apply<<<148, 128, 0, st>>>(a, hits, nhits, c.contact_cap);
    check_cuda(cudaGetLastError(), "contact apply");
    ++launches;
}

template <class T>
void tree_query(Ctx& c, const T* q, int64_t Q, const sd_params& p, const FinalizeOut& out, cudaStream_t st) {
    if (!c.dtree_ready) tree_upload(c);
    const DeviceTree& t = c.dtree;
    int64_t launches = 0;
    // Morton order of the queries over the root box (coherent traversal)
    const sd_bvh_node& root = c.tree[0];
    // the one-query-per-warp kernel (K3F, few queries) gains nothing from a
    // spatial order that pays for its sort launches (render beta 0.5:
    // 6.92 -> 5.44 ms, Terrain / Bunny 0.265 -> 0.20 ms); SDGPU_FEW_SORT=1
    // sorts anyway
    static const bool few_sort = [] {
        const char* e = std::getenv("SDGPU_FEW_SORT");
        return e && *e == '1';
    }();
    const bool sharded = out.pk_world > 1;
    const int64_t* perm = (!few_sort && !sharded && variant_is_frontier(Q))
                              ? nullptr
                              : sort_queries(c, q, Q, root.lo, root.hi, st, launches, true);

    // polynomial table: edge polys then triangle polys
    const int ne = int(c.edge_a.size() / 5), nt = int(c.tri_stored.size() / 13);
    const int npoly = std::max(1, ne + nt);
    std::vector<Poly<T>> ptab(npoly);
    for (int e = 0; e < ne; ++e) ptab[e] = make_poly<T>(c, SD_EDGE, e, p);
    for (int k = 0; k < nt; ++k) ptab[ne + k] = make_poly<T>(c, SD_TRIANGLE, k, p);
    Poly<T>* dpoly = static_cast<Poly<T>*>(c.polys.ensure(ptab.size() * sizeof(Poly<T>)));
    check_cuda(cudaMemcpyAsync(dpoly, ptab.data(), ptab.size() * sizeof(Poly<T>), cudaMemcpyHostToDevice, st),
               "upload polys");

    double* part = static_cast<double*>(c.part.ensure(size_t(5) * Q * sizeof(double)));
    int64_t* cnt = static_cast<int64_t*>(c.counters.ensure(size_t(Q) * 3 * sizeof(int64_t) + 64));
    unsigned long long* re = reinterpret_cast<unsigned long long*>(cnt + 3 * Q);
    check_cuda(cudaMemsetAsync(re, 0, sizeof(unsigned long long), st), "memset");

    TraverseArgs<T> a;
    a.q = q;
    a.perm = perm;
    a.Q = Q;
    a.box = t.box.as<NodeT<T>>();
    a.pairs = t.pairs.as<PairT<T>>();
    a.count = t.count.as<int32_t>();
    a.lgcount = t.lgcount.as<T>();
    a.diam64 = t.diam64.as<double>();
    a.leafrec = t.leafrec.as<T>();
    a.leafmeta = t.leafmeta.as<int32_t>();
    a.polys = dpoly;
    a.ph = make_phys<T>(c, p);
    a.lw_ff = T(std::log2(std::pow(std::max(c.A * c.sup_wtilde, 1e-300), p.alpha / std::max(p.alpha, p.alpha_u))));
    a.ne = ne;
    a.npoly = npoly;
    a.use_bh = p.beta > 0.0 ? 1 : 0;
    a.exact_boxes = t.exact_boxes ? 1 : 0;
    a.stack_depth = t.depth + 1;
    a.beta64 = p.beta;
    a.ph = make_phys<T>(c, p);
    if (!a.use_bh) {  // smooth.hpp:106: no far field; beta = 0 makes every box test fail
        a.beta64 = 0.0;
        a.ph.beta = T(0);
    }
    a.part = part;
    a.leaves = cnt;
    a.far = cnt + Q;
    a.hash = reinterpret_cast<uint64_t*>(cnt + 2 * Q);
    a.rechecks = re;
    a.qgeom = nullptr;
    a.qdim = nullptr;
    a.leafgeom = nullptr;
    int nsplits = 1;
    KernelTimer timer(c, st);
    // few / sparse queries: node-parallel K3F (one warp per query); dense
    // batches: K3 packets (tools/frontier_crossover.py: cfg4, 1k..262k
    // queries: K3F 0.10 / 0.32 / 0.73 / 2.06 / 6.8 ms vs K3 2.8 / 7.0 / 7.7 /
    // 6.3 / 7.3 ms; the full dense 4.19M batch: K3 29.7 ms in round 1)
    a.pk_world = out.pk_world;
    a.pk_rank = out.pk_rank;
    a.pk_chunk = out.pk_chunk;
    bool contact = false;  // K3C forked (fp32 K3Q walks)
    if (!(!sharded && use_frontier(Q, 65536) &&
          launch_frontier<T, PointVisit<T>>(c, c.dtree, a, out.hash != nullptr, st, launches, 32))) {
        if constexpr (sizeof(T) == 4) {
            static const bool no_contact = [] {  // SDGPU_NO_CONTACT=1 skips K3C (A/B timing only)
                const char* e = std::getenv("SDGPU_NO_CONTACT");
                return e && *e == '1';
            }();
            // (K3Q runs its cooperative flush exactly when these hold: see launch_pair_traversal)
            if (!no_contact && will_use_coop_flush<T>(c.dtree, a)) contact = contact_fork(c, a, st, launches);
        }
        nsplits = launch_pair_traversal<T, PointVisit<T>>(c, c.dtree, a, out.hash != nullptr, st, launches, 1,
                                                             out.leaves || out.far_field);
    }
    if constexpr (sizeof(T) == 4)
        if (contact) contact_join(c, a, st, launches);  // K3C: K3Q's near-contact face terms
    timer.stop();
    FinalizeOut fo = out;
    if (perm) {  // NaN queries flagged in the sorted keys (coalesced, no scattered query re-read)
        fo.nan_keys = static_cast<const uint32_t*>(c.keys.p) + Q;
        fo.qf = nullptr;
        fo.qd = nullptr;
        if (out.grad && !out.peers && out.pk_world <= 1)
            fo.aos = static_cast<double*>(c.aos.ensure(size_t(Q) * 4 * sizeof(double)));
    }
    check_cuda(launch_finalize(a.part, nsplits, Q, p.alpha, p.epsilon, 0, a.leaves, a.far, a.hash, perm, fo, st),
               "finalize");
    ++launches;
    c.last_launches = launches;
}
template void tree_query<float>(Ctx&, const float*, int64_t, const sd_params&, const FinalizeOut&, cudaStream_t);
template void tree_query<double>(Ctx&, const double*, int64_t, const sd_params&, const FinalizeOut&, cudaStream_t);

}  // namespace sdgpu

