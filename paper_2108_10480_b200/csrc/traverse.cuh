// traverse.cuh -- K3, the warp-coherent child-pair BVH traversal shared by
// the point-query path (bvh.cu) and the simplex-query path (simplex.cu):
// traversal record layouts, kernel arguments, the far-field term, the
// kernel template (parameterised by the per-lane query type) and its host
// launcher with the few-query split mode.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "context.h"

namespace sdgpu {

template <class T>
struct alignas(16) NodeT {  // 2 x (4 T): (lo, diam) (hi, link)
    T v[8];
};
template <class T>
struct alignas(16) PairT {  // both children of an internal node + their log2 n_B
    NodeT<T> l, r;
    T lgc[4];
};

template <class T>
struct TraverseArgs {
    const T* q;
    const int64_t* perm;  // sorted position -> query index
    int64_t Q;
    const NodeT<T>* box;
    const PairT<T>* pairs;  // [parent]: the two children of an internal node
    const int32_t* count;
    const T* lgcount;     // log2 n_B per node (far-field weight exponent)
    T lw_ff;              // log2 w_ff
    const double* diam64;
    const T* leafrec;
    const int32_t* leafmeta;
    const Poly<T>* polys;  // [0, ne): edge polys, [ne, ne + nt): tri polys
    int ne, npoly;
    int use_bh;
    int exact_boxes;  // every fp32 box equals its fp64 box (quantized geometry)
    int stack_depth;
    double beta64;
    Phys<T> ph;
    double* part;       // [5][Q] fp64 state in sorted order
    int64_t* leaves;    // sorted order
    int64_t* far;
    uint64_t* hash;
    unsigned long long* rechecks;  // fp64 re-decisions (diagnostic)
    // split mode (few queries): see pair_kernel
    int split_depth, nslots;
    int64_t npackets;
    const int32_t* slot_of;     // node -> depth-k slot, or -1
    const int32_t* split_nodes;  // slot -> node
    unsigned* items;            // [packet][slot] lane mask reaching the slot
    // simplex queries (simplex.cu): fp64 corners and dims per query, and
    // the fp64 leaf geometry (16 doubles per leaf slot)
    const double* qgeom;
    const int32_t* qdim;
    const double* leafgeom;
};

constexpr int kTravThreads = 128;

// shared-memory bytes of the polynomial table, padded so the stacks after it
// stay 16-byte aligned
template <class T>
__host__ __device__ constexpr size_t poly_bytes(int npoly) {
    return (sizeof(Poly<T>) * size_t(npoly) + 15) / 16 * 16;
}

// Far-field term of a whole subtree (smooth.hpp:67-75): n_B w_ff collapsed
// onto the box's closest point; gradient (q - y_B) / d_B.
template <class T>
__device__ __forceinline__ void far_term(const Phys<T>& ph, T lw, T d, T r, T dx, T dy, T dz, Acc<T>& acc) {
    const T xm = bump(acc, masked(ph, d, fma(ph.kappa, d, lw - acc.m)), [&] { return fma(ph.kappa, d, lw); });
    const T e = Math<T>::ex2(xm);
    const T er = e * r;
    acc.s += e;
    acc.gx = fma(er, dx, acc.gx);
    acc.gy = fma(er, dy, acc.gy);
    acc.gz = fma(er, dz, acc.gz);
}

// K3 (default): warp-coherent packet traversal over CHILD PAIRS. The root
// is tested alone; afterwards every warp step fetches both children of
// the current node (one pair record, broadcast) and each lane whose own
// traversal reached the node tests both (far field / exact leaf / descend)
// -- per-lane decisions are exactly collect_contributions'
// (smooth.hpp:101-131). The warp continues into the left child if any lane
// descends there (pushing the right child with its lane mask), else into
// the right child, else pops. Stack entries (node, its link, mask, depth)
// live in shared memory, one stack per warp.
//
// SPLIT = 1 / 2 (few queries): the same walk cut at tree depth k. The top
// pass (1) stops above depth k and records, per query packet and depth-k
// node, the mask of lanes that reach it; the subtree pass (2) runs one warp
// per (packet, depth-k node) from that node with that mask. Each lane still
// visits exactly its reference node set; the partial sums land in split
// slots merged by K4, so a batch of a few thousand queries fills the GPU.
//
// VIS is the per-lane query: load(a, qi, valid) reads it, visit<HASH>(...)
// tests one node for it (point queries: bvh.cu; simplex queries:
// simplex.cu) and returns "descend".
template <class T, class VIS, bool HASH, int SPLIT>
__global__ void __launch_bounds__(kTravThreads) pair_kernel(const __grid_constant__ TraverseArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<T>* polys = reinterpret_cast<Poly<T>*>(smem_raw);
    int4* stacks = reinterpret_cast<int4*>(smem_raw + poly_bytes<T>(a.npoly));
    for (int i = threadIdx.x; i < a.npoly * kPolyCoefs; i += blockDim.x)
        reinterpret_cast<T*>(polys)[i] = reinterpret_cast<const T*>(a.polys)[i];
    __syncthreads();

    const unsigned lane = threadIdx.x & 31u;
    int4* st = stacks + (threadIdx.x >> 5) * a.stack_depth;
    // packet (32 sorted queries) and, in the subtree pass, the depth-k slot
    const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t packet = SPLIT == 2 ? gwarp / a.nslots : gwarp;
    const int slot = SPLIT == 2 ? int(gwarp % a.nslots) : 0;
    if (SPLIT == 2 && packet >= a.npackets) return;
    const int64_t i = packet * 32 + lane;
    const bool valid = i < a.Q;
    const int64_t qi = valid ? (a.perm ? a.perm[i] : i) : 0;
    VIS qv;
    qv.load(a, qi, valid);
    double* part = a.part + (SPLIT == 2 ? size_t(1 + slot) * 5 * a.Q : 0);
    unsigned mask = __ballot_sync(0xffffffffu, valid);
    if (mask == 0u) return;
    Acc<T> acc;
    acc.init();
    int64_t nleaf = 0, nfar = 0;
    uint64_t h = 0;
    unsigned long long nre = 0;
    int32_t cur, cur_link;
    int depth;
    if constexpr (SPLIT == 2) {
        mask &= a.items[packet * a.nslots + slot];
        cur = a.split_nodes[slot];
        depth = a.split_depth;
    } else {
        cur = 0;
        depth = 0;
    }
    memcpy(&cur_link, &a.box[cur].v[7], sizeof(int32_t));
    if (mask) {  // the start node (root, or the depth-k node) is popped alone
        const NodeT<T> b0 = a.box[cur];
        const bool d = ((mask >> lane) & 1u) &&
                       qv.template visit<HASH>(a, polys, b0, cur, a.lgcount[cur], acc, nleaf, nfar, h, nre);
        mask = __ballot_sync(0xffffffffu, d);
    }
    int sp = 0;
    while (mask) {
        const int32_t lid = cur + 1, rid = cur_link;
        if (SPLIT == 1 && depth + 1 == a.split_depth) {  // children start subtrees: hand over
            if (lane == 0) {
                unsigned* it = a.items + packet * a.nslots;
                it[a.slot_of[lid]] = mask;
                it[a.slot_of[rid]] = mask;
            }
            __syncwarp();
            if (sp > 0) {
                --sp;
                const int4 e = st[sp];
                cur = e.x;
                cur_link = e.y;
                mask = unsigned(e.z);
                depth = e.w;
            } else {
                mask = 0u;
            }
            continue;
        }
        const PairT<T>& pr = a.pairs[cur];  // warp-uniform: broadcast loads
        const NodeT<T> bl = pr.l, br = pr.r;
        const T lgl = pr.lgc[0], lgr = pr.lgc[1];
        // the most likely next step descends into the left child: pull its
        // pair record into L1 while this one is being processed
        if (lane == 0) asm volatile("prefetch.global.L1 [%0];" ::"l"(a.pairs + lid));
        bool dl = false, dr = false;
        if ((mask >> lane) & 1u) {
            dl = qv.template visit<HASH>(a, polys, bl, lid, lgl, acc, nleaf, nfar, h, nre);
            dr = qv.template visit<HASH>(a, polys, br, rid, lgr, acc, nleaf, nfar, h, nre);
        }
        const unsigned DL = __ballot_sync(0xffffffffu, dl), DR = __ballot_sync(0xffffffffu, dr);
        int32_t llink, rlink;
        memcpy(&llink, &bl.v[7], sizeof(int32_t));
        memcpy(&rlink, &br.v[7], sizeof(int32_t));
        if (DL) {
            if (DR) {
                if (lane == 0) st[sp] = make_int4(rid, rlink, int(DR), depth + 1);
                __syncwarp();
                ++sp;
            }
            cur = lid;
            cur_link = llink;
            mask = DL;
            ++depth;
        } else if (DR) {
            cur = rid;
            cur_link = rlink;
            mask = DR;
            ++depth;
        } else if (sp > 0) {
            --sp;
            const int4 e = st[sp];
            cur = e.x;
            cur_link = e.y;
            mask = unsigned(e.z);
            depth = e.w;
        } else {
            mask = 0u;
        }
    }
    if (!valid) return;
    Tot tot;
    tot.init();
    tot.flush(acc);
    part[i] = tot.M;
    part[a.Q + i] = tot.s;
    part[2 * a.Q + i] = tot.gx;
    part[3 * a.Q + i] = tot.gy;
    part[4 * a.Q + i] = tot.gz;
    if constexpr (SPLIT == 2) {  // the top pass stored its counts first
        if (nleaf) atomicAdd(reinterpret_cast<unsigned long long*>(a.leaves + i), (unsigned long long)nleaf);
        if (nfar) atomicAdd(reinterpret_cast<unsigned long long*>(a.far + i), (unsigned long long)nfar);
        if (HASH && h) atomicAdd(reinterpret_cast<unsigned long long*>(a.hash + i), (unsigned long long)h);
    } else {
        a.leaves[i] = nleaf;
        a.far[i] = nfar;
        if (HASH) a.hash[i] = h;
    }
    if (nre) atomicAdd(a.rechecks, nre);
}

// Launches K3 (SPLIT 0, or the split pair 1 + 2) for VIS over the tree t
// and returns the number of fp64 partial slots written to a.part (merged by
// K4). a.part must hold 5 Q doubles; it is re-pointed when splitting.
template <class T, class VIS>
int launch_pair_traversal(Ctx& c, DeviceTree& t, TraverseArgs<T>& a, bool hash, cudaStream_t st, int64_t& launches) {
    const int64_t Q = a.Q;
    const size_t smem = poly_bytes<T>(a.npoly) + size_t(a.stack_depth) * (kTravThreads / 32) * sizeof(int4);
    // few queries: split the walk at depth k so that packets x 2^k warps fill
    // the GPU (>= ~32 warps per SM)
    const int64_t npackets = (Q + 31) / 32;
    // SDGPU_SPLIT = 0 disables, = k forces depth k (A/B runs and tests)
    const char* se = std::getenv("SDGPU_SPLIT");
    const int forced = se && *se ? std::atoi(se) : -1;
    int k = 0;
    if (t.depth >= 2) {
        const int kmax = std::min(12, t.depth - 1);
        if (forced >= 0) {
            k = std::min(forced, kmax);
        } else if (t.depth >= 3) {
            while (k < std::min(10, kmax) && npackets * (int64_t(1) << k) < 148 * 32) ++k;
        }
        while (k > 0 && size_t(1 + (size_t(1) << k)) * 5 * size_t(Q) * sizeof(double) > (size_t(1) << 31)) --k;
    }
    a.split_depth = k;
    a.npackets = npackets;
    a.nslots = 1;
    int nsplits = 1;
    if (k > 0) {
        split_tables(c, t, k);
        a.nslots = int(t.split_count);
        a.slot_of = t.slot_of.as<int32_t>();
        a.split_nodes = t.split_nodes.as<int32_t>();
        a.items = static_cast<unsigned*>(c.tmp2.ensure(size_t(npackets) * a.nslots * sizeof(unsigned)));
        check_cuda(cudaMemsetAsync(a.items, 0, size_t(npackets) * a.nslots * sizeof(unsigned), st), "memset");
        nsplits = 1 + a.nslots;
        a.part = static_cast<double*>(c.part.ensure(size_t(nsplits) * 5 * Q * sizeof(double)));
    }
    // the decision hash costs ~20 integer ops per decision: only when asked for
    auto pick = [&](auto split) {
        constexpr int S = decltype(split)::value;
        return hash ? pair_kernel<T, VIS, true, S> : pair_kernel<T, VIS, false, S>;
    };
    auto kern = k > 0 ? pick(std::integral_constant<int, 1>()) : pick(std::integral_constant<int, 0>());
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
    kern<<<unsigned((Q + kTravThreads - 1) / kTravThreads), kTravThreads, smem, st>>>(a);
    check_cuda(cudaGetLastError(), "traverse kernel");
    ++launches;
    if (k > 0) {
        auto sub = pick(std::integral_constant<int, 2>());
        check_cuda(cudaFuncSetAttribute(sub, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
        const int64_t warps = npackets * a.nslots;
        sub<<<unsigned((warps * 32 + kTravThreads - 1) / kTravThreads), kTravThreads, smem, st>>>(a);
        check_cuda(cudaGetLastError(), "subtree kernel");
        ++launches;
    }
    return nsplits;
}

}  // namespace sdgpu
