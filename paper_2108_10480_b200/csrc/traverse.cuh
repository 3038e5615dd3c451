// traverse.cuh -- K3, the warp-coherent child-pair BVH traversal shared by
// the point-query path (bvh.cu) and the simplex-query path (simplex.cu):
// traversal record layouts, kernel arguments, the far-field term, the
// kernel template (parameterised by the per-lane query type) and its host
// launcher with the few-query split mode.
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <type_traits>

#include "context.h"

namespace sdgpu {

template <class T>
struct alignas(16) NodeT {  // 2 x (4 T): (lo, diam) (hi, link)
    T v[8];
};
// Both children of an internal node + their log2 n_B, component-
// interleaved (w[2k] = left.v[k], w[2k + 1] = right.v[k]) so that the fp32
// walk tests both children with packed fp32x2 arithmetic straight from the
// loaded registers.
template <class T>
struct alignas(16) PairT {
    T w[16];
    T lgc[4];
    __host__ __device__ __forceinline__ NodeT<T> l() const {
        NodeT<T> n;
#pragma unroll
        for (int k = 0; k < 8; ++k) n.v[k] = w[2 * k];
        return n;
    }
    __host__ __device__ __forceinline__ NodeT<T> r() const {
        NodeT<T> n;
#pragma unroll
        for (int k = 0; k < 8; ++k) n.v[k] = w[2 * k + 1];
        return n;
    }
    __host__ __device__ __forceinline__ void set(const NodeT<T>& L, const NodeT<T>& R) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            w[2 * k] = L.v[k];
            w[2 * k + 1] = R.v[k];
        }
    }
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
    const int2* split_meta;     // slot -> (node, path length | first-slot bits << 8)
    const int32_t* split_path;  // [slot][split_depth] ancestors, root first
    // simplex queries (simplex.cu): fp64 corners and dims per query, and
    // the fp64 leaf geometry (16 doubles per leaf slot)
    const double* qgeom;
    const int32_t* qdim;
    const double* leafgeom;
    // query sharding (sd_query_points_device_shard): this rank walks its
    // chunks of pk_chunk packets of the sorted batch (shard_packet)
    int64_t pk_world = 1, pk_rank = 0, pk_chunk = 1;
    // K3Q leaf-queue capacity (entries per lane); leaf_coop: the queued
    // terms are evaluated by the whole warp (leaf_flush_coop) instead of
    // one per lane per round
    int lq_cap = 0;
    int leaf_coop = 0;
};

constexpr int kTravThreads = 128;
// K3Q launch bounds; A/B builds (tools/build_ab.sh): EXTRA=-DSD_TRAV_MINB=k
// (CTA floor) or -DSD_TRAV_MAXNREG=n. Measured (cfg4): both caps at 56
// registers run ~4 % slower than the unconstrained build, which lands on
// 56 by itself -- and any code added to the walk's loop takes it to 64+.
#ifdef SD_TRAV_MINB
#define SD_TRAV_BOUNDS __launch_bounds__(kTravThreads, SD_TRAV_MINB)
#elif defined(SD_TRAV_MAXNREG)
#define SD_TRAV_BOUNDS __maxnreg__(SD_TRAV_MAXNREG)
#else
#define SD_TRAV_BOUNDS __launch_bounds__(kTravThreads)
#endif

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
// the right child, else pops. Stack entries (node, its link, mask)
// live in shared memory, one stack per warp.
//
// SPLIT = 1 (few queries): one warp per (query packet, slot), the slots
// being the nodes at tree depth k plus the leaves above that depth, so that
// every root-to-leaf path crosses exactly one slot. The warp first re-tests
// the slot's ancestors (root first) for its lanes: a lane for which an
// ancestor is admissible does not reach the slot, and that ancestor's
// far-field term is emitted only by the warp of the first slot below it.
// The lanes that reach the slot then walk its subtree as above. Per lane the
// decisions and terms are exactly the unsplit walk's; the partial sums land
// in one fp64 state per slot, merged by K4, so a batch of a few hundred
// queries still spreads over thousands of warps.
//
// VIS is the per-lane query: load(a, qi, valid) reads it, visit<HASH>(...)
// tests one node for it (point queries: bvh.cu; simplex queries:
// simplex.cu) and returns "descend"; far_test<HASH>(...) is the
// admissibility test alone (emitting the far-field term only when asked).
__device__ __forceinline__ void st_shared_int4(uint32_t addr, int x, int y, int z) {
    asm volatile("st.shared.v4.s32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(0) : "memory");
}
__device__ __forceinline__ int4 ld_shared_int4(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}

template <class T, class VIS, bool HASH, int SPLIT>
__device__ __forceinline__ void pair_walk(const TraverseArgs<T>& a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<T>* polys = reinterpret_cast<Poly<T>*>(smem_raw);
    int4* stacks = reinterpret_cast<int4*>(smem_raw + poly_bytes<T>(a.npoly));
    for (int i = threadIdx.x; i < a.npoly * kPolyCoefs; i += blockDim.x)
        reinterpret_cast<T*>(polys)[i] = reinterpret_cast<const T*>(a.polys)[i];
    __syncthreads();

    const unsigned lane = threadIdx.x & 31u;
    const unsigned lanebit = 1u << lane;
    int4* st = stacks + (threadIdx.x >> 5) * a.stack_depth;
    // packet (32 sorted queries) and, when split, the slot
    const int64_t gwarp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t packet = SPLIT ? gwarp / a.nslots : shard_packet(gwarp, a.pk_world, a.pk_rank, a.pk_chunk);
    const int slot = SPLIT ? int(gwarp % a.nslots) : 0;
    if (SPLIT && packet >= a.npackets) return;
    const int64_t i = packet * 32 + lane;
    const bool valid = i < a.Q;
    const int64_t qi = valid ? (a.perm ? a.perm[i] : i) : 0;
    VIS qv;
    qv.load(a, qi, valid);
    double* part = a.part + (SPLIT ? size_t(slot) * 5 * a.Q : 0);
    unsigned mask = __ballot_sync(0xffffffffu, valid);
    if (mask == 0u) return;
    Acc<T> acc;
    acc.init();
    int32_t nleaf = 0, nfar = 0;  // per query: < 2^31 nodes
    uint64_t h = 0;
    unsigned long long nre = 0;
    int32_t cur = 0, cur_link;
    if constexpr (SPLIT) {
        const int2 sm = a.split_meta[slot];  // (node, path length | first-slot bits << 8)
        cur = sm.x;
        const int len = sm.y & 0xff;
        const unsigned first = unsigned(sm.y) >> 8;
        const int32_t* path = a.split_path + size_t(slot) * a.split_depth;
        for (int j = 0; j < len && mask; ++j) {
            const int32_t anc = path[j];
            const NodeT<T> b = a.box[anc];
            bool far = false;
            if ((mask >> lane) & 1u)
                far = qv.template far_test<HASH>(a, b, anc, a.lgcount[anc], ((first >> j) & 1u) != 0u, acc, nfar, h,
                                                 nre);
            mask &= ~__ballot_sync(0xffffffffu, far);
        }
    }
    memcpy(&cur_link, &a.box[cur].v[7], sizeof(int32_t));
    if (mask) {  // the start node (root, or the slot) is popped alone
        const NodeT<T> b0 = a.box[cur];
        const bool d = ((mask >> lane) & 1u) &&
                       qv.template visit<HASH>(a, polys, b0, cur, a.lgcount[cur], acc, nleaf, nfar, h, nre);
        mask = __ballot_sync(0xffffffffu, d);
    }
    // stack top as a shared-window byte address (one add per push / pop)
    const uint32_t st0 = smem_u32(st);
    uint32_t top = st0;
    while (mask) {
        const int32_t lid = cur + 1, rid = cur_link;
        const PairT<T>& pr = a.pairs[uint32_t(cur)];  // warp-uniform: broadcast loads
        const NodeT<T> bl = pr.l(), br = pr.r();
        const T lgl = pr.lgc[0], lgr = pr.lgc[1];
        // the most likely next step descends into the left child: pull its
        // pair record into L1 while this one is being processed
        asm volatile("prefetch.global.L1 [%0];" ::"l"(&pr + 1));  // = a.pairs + lid (one request per warp)
        bool dl = false, dr = false;
        if (mask & lanebit) qv.template visit_pair<HASH>(a, polys, bl, br, lid, rid, lgl, lgr, acc, nleaf, nfar, h, nre, dl, dr);
        const unsigned DL = __ballot_sync(0xffffffffu, dl), DR = __ballot_sync(0xffffffffu, dr);
        int32_t llink, rlink;
        memcpy(&llink, &bl.v[7], sizeof(int32_t));
        memcpy(&rlink, &br.v[7], sizeof(int32_t));
        if (DL) {
            if (DR) {
                if (lane == 0) st_shared_int4(top, rid, rlink, int(DR));
                __syncwarp();
                top += 16;
            }
            cur = lid;
            cur_link = llink;
            mask = DL;
        } else if (DR) {
            cur = rid;
            cur_link = rlink;
            mask = DR;
        } else if (top != st0) {
            top -= 16;
            const int4 e = ld_shared_int4(top);
            cur = e.x;
            cur_link = e.y;
            mask = unsigned(e.z);
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
    if constexpr (SPLIT != 0) {  // counters were zeroed; the slots add
        if (nleaf) atomicAdd(reinterpret_cast<unsigned long long*>(a.leaves + i), (unsigned long long)nleaf);
        if (nfar) atomicAdd(reinterpret_cast<unsigned long long*>(a.far + i), (unsigned long long)nfar);
        if (HASH && h) atomicAdd(reinterpret_cast<unsigned long long*>(a.hash + i), (unsigned long long)h);
    } else {
        a.leaves[i] = nleaf;
        a.far[i] = nfar;
        if (HASH) a.hash[i] = h;
    }
    // (the fp64 re-decision count nre is not reported by the packet walk)
}

template <class T, class VIS, bool HASH, int SPLIT>
__global__ void __launch_bounds__(kTravThreads) pair_kernel(const __grid_constant__ TraverseArgs<T> a) {
    pair_walk<T, VIS, HASH, SPLIT>(a);
}

// K3Q (default for dense point batches): the child-pair packet walk with
// per-lane DEFERRED EXACT LEAVES. Inline, a leaf child costs the warp the
// ~190-instruction triangle term for the ~3 lanes that reach it. Here a lane
// that reaches an exact leaf counts and hashes it at once (the decision is
// the reference's, made where the reference makes it) but only appends the
// leaf slot to its own shared-memory queue (kLeafQ entries per lane, lane-
// interleaved: entry k of a lane at [k][lane], conflict-free); the terms
// are evaluated in ROUNDS in which every lane with a pending entry pops one
// and adds its own term to its own accumulator -- no shuffles, each lane's
// query and shift stay in registers. A round runs when some lane's queue
// could overflow on the next step (>= kLeafQ - 1 pending; a step adds at
// most two) and the queues are drained after the walk. Per lane the set of
// terms is exactly collect_contributions'; only their summation order
// changes (fp32 rounding).
constexpr int kLeafQ = 40;      // default leaf queue entries per lane (SDGPU_LEAFQ), per-lane rounds
constexpr int kLeafQCoop = 24;  // the same with the warp-cooperative flush (fp32 default)

// Counter type of walks whose per-query counters were not asked for.
struct NoCount {
    __device__ __forceinline__ NoCount& operator++() { return *this; }
};
constexpr uint32_t kLeafStride = kTravThreads * 4;  // bytes between a lane's leaf entries


template <class T, class VIS, bool HASH, bool COUNT, bool COOP>
__device__ __forceinline__ void pair_walk_q(const TraverseArgs<T>& a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<T>* polys = reinterpret_cast<Poly<T>*>(smem_raw);
    int4* stacks = reinterpret_cast<int4*>(smem_raw + poly_bytes<T>(a.npoly));
    int32_t* lqs = reinterpret_cast<int32_t*>(stacks + (kTravThreads / 32) * a.stack_depth);
    for (int i = threadIdx.x; i < a.npoly * kPolyCoefs; i += blockDim.x)
        reinterpret_cast<T*>(polys)[i] = reinterpret_cast<const T*>(a.polys)[i];
    __syncthreads();

    constexpr unsigned FULL = 0xffffffffu;
    const unsigned lane = threadIdx.x & 31u;
    const unsigned lanebit = 1u << lane;
    const unsigned warp = threadIdx.x >> 5;
    int4* st = stacks + warp * a.stack_depth;
    const uint32_t lq0 = smem_u32(lqs + threadIdx.x);  // this lane's entry 0 (entries kLeafStride apart)
    const uint32_t lqw = smem_u32(lqs + (threadIdx.x & ~31u));  // the warp's lane 0
    const int lcap = a.lq_cap - 1;  // a step appends at most two entries per lane
    int nq = 0;  // pending leaf entries of this lane
    const int64_t packet =
        shard_packet((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, a.pk_world, a.pk_rank, a.pk_chunk);
    const int64_t i = packet * 32 + lane;
    const bool valid = i < a.Q;
    const int64_t qi = valid ? (a.perm ? a.perm[i] : i) : 0;
    VIS qv;
    qv.load(a, qi, valid);
    unsigned mask = __ballot_sync(FULL, valid);
    if (mask == 0u) return;
    Acc<T> acc;
    acc.init();
    using CNT = std::conditional_t<COUNT, int32_t, NoCount>;  // per query: < 2^31 nodes
    CNT nleaf{}, nfar{};
    uint64_t h = 0;
    unsigned long long nre = 0;
    int32_t cur = 0, cur_link;
    memcpy(&cur_link, &a.box[0].v[7], sizeof(int32_t));
    {  // the root is popped alone
        const NodeT<T> b0 = a.box[0];
        const bool d = valid && qv.template visit_q<HASH>(a, b0, 0, a.lgcount[0], acc, nleaf, nfar, h, nre, lq0, nq);
        mask = __ballot_sync(FULL, d);
    }
    if constexpr (VIS::template kFrame<T>) acc.m -= a.lw_ff;  // see PointVisit (-inf stays -inf)
    auto round = [&]() {
        if (nq > 0) {
            --nq;
            int slot;
            asm volatile("ld.shared.s32 %0, [%1];" : "=r"(slot) : "r"(lq0 + uint32_t(nq) * kLeafStride));
            qv.leaf_round(a, polys, slot, acc);
        }
    };
    const uint32_t st0 = smem_u32(st);
    uint32_t top = st0;
    while (mask) {
        const int32_t lid = cur + 1, rid = cur_link;
        const PairT<T>& pr = a.pairs[uint32_t(cur)];  // warp-uniform: broadcast loads
        asm volatile("prefetch.global.L1 [%0];" ::"l"(&pr + 1));  // = a.pairs + lid
        bool dl = false, dr = false;
        int32_t llink, rlink;
        qv.template visit_pair_q<HASH>(a, pr, lid, rid, (mask & lanebit) != 0u, acc, nleaf, nfar, h, nre, lq0, nq, dl,
                                       dr, llink, rlink);
        const unsigned DL = __ballot_sync(FULL, dl), DR = __ballot_sync(FULL, dr);
        // (one convergence point per step: the queue check with the ballots)
        const bool full = __any_sync(FULL, nq >= lcap);
        if (DL) {
            if (DR) {
                // every lane stores the same entry (one same-address write):
                // each lane later reads back its own store, no warp barrier
                st_shared_int4(top, rid, rlink, int(DR));
                top += 16;
            }
            cur = lid;
            cur_link = llink;
            mask = DL;
        } else if (DR) {
            cur = rid;
            cur_link = rlink;
            mask = DR;
        } else if (top != st0) {
            top -= 16;
            const int4 e = ld_shared_int4(top);
            cur = e.x;
            cur_link = e.y;
            mask = unsigned(e.z);
        } else {
            mask = 0u;
        }
        if (full) {
            if constexpr (COOP) qv.leaf_flush_coop(a, polys, acc, lqw, nq, lane);
            else
                while (__any_sync(FULL, nq >= lcap)) round();
        }
    }
    if constexpr (COOP) qv.leaf_flush_coop(a, polys, acc, lqw, nq, lane);
    else
        while (__any_sync(FULL, nq > 0)) round();
    if (!valid) return;
    if constexpr (VIS::template kFrame<T>) acc.m += a.lw_ff;
    Tot tot;
    tot.init();
    tot.flush(acc);
    a.part[i] = tot.M;
    a.part[a.Q + i] = tot.s;
    a.part[2 * a.Q + i] = tot.gx;
    a.part[3 * a.Q + i] = tot.gy;
    a.part[4 * a.Q + i] = tot.gz;
    if constexpr (COUNT) {
        a.leaves[i] = nleaf;
        a.far[i] = nfar;
    }
    if (HASH) a.hash[i] = h;
}

template <class T, class VIS, bool HASH, bool COUNT, bool COOP = false>
__global__ void SD_TRAV_BOUNDS pair_kernel_q(const __grid_constant__ TraverseArgs<T> a) {
    pair_walk_q<T, VIS, HASH, COUNT || HASH, COOP>(a);
}

// K3F (few queries, node-parallel): a group of G lanes per query (32 / G
// queries per warp); the lanes of a group test up to G nodes of their
// query's walk at once. A group pops the top G (or fewer) entries of its
// shared-memory stack, every lane tests its node exactly like the serial
// walk would (far field / exact leaf / descend), and the children of
// descending nodes are pushed (ballot + prefix count within the group). A
// node is tested iff all its ancestors descended -- the reference's visited
// set -- only the order of the terms differs. Each lane keeps its own
// accumulator; the G states of a query are merged in fp64 at the end. (The
// walk of one query is a narrow frontier -- ~4 live nodes near a surface --
// so G = 4..8 keeps most lanes busy; G = 32 is one query per warp.)
// Stack bound: the entries stay sorted by depth (children of the popped top
// entries are deeper than everything left below them), and entries of depth
// d are only created while depth-(d-1) entries on top are popped -- in the
// same batch as every depth-d entry above them -- so each level holds at
// most 2 G entries and 2 G (depth + 1) always suffice. The guard below can
// therefore not fire; it records a flag instead of writing past the stack.
template <class T, class VIS, bool HASH, int G>
__global__ void __launch_bounds__(kTravThreads) frontier_kernel(const __grid_constant__ TraverseArgs<T> a, int cap,
                                                                int* overflow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<T>* polys = reinterpret_cast<Poly<T>*>(smem_raw);
    int32_t* stacks = reinterpret_cast<int32_t*>(smem_raw + poly_bytes<T>(a.npoly));
    for (int i = threadIdx.x; i < a.npoly * kPolyCoefs; i += blockDim.x)
        reinterpret_cast<T*>(polys)[i] = reinterpret_cast<const T*>(a.polys)[i];
    __syncthreads();
    const unsigned lane = threadIdx.x & 31u;
    const unsigned grp = lane / G, r = lane % G;
    const unsigned gshift = grp * G;
    constexpr unsigned gmask = G == 32 ? 0xffffffffu : ((1u << G) - 1u);
    const int64_t i = ((int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5) * (32 / G) + grp;  // sorted position
    const bool valid = i < a.Q;
    int32_t* stk = stacks + size_t(threadIdx.x / G) * cap;
    const int64_t qi = valid ? (a.perm ? a.perm[i] : i) : 0;
    VIS qv;
    qv.load(a, qi, valid);
    Acc<T> acc;
    acc.init();
    int64_t nleaf = 0, nfar = 0;  // (64-bit here: measured faster in this kernel)
    uint64_t h = 0;
    unsigned long long nre = 0;
    if (r == 0) stk[0] = 0;
    __syncwarp();
    int n = valid ? 1 : 0;
    while (__any_sync(0xffffffffu, n > 0)) {
        const int take = n < G ? n : G;
        const int base = n - take;
        const int32_t id = int(r) < take ? stk[base + r] : -1;
        __syncwarp();
        bool d = false;
        if (id >= 0) {
            const NodeT<T> b = a.box[id];
            d = qv.template visit<HASH>(a, polys, b, id, a.lgcount[id], acc, nleaf, nfar, h, nre);
        }
        const unsigned D = (__ballot_sync(0xffffffffu, d) >> gshift) & gmask;
        const int pushed = 2 * __popc(D);
        if (base + pushed > cap) {  // unreachable (see above)
            if (r == 0) atomicExch(overflow, 1);
            n = 0;
            continue;
        }
        if (d) {
            const int pos = base + 2 * __popc(D & ((1u << r) - 1u));
            int32_t link;
            memcpy(&link, &a.box[id].v[7], sizeof(int32_t));
            stk[pos] = link;        // right child below ...
            stk[pos + 1] = id + 1;  // ... left child on top
        }
        __syncwarp();
        n = base + pushed;
    }
    // merge the group's states (fp64, anchored at the group maximum)
    Tot tot;
    tot.init();
    tot.flush(acc);
    double M = tot.M;
#pragma unroll
    for (int off = G / 2; off; off >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, off));
    const double f = (M == -INFINITY || tot.M == -INFINITY) ? 0.0 : exp2(tot.M - M);
    double s = tot.s * f, gx = tot.gx * f, gy = tot.gy * f, gz = tot.gz * f;
    unsigned long long L = (unsigned long long)nleaf, F = (unsigned long long)nfar, H = h;
#pragma unroll
    for (int off = G / 2; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        gx += __shfl_xor_sync(0xffffffffu, gx, off);
        gy += __shfl_xor_sync(0xffffffffu, gy, off);
        gz += __shfl_xor_sync(0xffffffffu, gz, off);
        L += __shfl_xor_sync(0xffffffffu, L, off);
        F += __shfl_xor_sync(0xffffffffu, F, off);
        H += __shfl_xor_sync(0xffffffffu, H, off);
    }
    if (r == 0 && valid) {
        a.part[i] = M;
        a.part[a.Q + i] = s;
        a.part[2 * a.Q + i] = gx;
        a.part[3 * a.Q + i] = gy;
        a.part[4 * a.Q + i] = gz;
        a.leaves[i] = int64_t(L);
        a.far[i] = int64_t(F);
        if (HASH) a.hash[i] = H;
    }
    if (nre) atomicAdd(a.rechecks, nre);
}

// K3F launcher with group width G (SDGPU_FRONTIER_G overrides): returns
// false (nothing launched) when the stacks would not fit in shared memory.
template <class T, class VIS>
bool launch_frontier(Ctx& c, DeviceTree& t, TraverseArgs<T>& a, bool hash, cudaStream_t st, int64_t& launches,
                     int G = 4) {
    const char* e = std::getenv("SDGPU_FRONTIER_G");
    if (e && *e) G = std::atoi(e);
    if (G != 4 && G != 8 && G != 16 && G != 32) G = 4;
    const int cap = 2 * G * (t.depth + 1);
    const size_t smem = poly_bytes<T>(a.npoly) + size_t(cap) * (kTravThreads / G) * sizeof(int32_t);
    if (smem > 200 * 1024) return false;
    int* flag = static_cast<int*>(c.flag.ensure(sizeof(int)));
    using K = void (*)(TraverseArgs<T>, int, int*);
    K kern;
    switch (G) {
        case 8: kern = hash ? frontier_kernel<T, VIS, true, 8> : frontier_kernel<T, VIS, false, 8>; break;
        case 16: kern = hash ? frontier_kernel<T, VIS, true, 16> : frontier_kernel<T, VIS, false, 16>; break;
        case 32: kern = hash ? frontier_kernel<T, VIS, true, 32> : frontier_kernel<T, VIS, false, 32>; break;
        default: kern = hash ? frontier_kernel<T, VIS, true, 4> : frontier_kernel<T, VIS, false, 4>; break;
    }
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
    const int64_t threads = (a.Q + 32 / G - 1) / (32 / G) * 32;
    kern<<<unsigned((threads + kTravThreads - 1) / kTravThreads), kTravThreads, smem, st>>>(a, cap, flag);
    check_cuda(cudaGetLastError(), "frontier kernel");
    ++launches;
    return true;
}

// Few-query mode choice: SDGPU_FRONTIER = 1 / 0 forces it on / off;
// default: node-parallel when the batch has at most `limit` queries.
inline bool use_frontier(int64_t Q, int64_t limit) {
    const char* e = std::getenv("SDGPU_FRONTIER");
    if (e && *e) return std::atoi(e) != 0;
    return Q <= limit;
}

// Split depth of launch_pair_traversal (0: unsplit). SDGPU_SPLIT = 0
// disables, = k forces depth k (A/B runs and tests).
template <class T>
int pair_split_depth(const DeviceTree& t, const TraverseArgs<T>& a, int weight = 1) {
    const int64_t npackets = (a.Q + 31) / 32;
    const char* se = std::getenv("SDGPU_SPLIT");
    const int forced = se && *se ? std::atoi(se) : -1;
    int k = 0;
    if (t.depth >= 2 && a.pk_world <= 1) {  // (sharded walks never split)
        const int kmax = std::min(14, t.depth);
        if (forced >= 0) {
            k = std::min(forced, kmax);
        } else {  // >= ~32 (x weight) warps per SM
            while (k < kmax && npackets * (int64_t(1) << k) < int64_t(148) * 32 * weight) ++k;
        }
        while (k > 0 && (size_t(1) << k) * 5 * size_t(a.Q) * sizeof(double) > (size_t(1) << 31)) --k;
    }
    return k;
}

// Leaf-queue switches of K3Q: SDGPU_LEAF_QUEUE = 0 turns the deferred leaf
// queues off (A/B); SDGPU_LEAF_COOP = 1 / 0: queued leaf terms evaluated by
// the whole warp (leaf_flush_coop) / one per lane per round; default: the
// cooperative flush in fp32 (cfg4 21.9 -> 20.4 ms), per-lane rounds in fp64
// (52.5 vs 55.5 ms).
inline bool leaf_queue_on() {
    const char* e = std::getenv("SDGPU_LEAF_QUEUE");
    return !(e && *e == '0');
}
template <class T>
int leaf_coop_default() {
    const char* e = std::getenv("SDGPU_LEAF_COOP");
    return (e && *e) ? (*e == '1' ? 1 : 0) : (sizeof(T) == 4 ? 1 : 0);
}

// True when launch_pair_traversal (point queries, weight 1) will run K3Q
// with the cooperative leaf flush -- the walk whose near-contact face terms
// K3C corrects (bvh.cu).
template <class T>
bool will_use_coop_flush(const DeviceTree& t, const TraverseArgs<T>& a) {
    return leaf_queue_on() && leaf_coop_default<T>() == 1 && pair_split_depth(t, a, 1) == 0;
}

// Launches K3 (unsplit, or split at depth k for few queries) for VIS over
// the tree t and returns the number of fp64 partial slots written to a.part
// (merged by K4). a.part must hold 5 Q doubles; it is re-pointed when
// splitting. `weight` raises the warp target for expensive node tests.
template <class T, class VIS>
int launch_pair_traversal(Ctx& c, DeviceTree& t, TraverseArgs<T>& a, bool hash, cudaStream_t st, int64_t& launches,
                          int weight = 1, bool count = true) {
    const int64_t Q = a.Q;
    size_t smem = poly_bytes<T>(a.npoly) + size_t(a.stack_depth) * (kTravThreads / 32) * sizeof(int4);
    const int64_t npackets = (Q + 31) / 32;
    const int k = pair_split_depth(t, a, weight);
    a.split_depth = k;
    a.npackets = npackets;
    a.nslots = 1;
    int nsplits = 1;
    if (k > 0) {
        split_tables(c, t, k);
        a.nslots = int(t.split_count);
        a.split_meta = t.split_meta.as<int2>();
        a.split_path = t.split_path.as<int32_t>();
        check_cuda(cudaMemsetAsync(a.leaves, 0, size_t(Q) * sizeof(int64_t), st), "memset");
        check_cuda(cudaMemsetAsync(a.far, 0, size_t(Q) * sizeof(int64_t), st), "memset");
        if (hash) check_cuda(cudaMemsetAsync(a.hash, 0, size_t(Q) * sizeof(uint64_t), st), "memset");
        nsplits = a.nslots;
        a.part = static_cast<double*>(c.part.ensure(size_t(nsplits) * 5 * Q * sizeof(double)));
    }
    auto kern = k > 0 ? (hash ? pair_kernel<T, VIS, true, 1> : pair_kernel<T, VIS, false, 1>)
                      : (hash ? pair_kernel<T, VIS, true, 0> : pair_kernel<T, VIS, false, 0>);
    if constexpr (VIS::kLeafQueue) {  // leaf queues: see leaf_queue_on / leaf_coop_default
        // SDGPU_LEAFQ: leaf-queue entries per lane (>= 3)
        auto cap = [](const char* name, int dflt) {
            const char* e = std::getenv(name);
            return e && *e ? std::max(0, std::min(64, std::atoi(e))) : dflt;
        };
        const bool lq_on = leaf_queue_on();
        a.leaf_coop = leaf_coop_default<T>();
        a.lq_cap = std::max(3, cap("SDGPU_LEAFQ", a.leaf_coop ? kLeafQCoop : kLeafQ));
        if (lq_on && k == 0) {
            smem += size_t(a.lq_cap) * kTravThreads * sizeof(int32_t);
            if (a.leaf_coop)
                kern = hash ? pair_kernel_q<T, VIS, true, true, true>
                            : (count ? pair_kernel_q<T, VIS, false, true, true> : pair_kernel_q<T, VIS, false, false, true>);
            else
                kern = hash ? pair_kernel_q<T, VIS, true, true>
                            : (count ? pair_kernel_q<T, VIS, false, true> : pair_kernel_q<T, VIS, false, false>);
        }
    }
    check_cuda(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
    const int64_t warps =
        a.pk_world > 1 ? shard_count(npackets, a.pk_world, a.pk_rank, a.pk_chunk) : npackets * a.nslots;
    if (warps == 0) return nsplits;
    kern<<<unsigned((warps * 32 + kTravThreads - 1) / kTravThreads), kTravThreads, smem, st>>>(a);
    check_cuda(cudaGetLastError(), "traverse kernel");
    ++launches;
    return nsplits;
}

}  // namespace sdgpu
