// exact.cu -- K1: exact all-primitive smooth distance, the GPU replacement
// of smooth_min_dist_flat (smooth.hpp:189-198) for a whole query batch.
//
// Layout of work: CTAs tile the queries (kThreads threads x QPT queries per
// thread, queries in registers) and, when there are too few query tiles to
// fill 148 SMs, also split the primitive range ("splits"); each CTA streams
// its primitive range through shared memory with TMA bulk copies
// (cp.async.bulk + mbarrier, kStages-deep ring) and every thread evaluates
// each staged primitive against its queries -- all lanes read the same
// record, so shared-memory loads are broadcasts. Primitives are grouped by
// (kind, weight polynomial) into segments on the host; one launch per
// segment keeps the polynomial coefficients in kernel-parameter constant
// memory (FFMA constant-bank operands) and the kind branch out of the loop.
// Per-query state (Acc: shift m, sums s, g) is carried between segment
// launches in `part`; K4 (epilogue.cu) merges splits and finalises.
#include "exact.h"
#include "pair.cuh"
#include "pair2.cuh"

#include <cooperative_groups.h>
#include <type_traits>

namespace sdgpu {

template <class T>
struct ExactArgs {
    const T* rec;       // first record of this segment
    int64_t count;      // primitives in the segment
    int64_t chunk;      // primitives per split
    const T* q;         // Q x 3 query points
    int64_t Q;
    double* part;       // [splits][5][Q] partial state (m, s, gx, gy, gz), fp64
    int first;          // first segment: initialise instead of loading
    Phys<T> ph;
    Poly<T> poly;
    const int64_t* perm;  // sorted position -> query index
    const float4* tbox;   // tile boxes of the segment (null: no tile bounds)
    T lwmax, lwspan;      // log2 w upper bound and spread over the segment
    int cluster;          // splits merged over DSMEM into split 0's partial
    float prune;          // PRUNE kernels: negligibility threshold in bits
};

// Tot b folded into a (same anchor semantics as Tot::flush).
__device__ __forceinline__ void tot_merge(Tot& a, const Tot& b) {
    if (b.M == -INFINITY) return;
    if (a.M == -INFINITY) {
        a = b;
        return;
    }
    const double M = fmax(a.M, b.M);
    const double fa = exp2(a.M - M), fb = exp2(b.M - M);
    a.s = fma(a.s, fa, b.s * fb);
    a.gx = fma(a.gx, fa, b.gx * fb);
    a.gy = fma(a.gy, fa, b.gy * fb);
    a.gz = fma(a.gz, fa, b.gz * fb);
    a.M = M;
}

// Tile bounds (per warp, per staged tile; see exact_kernel): terms of a
// tile never exceed 2^H relative to the shift after the proactive raise,
// and tiles whose bound is too loose for the fp32 range (|kappa| diag +
// spread of log2 w > H + kLooseMargin: the tile's largest term could sit
// below 2^-100 of the shift, within 26 bits of fp32 flush) keep the
// per-term checks. H leaves room for the gradient products e r, r = 1/d:
// H = 96 while the query is at least 2^-20 from the tile's box (r <= 2^20:
// e r summed over a 768-term tile < 2^126), H = 64 closer (r up to 2^50,
// the rsqrt floor: < 2^124). (A single H = 100 overflowed the gradient of
// a query within ~4e-9 of a face to -inf; a single H = 64 made cfg2 tiles
// loose and cost 9 %.)
constexpr float kTileHeadroom = 96.0f;
constexpr float kTileHeadroomNear = 64.0f;
constexpr float kNearBox = 9.5367431640625e-07f;  // 2^-20
constexpr float kLooseMargin = 100.0f;

constexpr int kThreads = 256;
// Staged primitives per unrolled step of K1's inner loop: fp32 triangles
// 6 (cfg3, 131,072 queries: 122.5 ms at 2, 120.8 at 4, 119.9 at 6, 120.1
// at 8 -- more independent pair chains per warp at the same 80 registers),
// fp64 6 (cfg1 points 0.876 -> 0.827 ms, cfg2 edges 31.45 -> 30.49 ms;
// 8: 0.822 / 30.60, 12: 0.838 / 32.41), fp32 edges 8 with 2 queries per
// thread (cfg2: 6.96 ms at 4 queries x 2 primitives; 2 queries x 2 / 3 /
// 4 / 5 / 8 primitives: 6.82 / 6.92 / 6.80 / 6.89 / 6.79 ms), fp32 points
// 2. A/B builds: EXTRA=-DSD_K1_UNROLL=k forces k for every kind,
// -DSD_K1_UNROLL64=k for fp64, -DSD_K1_UNROLL_EDGE / -DSD_K1_QPT_EDGE.
template <class T, int KIND>
constexpr int unroll_prims() {
#ifdef SD_K1_UNROLL
    return SD_K1_UNROLL;
#elif defined(SD_K1_UNROLL_EDGE)
    return sizeof(T) == 4 && KIND == 1 ? SD_K1_UNROLL_EDGE : ((sizeof(T) == 4 && KIND == 2) || sizeof(T) == 8 ? 6 : 2);
#elif defined(SD_K1_UNROLL64)
    return sizeof(T) == 4 && KIND == 2 ? 6 : (sizeof(T) == 8 ? SD_K1_UNROLL64 : 2);
#else
    return sizeof(T) == 4 && KIND == 1 ? 8 : ((sizeof(T) == 4 && KIND == 2) || sizeof(T) == 8 ? 6 : 2);
#endif
}
#ifndef SD_K1_STAGES  // A/B builds (tools/build_ab.sh): EXTRA=-DSD_K1_STAGES=n -DSD_K1_MINB=k
#define SD_K1_STAGES 3
#endif
constexpr int kStages = SD_K1_STAGES;

template <class T, int KIND>
constexpr int tile_prims() {
    // 6-12 KB (fp32) / 12-24 KB (fp64) per stage, so that 3 stages plus the
    // fp64 per-query totals leave room for 3 resident CTAs per SM
    return KIND == 0 ? 512 : 128;
}

// PRUNE (sd_set_exact_pruning, off by default): the positive terms of the
// sum let any single term bound it from below, so before the tile loop each
// query takes, over the tile boxes of the whole segment, the largest
// kappa d_hi + min log2 w -- a lower bound of log2 of its largest term and
// hence of log2 c. A tile whose upper bound kappa d_lo + max log2 w lies
// more than `prune` bits below that bound for every query of the warp is
// skipped: each dropped term is < 2^-prune c, N of them < N 2^-prune c
// (2^-30 relative at 48 bits and 2^18 primitives, far inside the fp32
// path's own rounding). Not the reference's sum term for term, so it is a
// separate kernel instance behind its own switch.
template <class T, int KIND, bool POLY, bool SAFE, int QPT, int MINB, bool PRUNE = false>
__global__ void __launch_bounds__(kThreads, MINB) exact_kernel(const __grid_constant__ ExactArgs<T> a) {
    constexpr int R = rec_size(KIND);
    constexpr int TILE = tile_prims<T, KIND>();
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* tiles = reinterpret_cast<T*>(smem_raw);
    // fp64 per-query totals live in shared memory (touched once per tile)
    Tot* tot = reinterpret_cast<Tot*>(smem_raw + size_t(kStages) * TILE * R * sizeof(T));
    __shared__ uint64_t full[kStages];

    const int split = blockIdx.y;
    const int64_t p0 = int64_t(split) * a.chunk;
    const int64_t p1 = min(a.count, p0 + a.chunk);
    const int64_t np = max(int64_t(0), p1 - p0);
    const int ntiles = int((np + TILE - 1) / TILE);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    // PRUNE: the split's tiles are visited from the tile nearest the CTA's
    // first query (t0, wrapping around), so the running totals bound the
    // sums tightly from the first tiles on
    [[maybe_unused]] __shared__ int t0s;
    int t0 = 0;
    auto tile_of = [&](int t) { return PRUNE ? (t0 + t < ntiles ? t0 + t : t0 + t - ntiles) : t; };
    auto issue = [&](int t) {
        const int s = t % kStages;
        const int64_t b = p0 + int64_t(tile_of(t)) * TILE;
        const int n = int(min(int64_t(TILE), p1 - b));
        const uint32_t bytes = uint32_t(n) * R * sizeof(T);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(tiles + size_t(s) * TILE * R, a.rec + b * R, bytes, &full[s]);
    };
    if constexpr (!PRUNE) {
        if (threadIdx.x == 0)
            for (int t = 0; t < kStages && t < ntiles; ++t) issue(t);
    }

    // queries of this thread
    T qx[QPT], qy[QPT], qz[QPT];
    Acc<T> acc[QPT];
    int64_t qi[QPT];
    double* part = a.part + size_t(split) * 5 * a.Q;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
        // a warp owns 32 x QPT consecutive (Morton-sorted) queries
        qi[k] = int64_t(blockIdx.x) * kThreads * QPT + int64_t(warp) * 32 * QPT + k * 32 + lane;
        const int64_t qc = min(qi[k], a.Q - 1);
        const int64_t qo = a.perm ? a.perm[qc] : qc;
        qx[k] = a.q[3 * qo];
        qy[k] = a.q[3 * qo + 1];
        qz[k] = a.q[3 * qo + 2];
        acc[k].init();
        Tot& tk = tot[k * kThreads + threadIdx.x];
        tk.init();
        if (!a.first && (!a.cluster || split == 0)) {  // clusters: the merged state lives in split 0
            tk.M = part[qc];
            tk.s = part[a.Q + qc];
            tk.gx = part[2 * a.Q + qc];
            tk.gy = part[3 * a.Q + qc];
            tk.gz = part[4 * a.Q + qc];
            acc[k].m = T(tk.M);
        }
        // unit-weight launches keep the shift relative to log2 w = S log2 A
        if constexpr (!POLY) acc[k].m -= a.ph.lw_unit;
    }

    // fp32: two queries per packed fp32x2 instruction
    constexpr bool PACKED = sizeof(T) == 4 && QPT % 2 == 0;
    [[maybe_unused]] Acc2 acc2[PACKED ? QPT / 2 : 1];
    [[maybe_unused]] f2 q2x[PACKED ? QPT / 2 : 1], q2y[PACKED ? QPT / 2 : 1], q2z[PACKED ? QPT / 2 : 1];
    if constexpr (PACKED) {
#pragma unroll
        for (int k = 0; k < QPT / 2; ++k) {
            acc2[k].from(acc[2 * k], acc[2 * k + 1]);
            q2x[k] = pack(qx[2 * k], qx[2 * k + 1]);
            q2y[k] = pack(qy[2 * k], qy[2 * k + 1]);
            q2z[k] = pack(qz[2 * k], qz[2 * k + 1]);
        }
    }

    // Evaluates the staged tile against this thread's queries; MODE as in
    // pair2.cuh exp_terms (fp64 always runs MODE 0).
    auto compute = [&](const T* tile, int n, auto mode) {
        constexpr int MODE = decltype(mode)::value;
#pragma unroll unroll_prims<T, KIND>()
        for (int i = 0; i < n; ++i) {
            T rec[R];
            using V = typename Vec4<T>::type;
            constexpr int NV = R * sizeof(T) / sizeof(V);
            const V* src = reinterpret_cast<const V*>(tile + size_t(i) * R);
#pragma unroll
            for (int j = 0; j < NV; ++j) reinterpret_cast<V*>(rec)[j] = src[j];
            if constexpr (PACKED) {
#pragma unroll
                for (int k = 0; k < QPT / 2; ++k) {
                    if constexpr (KIND == 0)
                        point_term2<MODE>(a.ph, q2x[k], q2y[k], q2z[k], (const float*)rec, acc2[k]);
                    else if constexpr (KIND == 1)
                        edge_term2<POLY, SAFE, MODE>(a.ph, a.poly, q2x[k], q2y[k], q2z[k], (const float*)rec, acc2[k]);
                    else
                        tri_term2<POLY, SAFE, MODE>(a.ph, a.poly, q2x[k], q2y[k], q2z[k], (const float*)rec, acc2[k]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < QPT; ++k) {
                    if constexpr (KIND == 0) point_term(a.ph, qx[k], qy[k], qz[k], rec[0], rec[1], rec[2], acc[k]);
                    else if constexpr (KIND == 1) edge_term<T, POLY, SAFE>(a.ph, a.poly, qx[k], qy[k], qz[k], rec, acc[k]);
                    else tri_term<T, POLY, SAFE>(a.ph, a.poly, qx[k], qy[k], qz[k], rec, acc[k]);
                }
            }
        }
    };

    // log2 of a running fp64 total, rounded down (exponent field), in the
    // launch's exponent frame (unit-weight launches: relative to lw_unit)
    [[maybe_unused]] auto total_log2 = [&](const Tot& tk) {
        const int ex = ((__double2hiint(tk.s) >> 20) & 0x7ff) - 1023;
        float lc = float(tk.M) + float(ex) - 1.f;  // (-1: float(M) may round up)
        if constexpr (!POLY) lc -= float(a.ph.lw_unit);
        return lc;
    };
    [[maybe_unused]] float seed[QPT];
    if constexpr (PRUNE) {
        const int64_t ntall = (a.count + TILE - 1) / TILE;
        float dmin2[QPT];
        int64_t gmin = 0;
#pragma unroll
        for (int k = 0; k < QPT; ++k) dmin2[k] = INFINITY;
        for (int64_t g = 0; g < ntall; ++g) {  // warp-uniform addresses: broadcast loads
            const float4 lo4 = __ldg(a.tbox + 2 * g), hi4 = __ldg(a.tbox + 2 * g + 1);
#pragma unroll
            for (int k = 0; k < QPT; ++k) {
                const float x = float(qx[k]), y = float(qy[k]), z = float(qz[k]);
                const float fx = fmaxf(fabsf(x - lo4.x), fabsf(x - hi4.x)),
                            fy = fmaxf(fabsf(y - lo4.y), fabsf(y - hi4.y)),
                            fz = fmaxf(fabsf(z - lo4.z), fabsf(z - hi4.z));
                const float d2 = fmaf(fx, fx, fmaf(fy, fy, fz * fz));
                if (k == 0 && d2 < dmin2[0]) gmin = g;
                dmin2[k] = fminf(dmin2[k], d2);
            }
        }
        if (threadIdx.x == 0) {
            const int64_t rel = gmin - p0 / TILE;  // (p0 is tile-aligned)
            t0s = ntiles > 0 ? int(max(int64_t(0), min(int64_t(ntiles - 1), rel))) : 0;
        }
        __syncthreads();
        t0 = t0s;
        if (threadIdx.x == 0)
            for (int t = 0; t < kStages && t < ntiles; ++t) issue(t);
#pragma unroll
        for (int k = 0; k < QPT; ++k) {  // (NaN queries: NaN seed, no tile is pruned)
            seed[k] = fmaf(float(a.ph.kappa), sqrtf(dmin2[k]) * (1.f + 1e-5f), float(a.lwmax) - float(a.lwspan)) - a.prune;
            // later segments of a mixed mesh: the sum of the earlier ones bounds c too
            const Tot& tk = tot[k * kThreads + threadIdx.x];
            if (tk.s > 0.0) seed[k] = fmaxf(seed[k], total_log2(tk) - a.prune);
        }
    }

    for (int t = 0; t < ntiles; ++t) {
        const int s = t % kStages;
        mbar_wait(&full[s], (t / kStages) & 1);
        const T* tile = tiles + size_t(s) * TILE * R;
        const int n = int(min(int64_t(TILE), p1 - (p0 + int64_t(tile_of(t)) * TILE)));
        int mode = 0;
        bool skip = false;
        if (a.tbox) {
            // Tile bounds from the tile's box: the nearest (dlo) and farthest
            // (dhi) possible distance of each query. dlo > 708/alpha masks
            // every term (smooth.hpp:85-88 zeroes them): the warp skips the
            // tile. dhi < 708/alpha: nothing can be masked. kappa dlo + lwmax
            // bounds every exponent: the shift is raised once here.
            const int64_t g = (p0 + int64_t(tile_of(t)) * TILE) / TILE;
            const float4 lo4 = __ldg(a.tbox + 2 * g), hi4 = __ldg(a.tbox + 2 * g + 1);
            const float span = float(-a.ph.kappa) * lo4.w + float(a.lwspan);
            bool all_skip = true, all_inside = true, any_loose = false;
#pragma unroll
            for (int k = 0; k < QPT; ++k) {
                const float x = float(qx[k]), y = float(qy[k]), z = float(qz[k]);
                const float ex = fmaxf(fmaxf(lo4.x - x, x - hi4.x), 0.f), ey = fmaxf(fmaxf(lo4.y - y, y - hi4.y), 0.f),
                            ez = fmaxf(fmaxf(lo4.z - z, z - hi4.z), 0.f);
                const float fx = fmaxf(fabsf(x - lo4.x), fabsf(x - hi4.x)),
                            fy = fmaxf(fabsf(y - lo4.y), fabsf(y - hi4.y)),
                            fz = fmaxf(fabsf(z - lo4.z), fabsf(z - hi4.z));
                const float dlo = sqrtf(fmaf(ex, ex, fmaf(ey, ey, ez * ez))) * (1.f - 1e-5f);
                const float dhi = sqrtf(fmaf(fx, fx, fmaf(fy, fy, fz * fz))) * (1.f + 1e-5f);
                const bool sk = qi[k] >= a.Q || dlo > float(a.ph.dmax);
                if constexpr (PRUNE) all_skip = all_skip && (sk || fmaf(float(a.ph.kappa), dlo, float(a.lwmax)) < seed[k]);
                else all_skip = all_skip && sk;
                all_inside = all_inside && (qi[k] >= a.Q || dhi < float(a.ph.dmax));
                const float H = dlo < kNearBox ? kTileHeadroomNear : kTileHeadroom;
                const bool loose = !sk && span > H + kLooseMargin;
                any_loose = any_loose || loose;
                if (!loose && !sk) {  // raise the shift to the tile's exponent bound
                    const T up = T(fmaf(float(a.ph.kappa), dlo, float(a.lwmax))) - T(H);
                    if constexpr (PACKED) {
                        Acc2& a2 = acc2[k / 2];
                        const float mk = (k & 1) ? hi(a2.m) : lo(a2.m);
                        if (float(up) > mk) {
                            Acc<float> u, v;
                            a2.to(u, v);
                            Acc<float>& w = (k & 1) ? v : u;
                            w.scale(Math<float>::ex2(w.m - float(up)));
                            w.m = float(up);
                            a2.from(u, v);
                        }
                    } else if (up > acc[k].m) {
                        acc[k].scale(Math<T>::ex2(acc[k].m - up));
                        acc[k].m = up;
                    }
                }
            }
            skip = __all_sync(0xffffffffu, all_skip);
            const bool inside = __all_sync(0xffffffffu, all_inside);
            mode = __any_sync(0xffffffffu, any_loose) ? 0 : (inside ? 2 : 1);
        }
        if (!skip) {
            if constexpr (PACKED) {
                if (mode == 2) compute(tile, n, std::integral_constant<int, 2>());
                else if (mode == 1) compute(tile, n, std::integral_constant<int, 1>());
                else compute(tile, n, std::integral_constant<int, 0>());
            } else {
                compute(tile, n, std::integral_constant<int, 0>());
            }
        }
        if constexpr (PACKED) {
#pragma unroll
            for (int k = 0; k < QPT / 2; ++k) acc2[k].to(acc[2 * k], acc[2 * k + 1]);
        }
#pragma unroll
        for (int k = 0; k < QPT; ++k) {
            if constexpr (!POLY) acc[k].m += a.ph.lw_unit;  // totals are absolute
            tot[k * kThreads + threadIdx.x].flush(acc[k]);
            if constexpr (!POLY) acc[k].m -= a.ph.lw_unit;
        }
        if constexpr (PRUNE) {
            // the running total is a lower bound of c as well (floor of its
            // log2 from the fp64 exponent field): usually tighter than the
            // box seed once a near tile has been summed
            if (!skip) {
#pragma unroll
                for (int k = 0; k < QPT; ++k) {
                    const Tot& tk = tot[k * kThreads + threadIdx.x];
                    if (tk.s > 0.0) seed[k] = fmaxf(seed[k], total_log2(tk) - a.prune);
                }
            }
        }
        if constexpr (PACKED) {
#pragma unroll
            for (int k = 0; k < QPT / 2; ++k) acc2[k].from(acc[2 * k], acc[2 * k + 1]);
        }
        __syncthreads();  // every thread is done with stage s
        if (threadIdx.x == 0 && t + kStages < ntiles) issue(t + kStages);
    }

    if (a.cluster) {  // fold the other splits' totals into split 0 over DSMEM
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        if (split == 0) {
            for (unsigned r = 1; r < cl.num_blocks(); ++r) {
                const Tot* rt = cl.map_shared_rank(tot, r);
#pragma unroll
                for (int k = 0; k < QPT; ++k) tot_merge(tot[k * kThreads + threadIdx.x], rt[k * kThreads + threadIdx.x]);
            }
        }
        cl.sync();  // the remote totals stay alive until split 0 has read them
        if (split != 0) return;
    }
#pragma unroll
    for (int k = 0; k < QPT; ++k) {
        if (qi[k] >= a.Q) continue;
        const Tot& tk = tot[k * kThreads + threadIdx.x];
        part[qi[k]] = tk.M;
        part[a.Q + qi[k]] = tk.s;
        part[2 * a.Q + qi[k]] = tk.gx;
        part[3 * a.Q + qi[k]] = tk.gy;
        part[4 * a.Q + qi[k]] = tk.gz;
    }
}

// Queries per thread (amortise record loads) and the launch-bounds CTA
// floor per (type, kind). fp64 values from tools/fp64_sweep.sh on a B200
// (ms per evaluation, QPT 1/2/4 x floor 1/2): points QPT 2 (cfg1 0.886 ms vs
// 0.906 / 1.001-1.183), edges QPT 2 with 2 CTAs/SM (cfg2 32.2 ms vs
// 33.5-37.2), triangles QPT 1 with 2 CTAs/SM (cfg3 torus, 32k queries:
// 109.5 ms vs 114.7-125.6).
template <class T, int KIND>
constexpr int qpt_for() {
#ifdef SD_K1_QPT_TRI  // A/B: queries per thread of the fp32 triangle kernel
    if constexpr (sizeof(T) == 4 && KIND == 2) return SD_K1_QPT_TRI;
#endif
#ifdef SD_K1_QPT_EDGE  // A/B: queries per thread of the fp32 edge kernel
    if constexpr (sizeof(T) == 4 && KIND == 1) return SD_K1_QPT_EDGE;
#endif
    if constexpr (sizeof(T) == 4) return KIND == 0 ? 4 : 2;  // (edges: 2 since round 2, see unroll_prims)
    else return KIND == 2 ? 1 : 2;
}
template <class T, int KIND>
constexpr int minb_for() {
    // fp32: 3 CTAs/SM (<= 85 registers): cfg2 6.89 ms vs 6.92 at one CTA floor
    // (126 registers), cfg3 1.113 s vs 1.128 s
#ifdef SD_K1_MINB
    if constexpr (sizeof(T) == 4) return SD_K1_MINB;
#endif
    return sizeof(T) == 4 ? 3 : (KIND != 0 ? 2 : 1);
}

template <class T, int KIND, int QPT>
static size_t smem_bytes() {
    return size_t(kStages) * tile_prims<T, KIND>() * rec_size(KIND) * sizeof(T) + size_t(QPT) * kThreads * sizeof(Tot);
}

template <class T, int KIND, bool POLY, bool SAFE, class F>
static auto with_kernel(F&& f, bool prune = false) {
    constexpr int QPT = qpt_for<T, KIND>();
    if (prune) return f(exact_kernel<T, KIND, POLY, SAFE, QPT, minb_for<T, KIND>(), true>, smem_bytes<T, KIND, QPT>(), QPT);
    return f(exact_kernel<T, KIND, POLY, SAFE, QPT, minb_for<T, KIND>()>, smem_bytes<T, KIND, QPT>(), QPT);
}

template <class T, int KIND, bool POLY, bool SAFE>
static cudaError_t launch_one(const ExactLaunch<T>& L, cudaStream_t st) {
    return with_kernel<T, KIND, POLY, SAFE>([&](auto kern, size_t smem, int QPT) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        ExactArgs<T> a;
        a.rec = L.rec;
        a.count = L.count;
        a.chunk = L.chunk;
        a.q = L.q;
        a.Q = L.Q;
        a.part = L.part;
        a.first = L.first;
        a.ph = L.ph;
        a.poly = L.poly;
        a.perm = L.perm;
        a.tbox = L.tbox;
        a.lwmax = L.lwmax;
        a.lwspan = L.lwspan;
        a.cluster = L.cluster ? 1 : 0;
        a.prune = L.prune;
        const int64_t qblocks = (L.Q + int64_t(kThreads) * QPT - 1) / (int64_t(kThreads) * QPT);
        dim3 grid(unsigned(qblocks), unsigned(L.splits));
        if (!L.cluster) {
            kern<<<grid, kThreads, smem, st>>>(a);
            return cudaGetLastError();
        }
        if (L.splits > 8) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (e != cudaSuccess) return e;
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = unsigned(L.splits);
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, a);
    }, L.prune > 0.f && L.tbox != nullptr);
}

template <class T, int KIND, bool POLY, bool SAFE>
static int occupancy_one() {
    return with_kernel<T, KIND, POLY, SAFE>([&](auto kern, size_t smem, int) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 1;
        int n = 1;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, kThreads, smem) != cudaSuccess) return 1;
        return n > 0 ? n : 1;
    });
}

template <class T>
int exact_blocks_per_sm(int kind, bool has_poly, bool safe) {
    if (kind == 0) return occupancy_one<T, 0, false, false>();
    if (kind == 1) return !has_poly ? occupancy_one<T, 1, false, false>()
                                    : (safe ? occupancy_one<T, 1, true, true>() : occupancy_one<T, 1, true, false>());
    return !has_poly ? occupancy_one<T, 2, false, false>()
                     : (safe ? occupancy_one<T, 2, true, true>() : occupancy_one<T, 2, true, false>());
}
template int exact_blocks_per_sm<float>(int, bool, bool);
template int exact_blocks_per_sm<double>(int, bool, bool);

int exact_tile_prims(int kind) { return kind == 0 ? tile_prims<float, 0>() : tile_prims<float, 1>(); }

template <class T>
int64_t exact_queries_per_cta(int kind) {
    const int q = kind == 0 ? qpt_for<T, 0>() : (kind == 1 ? qpt_for<T, 1>() : qpt_for<T, 2>());
    return int64_t(kThreads) * q;
}
template int64_t exact_queries_per_cta<float>(int);
template int64_t exact_queries_per_cta<double>(int);

template <class T>
cudaError_t launch_exact(const ExactLaunch<T>& L, cudaStream_t st) {
    if (L.kind == 0) return launch_one<T, 0, false, false>(L, st);
    if (L.kind == 1) {
        if (!L.has_poly) return launch_one<T, 1, false, false>(L, st);
        return L.safe ? launch_one<T, 1, true, true>(L, st) : launch_one<T, 1, true, false>(L, st);
    }
    if (L.kind == 2) {
        if (!L.has_poly) return launch_one<T, 2, false, false>(L, st);
        return L.safe ? launch_one<T, 2, true, true>(L, st) : launch_one<T, 2, true, false>(L, st);
    }
    return cudaErrorInvalidValue;
}

template cudaError_t launch_exact<float>(const ExactLaunch<float>&, cudaStream_t);
template cudaError_t launch_exact<double>(const ExactLaunch<double>&, cudaStream_t);

}  // namespace sdgpu
