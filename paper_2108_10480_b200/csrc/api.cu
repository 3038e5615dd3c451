// api.cu -- the C ABI of include/sdgpu.h: context lifetime, geometry and
// weight upload (AoS fp64 mesh -> per-kind SoA-ish records grouped into
// (kind, polynomial) segments), and query dispatch to K1/K3/K4.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <fstream>
#include <stdexcept>

#include <zlib.h>

#include "context.h"
#include "weights_host.h"

namespace sdgpu {

static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }

void check_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw CudaError{e, where};
}

struct ArgError {
    std::string msg;
};
struct StateError {
    std::string msg;
};

template <class F>
static int guard(F&& f) {
    try {
        f();
        return SD_OK;
    } catch (const ArgError& e) {
        set_error(e.msg);
        return SD_E_ARG;
    } catch (const StateError& e) {
        set_error(e.msg);
        return SD_E_STATE;
    } catch (const CudaError& e) {
        set_error(std::string("CUDA error in ") + e.where + ": " + cudaGetErrorString(e.code));
        return SD_E_CUDA;
    } catch (const std::bad_alloc&) {
        set_error("out of host memory");
        return SD_E_NOMEM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return SD_E_ARG;
    }
}

struct DeviceScope {  // makes ctx->device current for the duration of a call
    int prev = -1;
    explicit DeviceScope(int dev) {
        check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceScope() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ------------------------------------------------------------ host math
struct D3 {
    double x, y, z;
};
static inline D3 sub(D3 a, D3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
static inline double dot3(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline D3 cross3(D3 a, D3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
static inline D3 scale3(D3 a, double s) { return {a.x * s, a.y * s, a.z * s}; }

static inline D3 vtx(const Ctx& c, int32_t i) { return {c.xyz[3 * size_t(i)], c.xyz[3 * size_t(i) + 1], c.xyz[3 * size_t(i) + 2]}; }

template <class T>
void build_record(const Ctx& c, int64_t prim, T* out) {
    const int k = c.kind[prim];
    const int32_t* s = &c.sv[3 * size_t(prim)];
    const D3 a = vtx(c, s[0]);
    for (int i = 0; i < rec_size(k); ++i) out[i] = T(0);
    out[0] = T(a.x);
    out[1] = T(a.y);
    out[2] = T(a.z);
    if (k == SD_EDGE) {
        const D3 e = sub(vtx(c, s[1]), a);
        const double e2 = dot3(e, e);
        const double inv = e2 > 0 ? 1.0 / e2 : 0.0;  // exact.hpp:71: t = 0 if |e|^2 <= 0
        out[3] = T(e.x); out[4] = T(e.y); out[5] = T(e.z);
        out[6] = T(inv);
        out[7] = T(e.x * inv); out[8] = T(e.y * inv); out[9] = T(e.z * inv);
    } else if (k == SD_TRIANGLE) {
        const D3 b = vtx(c, s[1]), cc = vtx(c, s[2]);
        const D3 ab = sub(b, a), ac = sub(cc, a), bc = sub(cc, b);
        const double A = dot3(ab, ab), B = dot3(ab, ac), C = dot3(ac, ac), BC = dot3(bc, bc);
        const double det = A * C - B * B;
        out[3] = T(ab.x); out[4] = T(ab.y); out[5] = T(ab.z);
        out[6] = T(ac.x); out[7] = T(ac.y); out[8] = T(ac.z);
        out[9] = T(A); out[10] = T(B); out[11] = T(C);
        out[12] = T(1.0 / A); out[13] = T(1.0 / C); out[14] = T(1.0 / BC); out[15] = T(1.0 / det);
        // barycentric shape gradients without the 1/alpha (weights.hpp:689-696)
        const D3 n = cross3(ab, ac);
        const double nn = dot3(n, n);
        const double inv = nn > 0 ? 1.0 / nn : 0.0;
        const D3 g1 = scale3(cross3(n, sub(a, cc)), inv), g2 = scale3(cross3(n, ab), inv);
        out[16] = T(g1.x); out[17] = T(g1.y); out[18] = T(g1.z);
        out[19] = T(g2.x); out[20] = T(g2.y); out[21] = T(g2.z);
    }
}
template void build_record<float>(const Ctx&, int64_t, float*);
template void build_record<double>(const Ctx&, int64_t, double*);

template <class T>
Phys<T> make_phys(const Ctx& c, const sd_params& p) {
    const double S = p.alpha / std::max(p.alpha, p.alpha_u);  // params.hpp:21
    Phys<T> ph;
    ph.kappa = T(-p.alpha * 1.4426950408889634);
    ph.dmax = T(708.0 / p.alpha);
    ph.S = T(S);
    ph.A = T(c.A);
    ph.lw_unit = T(S * std::log2(std::max(c.A, 1e-300)));
    ph.lw_floor = T(S * std::log2(1e-300));
    ph.w_ff = T(std::pow(std::max(c.A * c.sup_wtilde, 1e-300), S));  // weights.hpp:576-578
    ph.beta = T(p.beta);
    return ph;
}
template Phys<float> make_phys<float>(const Ctx&, const sd_params&);
template Phys<double> make_phys<double>(const Ctx&, const sd_params&);

// Expands the 13 stored slots to the symmetric 8x8 grid (weights.hpp:155-161).
static void tri_grid(const Ctx& c, int poly, double g[8][8]) {
    static const int kStored[13][2] = {{0, 0}, {0, 2}, {0, 3}, {0, 4}, {0, 5}, {0, 6}, {0, 7},
                                       {2, 2}, {2, 3}, {2, 4}, {2, 5}, {3, 3}, {3, 4}};
    for (int j = 0; j < 8; ++j)
        for (int k = 0; k < 8; ++k) g[j][k] = 0.0;
    const double* st = &c.tri_stored[13 * size_t(poly)];
    for (int m = 0; m < 13; ++m) {
        g[kStored[m][0]][kStored[m][1]] = st[m];
        g[kStored[m][1]][kStored[m][0]] = st[m];
    }
}

static double binom(int n, int k) {
    double r = 1.0;
    for (int i = 0; i < k; ++i) r = r * (n - i) / (i + 1);
    return r;
}

// True when A w~ > 0 is certified on the whole domain by the Bernstein
// coefficients (the minimum Bernstein coefficient bounds the polynomial
// from below), so the kernels may drop the 1e-300 floor selects.
static double bernstein_min(const Ctx& c, int kind, int poly) {
    double lo = INFINITY;
    if (kind == SD_EDGE) {  // degree-4 Bernstein on [0, 1]
        const double* a = &c.edge_a[5 * size_t(poly)];
        for (int i = 0; i <= 4; ++i) {
            double b = 0.0;
            for (int j = 0; j <= i; ++j) b += binom(i, j) / binom(4, j) * a[j];
            lo = std::min(lo, b);
        }
    } else {  // degree-7 Bernstein on the triangle
        double g[8][8];
        tri_grid(c, poly, g);
        for (int a = 0; a <= 7; ++a)
            for (int b = 0; a + b <= 7; ++b) {
                double s = 0.0;
                for (int j = 0; j <= a; ++j)
                    for (int k = 0; k <= b; ++k)
                        s += g[j][k] * binom(a, j) * binom(b, k) / (binom(7, j + k) * binom(j + k, j));
                lo = std::min(lo, s);
            }
    }
    return lo;
}

bool poly_certified_positive(const Ctx& c, int kind, int poly) {
    if (poly < 0) return true;
    return c.A * bernstein_min(c, kind, poly) > 1e-6;
}

static double poly_lower_bound(const Ctx& c, int kind, int poly) {
    return poly < 0 ? 1.0 : std::max(0.0, bernstein_min(c, kind, poly));
}

// Coefficient packing and pre-scaling documented in pair.cuh (Poly).
template <class T>
Poly<T> make_poly(const Ctx& c, int kind, int poly, const sd_params& p) {
    Poly<T> out;
    for (int i = 0; i < kPolyCoefs; ++i) out.c[i] = T(0);
    if (poly < 0) return out;
    const double S = p.alpha / std::max(p.alpha, p.alpha_u);
    const double A = c.A, K = S * c.A / (p.alpha * p.alpha);
    if (kind == SD_EDGE) {
        const double* a = &c.edge_a[5 * size_t(poly)];
        for (int i = 0; i < 5; ++i) out.c[i] = T(A * a[i]);
        out.c[5] = T(K * a[1]);
        out.c[6] = T(K * 2 * a[2]);
        out.c[7] = T(K * 3 * a[3]);
        out.c[8] = T(K * 4 * a[4]);
        return out;
    }
    double g[8][8];
    tri_grid(c, poly, g);
    // w~ is symmetric in (x, y) (weights.hpp:155-170 mirrors every stored
    // coefficient), so it is a polynomial in s = x + y and p = x y:
    // c_jj x^j y^j = c_jj p^j and c_jk (x^j y^k + x^k y^j) = c_jk p^j P_{k-j}
    // with the power sums P_0 = 2, P_1 = s, P_m = s P_{m-1} - p P_{m-2}.
    // a[i][j] (coefficient of s^i p^j, i + 2 j <= 7): 20 terms instead of
    // the 23 + 16 + 16 of the (x, y) rows, and the partials follow from
    // d/dx = W_s + y W_p, d/dy = W_s + x W_p (tri_poly, pair.cuh).
    double P[8][8][4] = {};  // P[m][i][j]
    P[0][0][0] = 2.0;
    P[1][1][0] = 1.0;
    for (int m = 2; m < 8; ++m)
        for (int i = 0; i < 8; ++i)
            for (int j = 0; j < 4; ++j)
                P[m][i][j] = (i > 0 ? P[m - 1][i - 1][j] : 0.0) - (j > 0 ? P[m - 2][i][j - 1] : 0.0);
    double a[8][4] = {};
    for (int j = 0; j < 8; ++j)
        for (int k = j; j + k <= 7; ++k) {
            if (k == j) {
                a[0][j] += g[j][j];
                continue;
            }
            for (int i = 0; i < 8; ++i)
                for (int jj = 0; jj + j < 4; ++jj) a[i][jj + j] += g[j][k] * P[k - j][i][jj];
        }
    // layout (kTriSP*): value rows A_j(s) = sum_i a_ij s^i (x A) for j = 0..3
    // (degrees 7, 5, 3, 1), then the s-derivative rows B_j(s) = sum_i i a_ij
    // s^(i-1) (x K) (degrees 6, 4, 2, 0), then K / A, 2 K / A, 3 K / A
    int n = 0;
    const int deg[4] = {7, 5, 3, 1};
    for (int j = 0; j < 4; ++j)
        for (int i = 0; i <= deg[j]; ++i) out.c[n++] = T(A * a[i][j]);
    for (int j = 0; j < 4; ++j)
        for (int i = 1; i <= deg[j]; ++i) out.c[n++] = T(K * i * a[i][j]);
    out.c[n++] = T(K / A);
    out.c[n++] = T(2.0 * K / A);
    out.c[n++] = T(3.0 * K / A);
    if (n != kTriSPCoefs) throw std::logic_error("triangle polynomial packing");
    return out;
}
template Poly<float> make_poly<float>(const Ctx&, int, int, const sd_params&);
template Poly<double> make_poly<double>(const Ctx&, int, int, const sd_params&);

// --------------------------------------------------------- exact layout
static uint64_t spread21h(uint64_t v) {
    v &= 0x1fffffull;
    v = (v | (v << 32)) & 0x1f00000000ffffull;
    v = (v | (v << 16)) & 0x1f0000ff0000ffull;
    v = (v | (v << 8)) & 0x100f00f00f00f00full;
    v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

// Records per kind, grouped into (kind, polynomial) segments, Morton-ordered
// inside each segment so that every staged tile is spatially compact; one
// bounding box per tile (float, rounded outward) for the culling bounds of
// exact.cu. Summation order is free: the reference's sum is re-associated
// anyway by the parallel reduction.
template <class T>
static void prepare_exact(Ctx& c) {
    if (c.exact_ready) return;
    c.segs.clear();
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t v = 0; v < c.V; ++v)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], c.xyz[3 * size_t(v) + a]);
            hi[a] = std::max(hi[a], c.xyz[3 * size_t(v) + a]);
        }
    for (int a = 0; a < 3; ++a) {
        c.scene_lo[a] = c.V ? lo[a] : 0.0;
        c.scene_hi[a] = c.V ? hi[a] : 0.0;
    }
    auto corners = [&](int64_t i, double blo[3], double bhi[3]) {
        for (int a = 0; a < 3; ++a) {
            blo[a] = INFINITY;
            bhi[a] = -INFINITY;
        }
        for (int k = 0; k <= c.kind[i]; ++k)
            for (int a = 0; a < 3; ++a) {
                const double x = c.xyz[3 * size_t(c.sv[3 * i + k]) + a];
                blo[a] = std::min(blo[a], x);
                bhi[a] = std::max(bhi[a], x);
            }
    };
    std::vector<uint64_t> key(size_t(c.N));
    for (int64_t i = 0; i < c.N; ++i) {
        double blo[3], bhi[3];
        corners(i, blo, bhi);
        uint64_t m = 0;
        for (int a = 0; a < 3; ++a) {
            const double span = c.scene_hi[a] - c.scene_lo[a];
            const double f = span > 0 ? (0.5 * (blo[a] + bhi[a]) - c.scene_lo[a]) / span * 2097151.0 : 0.0;
            m |= spread21h(uint64_t(std::min(std::max(f, 0.0), 2097151.0))) << (2 - a);
        }
        key[i] = m;
    }
    for (int k = 0; k < 3; ++k) {
        std::vector<int64_t> ids;
        for (int64_t i = 0; i < c.N; ++i)
            if (c.kind[i] == k) ids.push_back(i);
        auto pk = [&](int64_t i) { return k == SD_POINT ? -1 : c.poly_index[i]; };
        std::stable_sort(ids.begin(), ids.end(), [&](int64_t a, int64_t b) {
            return pk(a) != pk(b) ? pk(a) < pk(b) : key[a] < key[b];
        });
        const int R = rec_size(k);
        std::vector<T> host(ids.size() * size_t(R));
        for (size_t j = 0; j < ids.size(); ++j) build_record<T>(c, ids[j], &host[j * R]);
        T* d = static_cast<T*>(c.rec[k].ensure(host.size() * sizeof(T)));
        if (!host.empty())
            check_cuda(cudaMemcpy(d, host.data(), host.size() * sizeof(T), cudaMemcpyHostToDevice), "upload records");
        const int64_t TILE = exact_tile_prims(k);
        std::vector<float4> boxes;
        size_t j = 0;
        while (j < ids.size()) {
            const int poly = pk(ids[j]);
            size_t e = j;
            while (e < ids.size() && pk(ids[e]) == poly) ++e;
            c.segs.push_back({k, poly, int64_t(j), int64_t(e - j), int64_t(boxes.size() / 2)});
            for (size_t t = j; t < e; t += size_t(TILE)) {
                double blo[3] = {INFINITY, INFINITY, INFINITY}, bhi[3] = {-INFINITY, -INFINITY, -INFINITY};
                for (size_t u = t; u < std::min(e, t + size_t(TILE)); ++u) {
                    double plo[3], phi[3];
                    corners(ids[u], plo, phi);
                    for (int a = 0; a < 3; ++a) {
                        blo[a] = std::min(blo[a], plo[a]);
                        bhi[a] = std::max(bhi[a], phi[a]);
                    }
                }
                float fl[3], fh[3];
                for (int a = 0; a < 3; ++a) {
                    fl[a] = float(blo[a]);
                    fh[a] = float(bhi[a]);
                    if (double(fl[a]) > blo[a]) fl[a] = std::nextafter(fl[a], -INFINITY);
                    if (double(fh[a]) < bhi[a]) fh[a] = std::nextafter(fh[a], INFINITY);
                }
                const double dg = std::sqrt(double(fh[0] - fl[0]) * (fh[0] - fl[0]) +
                                            double(fh[1] - fl[1]) * (fh[1] - fl[1]) +
                                            double(fh[2] - fl[2]) * (fh[2] - fl[2]));
                boxes.push_back(make_float4(fl[0], fl[1], fl[2], float(dg) * (1.0f + 1e-6f)));
                boxes.push_back(make_float4(fh[0], fh[1], fh[2], 0.0f));
            }
            j = e;
        }
        float4* db = static_cast<float4*>(c.tbox[k].ensure(boxes.size() * sizeof(float4)));
        if (!boxes.empty())
            check_cuda(cudaMemcpy(db, boxes.data(), boxes.size() * sizeof(float4), cudaMemcpyHostToDevice),
                       "upload tile boxes");
    }
    c.exact_ready = true;
}

template <class T>
__global__ void convert_queries(const double* __restrict__ in, T* __restrict__ out, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = T(in[i]);
}

template <class T>
static void exact_query(Ctx& c, const T* q, int64_t Q, const sd_params& p, const FinalizeOut& out,
                        cudaStream_t st) {
    prepare_exact<T>(c);
    if (c.segs.empty()) {
        check_cuda(launch_empty_result(Q, out, st), "empty result");
        c.last_launches = 1;
        return;
    }
    // splits of the primitive range: enough CTAs to fill every SM, and a
    // CTA count close to a whole number of waves (all CTAs do equal work,
    // so a partial last wave is pure loss)
    int64_t maxcount = 0;
    const Segment* big = &c.segs[0];
    for (const Segment& s : c.segs)
        if (s.count > maxcount) maxcount = s.count, big = &s;
    const int64_t qpc = exact_queries_per_cta<T>(big->kind);
    const int64_t qblocks = (Q + qpc - 1) / qpc;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
    const int64_t slots = int64_t(sms) * exact_blocks_per_sm<T>(big->kind, big->poly >= 0,
                                                                  poly_certified_positive(c, big->kind, big->poly));
    const int64_t max_splits = std::max<int64_t>(1, std::min<int64_t>(64, maxcount / 256));
    int64_t splits = 1;
    double best = -1.0;
    for (int64_t s = 1; s <= max_splits; ++s) {
        const double waves = double(qblocks * s) / double(slots);
        const double eff = waves / std::ceil(waves);
        const double score = eff - (waves < 1.0 ? 1.0 : 0.0) - 0.002 * double(s);  // prefer few splits
        if (score > best + 1e-9) best = score, splits = s;
        if (waves >= 1.0 && eff >= 0.97) break;
    }
    if (const char* fs = std::getenv("SDGPU_EXACT_SPLITS"); fs && *fs)  // forced split count (tests, A/B)
        splits = std::max<int64_t>(1, std::min<int64_t>(64, std::atoi(fs)));
    double* part = static_cast<double*>(c.part.ensure(size_t(splits) * 5 * Q * sizeof(double)));
    const Phys<T> ph = make_phys<T>(c, p);
    int64_t launches = 0;
    // queries in Morton order so that a warp's queries share tile bounds
    // (Morton over the scene box; a Hilbert order over the joined boxes
    // measured the same on cfg2: 6.885 vs 6.890 ms)
    const int64_t* perm = sort_queries<T>(c, q, Q, c.scene_lo, c.scene_hi, st, launches, false);
    const double S = p.alpha / std::max(p.alpha, p.alpha_u);
    bool first = true;
    // SDGPU_CLUSTER=1: the split CTAs of a query block form one thread-block
    // cluster (2..16 CTAs; more than 8 is a non-portable size, allowed on
    // B200) and merge their fp64 totals over distributed shared memory, so
    // that only split 0 writes a partial. Off by default: the partial round
    // trip costs ~0.4 % of HBM bandwidth (cfg2: 252 MB over 6.9 ms), while
    // cluster co-scheduling cost 32 % on cfg2 (12-CTA clusters: 9.19 vs
    // 6.94 ms) and 5 % on cfg3 (3-CTA clusters: 1021 vs 974 ms).
    const char* ce = std::getenv("SDGPU_CLUSTER");
    const bool cluster = splits > 1 && splits <= 16 && ce && *ce == '1';
    KernelTimer timer(c, st);
    for (const Segment& s : c.segs) {
        ExactLaunch<T> L;
        L.kind = s.kind;
        L.has_poly = s.poly >= 0;
        L.safe = poly_certified_positive(c, s.kind, s.poly);
        L.rec = c.rec[s.kind].as<T>() + s.offset * rec_size(s.kind);
        L.count = s.count;
        L.splits = int(splits);
        L.cluster = cluster;
        const int64_t TILE = exact_tile_prims(s.kind);
        L.chunk = ((s.count + splits - 1) / splits + TILE - 1) / TILE * TILE;  // tile-aligned splits
        L.perm = perm;
        L.tbox = c.tbox[s.kind].as<float4>() + 2 * s.tile0;
        if (s.poly < 0) {  // unit weights: the shift is kept relative to S log2 A in the kernel
            L.lwmax = T(0);
            L.lwspan = T(0);
        } else {
            const double hi = S * std::log2(std::max(c.A * c.sup_wtilde, 1e-300));
            const double lo = S * std::log2(std::max(c.A * poly_lower_bound(c, s.kind, s.poly), 1e-300));
            L.lwmax = T(hi);
            L.lwspan = T(hi - lo);
        }
        L.prune = float(c.exact_prune_bits);
        L.q = q;
        L.Q = Q;
        L.part = part;
        L.first = first ? 1 : 0;
        L.ph = ph;
        L.poly = make_poly<T>(c, s.kind, s.poly, p);
        check_cuda(launch_exact<T>(L, st), "exact kernel launch");
        ++launches;
        first = false;
    }
    timer.stop();
    check_cuda(launch_finalize(part, cluster ? 1 : int(splits), Q, p.alpha, p.epsilon, c.N, nullptr, nullptr, nullptr, perm,
                                  out, st),
               "finalize launch");
    c.last_launches = launches + 1;
}

static void check_params(const sd_params* p) {
    if (!p) throw ArgError{"params is NULL"};
    if (!(p->alpha > 0) || !std::isfinite(p->alpha)) throw ArgError{"alpha must be positive and finite"};
    if (!(p->alpha_u > 0)) throw ArgError{"alpha_u must be positive"};
    if (!(p->beta >= 0) || !std::isfinite(p->beta)) throw ArgError{"beta must be >= 0"};
    if (!(p->epsilon >= 0)) throw ArgError{"epsilon must be >= 0"};
}

static void check_ready(const Ctx& c, int mode) {
    if (!c.have_geom) throw StateError{"no geometry: call sd_set_geometry first"};
    if (!c.have_weights) throw StateError{"no weight table: call sd_set_weights first"};
    if (mode == SD_BVH && !c.have_tree && c.N > 0) throw StateError{"no tree: call sd_set_bvh or sd_build_bvh first"};
    if (mode != SD_EXACT && mode != SD_BVH) throw ArgError{"mode must be SD_EXACT or SD_BVH"};
}

template <class T>
static void dispatch(Ctx& c, const T* q, int64_t Q, const sd_params& p, int mode, const FinalizeOut& out,
                     cudaStream_t st) {
    if (Q == 0) {
        c.last_launches = 0;
        return;
    }
    FinalizeOut o = out;
    if constexpr (sizeof(T) == 4) o.qf = q;
    else o.qd = q;
    if (mode == SD_BVH && c.N > 0) tree_query<T>(c, q, Q, p, o, st);
    else exact_query<T>(c, q, Q, p, o, st);
}

// fp64 query points already on the device, converted to the context
// precision and evaluated (batched callers, callers.cu). Uses c.qT.
void query_batch_f64(Ctx& c, const double* q, int64_t Q, const sd_params& p, int mode, const FinalizeOut& out,
                     cudaStream_t st) {
    if (c.precision == SD_FP32) {
        float* qf = static_cast<float*>(c.qT.ensure(size_t(std::max<int64_t>(Q, 1)) * 3 * sizeof(float)));
        if (Q > 0) {
            convert_queries<float><<<unsigned((3 * Q + 255) / 256), 256, 0, st>>>(q, qf, 3 * Q);
            check_cuda(cudaGetLastError(), "convert queries");
        }
        dispatch<float>(c, qf, Q, p, mode, out, st);
    } else {
        dispatch<double>(c, q, Q, p, mode, out, st);
    }
}

// Surface-area cost of a tree: sum over internal nodes of the box area,
// relative to the root's.
static double sah_cost(const std::vector<sd_bvh_node>& t) {
    if (t.empty()) return 0.0;
    auto area = [](const sd_bvh_node& n) {
        const double x = std::max(0.0, n.hi[0] - n.lo[0]), y = std::max(0.0, n.hi[1] - n.lo[1]),
                     z = std::max(0.0, n.hi[2] - n.lo[2]);
        return 2.0 * (x * y + y * z + x * z);
    };
    double sum = 0.0;
    for (const sd_bvh_node& n : t)
        if (n.left >= 0) sum += area(n);
    const double root = area(t[0]);
    return root > 0.0 ? sum / root : sum;
}

// Metadata of a table given as bare coefficients: edge valences follow from
// w~(0) = 1/v0, w~(1) = 1/v1 (weights.hpp:46-76) and the extrema are closed
// form; triangle valences are unknown (0) and the extrema are sampled.
static void set_default_meta(Ctx& c) {
    const size_t ne = c.edge_a.size() / 5, nt = c.tri_stored.size() / 13;
    c.edge_val.assign(2 * ne, 0);
    c.edge_ext.assign(2 * ne, 0.0);
    for (size_t k = 0; k < ne; ++k) {
        const double* a = &c.edge_a[5 * k];
        const double w0 = a[0], w1 = a[0] + a[1] + a[2] + a[3] + a[4];
        c.edge_val[2 * k] = w0 > 0 ? int32_t(std::lround(1.0 / w0)) : 0;
        c.edge_val[2 * k + 1] = w1 > 0 ? int32_t(std::lround(1.0 / w1)) : 0;
        double sup = -INFINITY, inf = INFINITY;
        for (int i = 0; i <= 1000; ++i) {
            const double t = i / 1000.0;
            const double v = a[0] + t * (a[1] + t * (a[2] + t * (a[3] + t * a[4])));
            sup = std::max(sup, v);
            inf = std::min(inf, v);
        }
        c.edge_ext[2 * k] = sup;
        c.edge_ext[2 * k + 1] = inf;
    }
    c.tri_val.assign(2 * nt, 0);
    c.tri_ext.assign(3 * nt, 0.0);
    static const int kS[13][2] = {{0, 0}, {0, 2}, {0, 3}, {0, 4}, {0, 5}, {0, 6}, {0, 7},
                                  {2, 2}, {2, 3}, {2, 4}, {2, 5}, {3, 3}, {3, 4}};
    for (size_t k = 0; k < nt; ++k) {
        double g[8][8] = {};
        for (int m = 0; m < 13; ++m) g[kS[m][0]][kS[m][1]] = g[kS[m][1]][kS[m][0]] = c.tri_stored[13 * k + m];
        double sup = -INFINITY, inf = INFINITY;
        const int N = 128;
        for (int i = 0; i <= N; ++i)
            for (int j = 0; i + j <= N; ++j) {
                const double x = double(i) / N, y = double(j) / N;
                double v = 0;
                for (int jj = 7; jj >= 0; --jj) {
                    double row = 0;
                    for (int kk = 7; kk >= 0; --kk) row = row * y + g[jj][kk];
                    v = v * x + row;
                }
                sup = std::max(sup, v);
                inf = std::min(inf, v);
            }
        c.tri_ext[3 * k] = sup;
        c.tri_ext[3 * k + 1] = inf;
    }
}

}  // namespace sdgpu

using namespace sdgpu;

extern "C" {

const char* sd_last_error(void) { return g_err.c_str(); }
int sd_abi_version(void) { return SDGPU_ABI_VERSION; }

int sd_create(sd_ctx** out, int device, int precision) {
    return guard([&] {
        if (!out) throw ArgError{"out is NULL"};
        if (precision != SD_FP32 && precision != SD_FP64) throw ArgError{"precision must be SD_FP32 or SD_FP64"};
        int n = 0;
        check_cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) throw ArgError{"device index out of range"};
        auto* c = new sd_ctx;
        c->device = device;
        c->precision = precision;
        {
            DeviceScope ds(device);
            cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
            if (e != cudaSuccess) {
                delete c;
                check_cuda(e, "cudaStreamCreate");
            }
        }
        *out = c;
    });
}

int sd_destroy(sd_ctx* c) {
    return guard([&] {
        if (!c) return;
        {
            DeviceScope ds(c->device);
            if (c->stream) cudaStreamDestroy(c->stream);
            if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
            c->stream = c->copy_stream = nullptr;
            for (auto& pr : c->ev_pairs) c->ev_pool.insert(c->ev_pool.end(), {pr.first, pr.second});
            for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
            for (auto& sl : c->slots)
                for (cudaEvent_t e : {sl.in, sl.done, sl.out})
                    if (e) cudaEventDestroy(e);
            if (c->in_stream) cudaStreamDestroy(c->in_stream);
            if (c->out_stream) cudaStreamDestroy(c->out_stream);
            if (c->aux_stream) cudaStreamDestroy(c->aux_stream);
            if (c->aux_fork) cudaEventDestroy(c->aux_fork);
            if (c->aux_join) cudaEventDestroy(c->aux_join);
        }
        delete c;
    });
}

// mesh.hpp:55-87 validation, then the fp32 rounding of SURVEY 7.
int sd_set_geometry(sd_ctx* c, const double* xyz, int64_t V, const int32_t* sv, const uint8_t* kinds, int64_t N) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (V < 0 || N < 0 || (V > 0 && !xyz) || (N > 0 && (!sv || !kinds))) throw ArgError{"bad geometry arrays"};
        if (V > INT32_MAX) throw ArgError{"too many vertices for int32 indices"};
        std::vector<double> x(xyz, xyz + 3 * V);
        if (c->precision == SD_FP32)
            for (double& v : x) v = double(float(v));
        for (double v : x)
            if (!std::isfinite(v)) throw ArgError{"non-finite vertex coordinate"};
        for (int64_t i = 0; i < N; ++i) {
            if (kinds[i] > SD_TRIANGLE) throw ArgError{"simplex " + std::to_string(i) + ": bad kind"};
            const int nv = kinds[i] + 1;
            for (int a = 0; a < nv; ++a)
                if (sv[3 * i + a] < 0 || sv[3 * i + a] >= V)
                    throw ArgError{"simplex " + std::to_string(i) + ": vertex index " + std::to_string(sv[3 * i + a]) +
                                   " out of range [0, " + std::to_string(V) + ")"};
            for (int a = 0; a < nv; ++a)
                for (int b = a + 1; b < nv; ++b) {
                    const int32_t ia = sv[3 * i + a], ib = sv[3 * i + b];
                    if (ia == ib || (x[3 * ia] == x[3 * ib] && x[3 * ia + 1] == x[3 * ib + 1] &&
                                     x[3 * ia + 2] == x[3 * ib + 2]))
                        throw ArgError{"degenerate simplex " + std::to_string(i)};
                }
            if (kinds[i] == SD_TRIANGLE) {
                const D3 a = {x[3 * sv[3 * i]], x[3 * sv[3 * i] + 1], x[3 * sv[3 * i] + 2]};
                const D3 b = {x[3 * sv[3 * i + 1]], x[3 * sv[3 * i + 1] + 1], x[3 * sv[3 * i + 1] + 2]};
                const D3 cc = {x[3 * sv[3 * i + 2]], x[3 * sv[3 * i + 2] + 1], x[3 * sv[3 * i + 2] + 2]};
                const D3 n = cross3(sub(b, a), sub(cc, a));
                if (std::sqrt(dot3(n, n)) == 0.0) throw ArgError{"degenerate simplex " + std::to_string(i) + " (zero area)"};
            }
        }
        c->xyz.swap(x);
        c->sv.assign(sv, sv + 3 * N);
        c->kind.assign(kinds, kinds + N);
        c->V = V;
        c->N = N;
        c->have_geom = true;
        c->have_weights = false;
        c->exact_ready = false;
        c->have_tree = false;
        c->dtree_ready = false;
        c->sx_tree_ready = c->sx_prim_ready = false;
        c->tree.clear();
    });
}

int sd_set_weights(sd_ctx* c, double A, double sup, int32_t ne, const double* edge_a, int32_t nt,
                   const double* tri_stored, const int32_t* poly_index) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_geom) throw StateError{"set the geometry before the weights"};
        if (ne < 0 || nt < 0 || (ne > 0 && !edge_a) || (nt > 0 && !tri_stored) || (c->N > 0 && !poly_index))
            throw ArgError{"bad weight arrays"};
        if (!(A >= 1.0) || !std::isfinite(sup)) throw ArgError{"WeightSet::A must be >= 1 and sup finite"};
        for (int64_t i = 0; i < c->N; ++i) {
            const int32_t pi = poly_index[i];
            const int k = c->kind[i];
            if (pi < -1 || (k == SD_EDGE && pi >= ne) || (k == SD_TRIANGLE && pi >= nt))
                throw ArgError{"poly_index[" + std::to_string(i) + "] out of range"};
        }
        c->A = A;
        c->sup_wtilde = sup;
        c->edge_a.assign(edge_a, edge_a + 5 * size_t(ne));
        c->tri_stored.assign(tri_stored, tri_stored + 13 * size_t(nt));
        c->poly_index.assign(poly_index, poly_index + c->N);
        set_default_meta(*c);
        c->have_weights = true;
        c->exact_ready = false;
        c->dtree_ready = false;
        c->sx_tree_ready = c->sx_prim_ready = false;
    });
}

int sd_build_weights(sd_ctx* c) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_geom) throw StateError{"set the geometry before building weights"};
        // adjacency + polynomial assignment on the device (adjacency.cu);
        // SDGPU_WEIGHTS_HOST=1 runs the host hash-map pass instead (A/B)
        const char* e = std::getenv("SDGPU_WEIGHTS_HOST");
        WeightTableHost t;
        if (e && *e == '1') {
            t = build_weight_table(c->sv, c->kind, c->V);
        } else {
            DeviceScope ds(c->device);
            t = weight_table_from_assignment(gpu_weight_assignment(*c));
        }
        std::vector<double> ts;
        for (const TriWeight& w : t.tri) ts.insert(ts.end(), w.stored, w.stored + 13);
        c->A = t.A;
        c->sup_wtilde = t.sup;
        c->edge_a = t.edge_a;
        c->tri_stored = ts;
        c->poly_index = t.poly_index;
        c->edge_val = t.edge_val;
        c->edge_ext.clear();
        for (size_t k = 0; k < t.edge_sup.size(); ++k) {
            c->edge_ext.push_back(t.edge_sup[k]);
            c->edge_ext.push_back(t.edge_inf[k]);
        }
        c->tri_val.clear();
        c->tri_ext.clear();
        for (const TriWeight& w : t.tri) {
            c->tri_val.push_back(w.v);
            c->tri_val.push_back(w.e);
            c->tri_ext.push_back(w.sup);
            c->tri_ext.push_back(w.inf);
            c->tri_ext.push_back(0.0);  // residual: not recomputed
        }
        c->have_weights = true;
        c->exact_ready = false;
        c->dtree_ready = false;
        c->sx_tree_ready = c->sx_prim_ready = false;
    });
}

int sd_weights_info(sd_ctx* c, double* A, double* sup, int32_t* ne, int32_t* nt) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_weights) throw StateError{"no weight table"};
        if (A) *A = c->A;
        if (sup) *sup = c->sup_wtilde;
        if (ne) *ne = int32_t(c->edge_a.size() / 5);
        if (nt) *nt = int32_t(c->tri_stored.size() / 13);
    });
}

int sd_export_weights(sd_ctx* c, double* edge_a, double* tri_stored, int32_t* poly_index) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_weights) throw StateError{"no weight table"};
        if (edge_a) std::memcpy(edge_a, c->edge_a.data(), c->edge_a.size() * sizeof(double));
        if (tri_stored) std::memcpy(tri_stored, c->tri_stored.data(), c->tri_stored.size() * sizeof(double));
        if (poly_index) std::memcpy(poly_index, c->poly_index.data(), c->poly_index.size() * sizeof(int32_t));
    });
}

int sd_set_bvh(sd_ctx* c, const sd_bvh_node* nodes, int64_t n) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_geom) throw StateError{"set the geometry before the tree"};
        if (n != (c->N > 0 ? 2 * c->N - 1 : 0) || (n > 0 && !nodes))
            throw ArgError{"tree must have 2N - 1 nodes (one primitive per leaf)"};
        c->tree.assign(nodes, nodes + n);
        c->tree_trusted = false;
        c->have_tree = true;
        c->dtree_ready = false;
        c->sx_tree_ready = c->sx_prim_ready = false;
    });
}

int sd_build_bvh(sd_ctx* c, int method) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_geom) throw StateError{"set the geometry before building a tree"};
        DeviceScope ds(c->device);
        const char* mh = std::getenv("SDGPU_MEDIAN_HOST");
        if (method == SD_BVH_MEDIAN && mh && *mh == '1') tree_build_median_host(*c);
        else if (method == SD_BVH_MEDIAN) tree_build_median_gpu(*c);
        else if (method == SD_BVH_LBVH) tree_build_lbvh(*c);
        else if (method == SD_BVH_AUTO) {
            // both device builders; keep the tree with the smaller surface-area
            // cost sum_internal area / area(root) -- it predicted the faster
            // traversal on every measured workload (tools/tree_cost.py)
            tree_build_median_gpu(*c);
            std::vector<sd_bvh_node> median;
            median.swap(c->tree);
            tree_build_lbvh(*c);
            if (sah_cost(median) < sah_cost(c->tree)) c->tree.swap(median);
            c->dtree_ready = false;
            c->sx_tree_ready = c->sx_prim_ready = false;
        } else {
            throw ArgError{"unknown tree builder"};
        }
        c->have_tree = true;
    });
}

// ------------------------------------------------- reference caches
// SDBV0001 (bvh.hpp:190-236): magic, u64 node count, per node lo[3] hi[3]
// (f64) left right primitive count (i32) diameter (f64) -- exactly the
// 72-byte sd_bvh_node record, so the payload is the node array itself.
static const char kBvhMagic[8] = {'S', 'D', 'B', 'V', '0', '0', '0', '1'};
static const char kWtMagic[8] = {'S', 'D', 'W', 'T', '0', '0', '0', '1'};
static_assert(sizeof(sd_bvh_node) == 72, "SDBV0001 record");

int sd_save_bvh_cache(sd_ctx* c, const char* path) {
    return guard([&] {
        if (!c || !path) throw ArgError{"NULL argument"};
        if (!c->have_tree) throw StateError{"no tree to save"};
        std::ofstream out(path, std::ios::binary);
        if (!out) throw ArgError{std::string("cannot open ") + path + " for writing"};
        out.write(kBvhMagic, 8);
        const uint64_t n = c->tree.size();
        out.write(reinterpret_cast<const char*>(&n), sizeof(n));
        out.write(reinterpret_cast<const char*>(c->tree.data()), std::streamsize(n * sizeof(sd_bvh_node)));
        if (!out) throw ArgError{std::string("write failed: ") + path};
    });
}

int sd_load_bvh_cache(sd_ctx* c, const char* path) {
    return guard([&] {
        if (!c || !path) throw ArgError{"NULL argument"};
        if (!c->have_geom) throw StateError{"set the geometry before the tree"};
        std::ifstream in(path, std::ios::binary);
        if (!in) throw ArgError{std::string("cannot open ") + path};
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kBvhMagic, 8) != 0) throw ArgError{std::string(path) + ": not a BVH cache (bad magic)"};
        uint64_t n = 0;
        in.read(reinterpret_cast<char*>(&n), sizeof(n));
        if (!in || int64_t(n) != (c->N > 0 ? 2 * c->N - 1 : 0))
            throw ArgError{std::string(path) + ": node count does not match the mesh"};
        std::vector<sd_bvh_node> nodes(n);
        in.read(reinterpret_cast<char*>(nodes.data()), std::streamsize(n * sizeof(sd_bvh_node)));
        if (!in) throw ArgError{std::string(path) + ": truncated BVH cache"};
        c->tree.swap(nodes);
        c->tree_trusted = false;
        c->have_tree = true;
        c->dtree_ready = false;
        c->sx_tree_ready = c->sx_prim_ready = false;
    });
}

// SDWT0001 (weights.hpp:700-781): magic, A, sup (f64), u64 counts (edge,
// triangle polynomials, poly_index), per edge valence0 valence1 (i32)
// a[5] sup inf (f64), per triangle v e (i32) stored[13] sup inf residual
// (f64), then poly_index (i32). Little-endian, packed.
int sd_save_weight_cache(sd_ctx* c, const char* path) {
    return guard([&] {
        if (!c || !path) throw ArgError{"NULL argument"};
        if (!c->have_weights) throw StateError{"no weight table to save"};
        std::ofstream out(path, std::ios::binary);
        if (!out) throw ArgError{std::string("cannot open ") + path + " for writing"};
        auto pod = [&](const auto& v) { out.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
        out.write(kWtMagic, 8);
        const uint64_t ne = c->edge_a.size() / 5, nt = c->tri_stored.size() / 13, np = c->poly_index.size();
        pod(c->A);
        pod(c->sup_wtilde);
        pod(ne);
        pod(nt);
        pod(np);
        for (uint64_t k = 0; k < ne; ++k) {
            pod(c->edge_val[2 * k]);
            pod(c->edge_val[2 * k + 1]);
            for (int j = 0; j < 5; ++j) pod(c->edge_a[5 * k + j]);
            pod(c->edge_ext[2 * k]);
            pod(c->edge_ext[2 * k + 1]);
        }
        for (uint64_t k = 0; k < nt; ++k) {
            pod(c->tri_val[2 * k]);
            pod(c->tri_val[2 * k + 1]);
            for (int j = 0; j < 13; ++j) pod(c->tri_stored[13 * k + j]);
            pod(c->tri_ext[3 * k]);
            pod(c->tri_ext[3 * k + 1]);
            pod(c->tri_ext[3 * k + 2]);
        }
        out.write(reinterpret_cast<const char*>(c->poly_index.data()), std::streamsize(np * sizeof(int32_t)));
        if (!out) throw ArgError{std::string("write failed: ") + path};
    });
}

int sd_load_weight_cache(sd_ctx* c, const char* path) {
    return guard([&] {
        if (!c || !path) throw ArgError{"NULL argument"};
        if (!c->have_geom) throw StateError{"set the geometry before the weights"};
        std::ifstream in(path, std::ios::binary);
        if (!in) throw ArgError{std::string("cannot open ") + path};
        auto pod = [&](auto& v) { in.read(reinterpret_cast<char*>(&v), sizeof(v)); };
        char magic[8];
        in.read(magic, 8);
        if (!in || std::memcmp(magic, kWtMagic, 8) != 0)
            throw ArgError{std::string(path) + ": not a weight cache (bad magic)"};
        double A = 1, sup = 1;
        uint64_t ne = 0, nt = 0, np = 0;
        pod(A);
        pod(sup);
        pod(ne);
        pod(nt);
        pod(np);
        if (!in || int64_t(np) != c->N || ne > (uint64_t(1) << 31) || nt > (uint64_t(1) << 31))
            throw ArgError{std::string(path) + ": weight cache does not match the mesh"};
        std::vector<double> ea(5 * ne), ts(13 * nt), eext(2 * ne), text(3 * nt);
        std::vector<int32_t> ev(2 * ne), tv(2 * nt), pi(np);
        for (uint64_t k = 0; k < ne; ++k) {
            pod(ev[2 * k]);
            pod(ev[2 * k + 1]);
            for (int j = 0; j < 5; ++j) pod(ea[5 * k + j]);
            pod(eext[2 * k]);
            pod(eext[2 * k + 1]);
        }
        for (uint64_t k = 0; k < nt; ++k) {
            pod(tv[2 * k]);
            pod(tv[2 * k + 1]);
            for (int j = 0; j < 13; ++j) pod(ts[13 * k + j]);
            pod(text[3 * k]);
            pod(text[3 * k + 1]);
            pod(text[3 * k + 2]);
        }
        in.read(reinterpret_cast<char*>(pi.data()), std::streamsize(np * sizeof(int32_t)));
        if (!in) throw ArgError{std::string(path) + ": truncated weight cache"};
        const int rc = sd_set_weights(c, A, sup, int32_t(ne), ea.data(), int32_t(nt), ts.data(), pi.data());
        if (rc != SD_OK) throw ArgError{sd_last_error()};
        c->edge_val = ev;
        c->edge_ext = eext;
        c->tri_val = tv;
        c->tri_ext = text;
    });
}

int sd_bvh_size(sd_ctx* c, int64_t* n) {
    return guard([&] {
        if (!c || !n) throw ArgError{"NULL argument"};
        *n = int64_t(c->tree.size());
    });
}

int sd_export_bvh(sd_ctx* c, sd_bvh_node* out, int64_t cap) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!c->have_tree) throw StateError{"no tree"};
        if (cap < int64_t(c->tree.size()) || (!out && !c->tree.empty())) throw ArgError{"output too small"};
        std::memcpy(out, c->tree.data(), c->tree.size() * sizeof(sd_bvh_node));
    });
}

int sd_query_points_device(sd_ctx* c, const void* q, int64_t Q, const sd_params* p, int mode, const sd_outputs* o,
                           void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (Q < 0 || (Q > 0 && (!q || !o || !o->d_hat))) throw ArgError{"bad query / output pointers"};
        DeviceScope ds(c->device);
        FinalizeOut out{o->d_hat, o->grad, o->c, o->grad_c, o->leaves, o->far_field, o->decision_hash};
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (c->precision == SD_FP32) dispatch<float>(*c, static_cast<const float*>(q), Q, *p, mode, out, st);
        else dispatch<double>(*c, static_cast<const double*>(q), Q, *p, mode, out, st);
    });
}

constexpr int kShardChunk = 1024;  // max packets per round-robin chunk of sd_query_points_device_shard

int sd_query_points_device_shard(sd_ctx* c, const void* q, int64_t Q, const sd_params* p, const sd_outputs* o,
                                 int32_t world, int32_t rank, void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, SD_BVH);
        if (world < 1 || rank < 0 || rank >= world) throw ArgError{"bad world / rank"};
        if (Q < 0 || (Q > 0 && (!q || !o || !o->d_hat))) throw ArgError{"bad query / output pointers"};
        if (!(p->beta > 0.0)) throw ArgError{"sd_query_points_device_shard is the tree path: beta must be > 0"};
        DeviceScope ds(c->device);
        FinalizeOut out{o->d_hat, o->grad, o->c, o->grad_c, o->leaves, o->far_field, o->decision_hash};
        out.pk_world = world;
        out.pk_rank = rank;
        // chunks of packets dealt round robin: spatial locality within a
        // chunk (the rank's node working set stays regional), balance across
        // at least 16 chunks per rank; SDGPU_SHARD_CHUNK overrides.
        // tools/scaling_projection.py (cfg4, each share timed alone on one
        // GPU): 8 ranks 4.51x (1 packet per chunk) / 5.03x (64) / 5.33x
        // (1024); cost-balanced contiguous blocks 3.94x
        const char* ch = std::getenv("SDGPU_SHARD_CHUNK");
        const int64_t npk = (Q + 31) / 32;
        out.pk_chunk = ch && *ch ? std::max(1, std::atoi(ch))
                                 : std::max<int64_t>(1, std::min<int64_t>(kShardChunk, npk / (int64_t(world) * 16)));
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (c->precision == SD_FP32) dispatch<float>(*c, static_cast<const float*>(q), Q, *p, SD_BVH, out, st);
        else dispatch<double>(*c, static_cast<const double*>(q), Q, *p, SD_BVH, out, st);
    });
}

int sd_query_points(sd_ctx* c, const double* q, int64_t Q, const sd_params* p, int mode, const sd_outputs* o) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (Q < 0 || (Q > 0 && (!q || !o || !o->d_hat))) throw ArgError{"bad query / output pointers"};
        if (Q == 0) return;
        DeviceScope ds(c->device);
        cudaStream_t st = c->stream;
        double* qd = static_cast<double*>(c->qd.ensure(size_t(Q) * 3 * sizeof(double)));
        FinalizeOut out;
        out.d_hat = static_cast<double*>(c->out_d.ensure(size_t(Q) * sizeof(double)));
        if (o->grad) out.grad = static_cast<double*>(c->out_g.ensure(size_t(Q) * 3 * sizeof(double)));
        if (o->c) out.c = static_cast<double*>(c->out_c.ensure(size_t(Q) * sizeof(double)));
        if (o->grad_c) out.grad_c = static_cast<double*>(c->out_gc.ensure(size_t(Q) * 3 * sizeof(double)));
        if (o->leaves) out.leaves = static_cast<int64_t*>(c->out_l.ensure(size_t(Q) * sizeof(int64_t)));
        if (o->far_field) out.far_field = static_cast<int64_t*>(c->out_f.ensure(size_t(Q) * sizeof(int64_t)));
        if (o->decision_hash) out.hash = static_cast<uint64_t*>(c->out_h.ensure(size_t(Q) * sizeof(uint64_t)));
        float* qf = c->precision == SD_FP32 ? static_cast<float*>(c->qT.ensure(size_t(Q) * 3 * sizeof(float))) : nullptr;
        // Optional chunk pipeline (SDGPU_PIPELINE=1: 4 chunks, =k: k chunks;
        // batches >= 2^17): every
        // chunk's H2D is queued on the copy stream up front, chunk k computes
        // on the context stream once its queries landed, and its results go
        // back on the copy stream while chunk k+1 computes. Off by default:
        // on cfg2 the transfers are ~4 % of the step and four quarter-size
        // exact launches lose more than the overlap gains (e2e 6.6e11 vs
        // 7.05e11 pair-evals/s unpipelined; tools/e2e_chunks.py medians: 1 chunk
        // 7.18 ms, 2 chunks 7.25 ms, 4 chunks 7.88 ms).
        const char* pe = std::getenv("SDGPU_PIPELINE");
        const int want = pe && *pe ? std::atoi(pe) : 0;  // 1: four chunks, k >= 2: k chunks
        const int chunks = (Q >= (int64_t(1) << 17) && want > 0) ? (want == 1 ? 4 : std::min(want, 16)) : 1;
        cudaStream_t cs = st;
        if (chunks > 1) {
            if (!c->copy_stream) check_cuda(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
            cs = c->copy_stream;
        }
        std::vector<std::unique_ptr<ScopedEvent>> evs;
        std::vector<cudaEvent_t> ev;
        for (int k = 0; k < 2 * chunks; ++k) {
            evs.push_back(std::make_unique<ScopedEvent>(cudaEventDisableTiming));
            ev.push_back(*evs.back());
        }
        const int64_t per = (Q + chunks - 1) / chunks;
        for (int k = 0; k < chunks; ++k) {
            const int64_t off = k * per, n = std::min(Q, off + per) - off;
            check_cuda(cudaMemcpyAsync(qd + 3 * off, q + 3 * off, size_t(n) * 3 * sizeof(double), cudaMemcpyHostToDevice,
                                       cs),
                       "H2D queries");
            check_cuda(cudaEventRecord(ev[2 * k], cs), "event");
        }
        int64_t launches = 0;
        auto shift = [](auto* ptr, int64_t by) { return ptr ? ptr + by : ptr; };
        for (int k = 0; k < chunks; ++k) {
            const int64_t off = k * per, n = std::min(Q, off + per) - off;
            check_cuda(cudaStreamWaitEvent(st, ev[2 * k], 0), "wait");
            FinalizeOut oc = out;
            oc.d_hat = shift(out.d_hat, off);
            oc.grad = shift(out.grad, 3 * off);
            oc.c = shift(out.c, off);
            oc.grad_c = shift(out.grad_c, 3 * off);
            oc.leaves = shift(out.leaves, off);
            oc.far_field = shift(out.far_field, off);
            oc.hash = shift(out.hash, off);
            if (qf) {
                convert_queries<float><<<unsigned((3 * n + 255) / 256), 256, 0, st>>>(qd + 3 * off, qf + 3 * off, 3 * n);
                check_cuda(cudaGetLastError(), "convert queries");
                dispatch<float>(*c, qf + 3 * off, n, *p, mode, oc, st);
                ++launches;
            } else {
                dispatch<double>(*c, qd + 3 * off, n, *p, mode, oc, st);
            }
            launches += c->last_launches;
            check_cuda(cudaEventRecord(ev[2 * k + 1], st), "event");
            check_cuda(cudaStreamWaitEvent(cs, ev[2 * k + 1], 0), "wait");
            auto d2h = [&](void* dst, const void* src, size_t bytes) {
                if (dst) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, cs), "D2H results");
            };
            d2h(o->d_hat ? o->d_hat + off : nullptr, oc.d_hat, size_t(n) * sizeof(double));
            d2h(o->grad ? o->grad + 3 * off : nullptr, oc.grad, size_t(n) * 3 * sizeof(double));
            d2h(o->c ? o->c + off : nullptr, oc.c, size_t(n) * sizeof(double));
            d2h(o->grad_c ? o->grad_c + 3 * off : nullptr, oc.grad_c, size_t(n) * 3 * sizeof(double));
            d2h(o->leaves ? o->leaves + off : nullptr, oc.leaves, size_t(n) * sizeof(int64_t));
            d2h(o->far_field ? o->far_field + off : nullptr, oc.far_field, size_t(n) * sizeof(int64_t));
            d2h(o->decision_hash ? o->decision_hash + off : nullptr, oc.hash, size_t(n) * sizeof(uint64_t));
        }
        check_cuda(cudaStreamSynchronize(cs), "query");
        check_cuda(cudaStreamSynchronize(st), "query");
        c->last_launches = launches;
    });
}

int sd_finalize_device(sd_ctx* c, const double* cs, const double* gc, int64_t Q, const sd_params* p, double* d_hat,
                       double* grad, void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        if (Q < 0 || (Q > 0 && (!cs || !gc || !d_hat))) throw ArgError{"bad pointers"};
        DeviceScope ds(c->device);
        check_cuda(launch_finalize_sums(cs, gc, Q, p->alpha, p->epsilon, d_hat, grad, static_cast<cudaStream_t>(stream)),
                   "finalize");
        c->last_launches = Q > 0 ? 1 : 0;
    });
}

int sd_scatter_partials(sd_ctx* c, const double* cs, const double* gc, int64_t Q, double* const* peer_bufs,
                        int32_t world, int32_t rank, int64_t q_per_owner, void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (Q < 0 || world < 1 || rank < 0 || rank >= world || q_per_owner <= 0 || q_per_owner * world < Q ||
            (Q > 0 && (!cs || !gc || !peer_bufs)))
            throw ArgError{"bad exchange arguments"};
        DeviceScope ds(c->device);
        check_cuda(launch_scatter_partials(cs, gc, Q, peer_bufs, rank, q_per_owner, static_cast<cudaStream_t>(stream)),
                   "scatter partials");
        c->last_launches = Q > 0 ? 1 : 0;
    });
}

int sd_query_points_scatter(sd_ctx* c, const void* q, int64_t Q, const sd_params* p, int mode,
                            double* const* peer_bufs, int32_t world, int32_t rank, int64_t q_per_owner,
                            int64_t* leaves, int64_t* far_field, void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (Q < 0 || world < 1 || rank < 0 || rank >= world || q_per_owner <= 0 || q_per_owner * world < Q ||
            (Q > 0 && (!q || !peer_bufs)))
            throw ArgError{"bad exchange arguments"};
        if (Q == 0) return;
        DeviceScope ds(c->device);
        FinalizeOut out;
        out.peers = peer_bufs;
        out.peer_rank = rank;
        out.peer_qown = q_per_owner;
        out.leaves = leaves;
        out.far_field = far_field;
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        if (c->precision == SD_FP32) dispatch<float>(*c, static_cast<const float*>(q), Q, *p, mode, out, st);
        else dispatch<double>(*c, static_cast<const double*>(q), Q, *p, mode, out, st);
    });
}

int sd_reduce_owned(sd_ctx* c, const double* sbuf, int64_t q_per_owner, int64_t n_owned, int32_t world,
                    const sd_params* p, double* d_hat, double* grad, void* stream) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        if (q_per_owner <= 0 || n_owned < 0 || n_owned > q_per_owner || world < 1 || (n_owned > 0 && (!sbuf || !d_hat)))
            throw ArgError{"bad exchange arguments"};
        DeviceScope ds(c->device);
        check_cuda(launch_reduce_owned(sbuf, q_per_owner, n_owned, world, p->alpha, p->epsilon, d_hat, grad,
                                       static_cast<cudaStream_t>(stream)),
                   "reduce owned");
        c->last_launches = n_owned > 0 ? 1 : 0;
    });
}

int sd_mesh_dist_points(sd_ctx* c, const double* qxyz, int64_t Vq, const int32_t* qpoints, int64_t Nq,
                        const sd_params* p, double alpha_q, int mode, double* d_hat, double* vertex_grads,
                        double* per_primitive) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (!(alpha_q > 0) || !std::isfinite(alpha_q)) throw ArgError{"alpha_q must be positive and finite"};
        if (Vq < 0 || (Vq > 0 && !qxyz) || !d_hat || (Vq > 0 && !vertex_grads)) throw ArgError{"bad query mesh arrays"};
        if (!qpoints) Nq = Vq;
        if (Nq < 0) throw ArgError{"bad point count"};
        std::vector<double> q(size_t(Nq) * 3);
        for (int64_t j = 0; j < Nq; ++j) {
            const int64_t v = qpoints ? qpoints[j] : j;
            if (v < 0 || v >= Vq) throw ArgError{"query point " + std::to_string(j) + ": vertex index out of range"};
            for (int a = 0; a < 3; ++a) q[3 * j + a] = qxyz[3 * v + a];
        }
        DeviceScope ds(c->device);
        cudaStream_t st = c->stream;
        int64_t launches = 0;
        FinalizeOut out;
        out.d_hat = static_cast<double*>(c->out_d.ensure(size_t(std::max<int64_t>(Nq, 1)) * sizeof(double)));
        out.grad = static_cast<double*>(c->out_g.ensure(size_t(std::max<int64_t>(Nq, 1)) * 3 * sizeof(double)));
        if (Nq > 0) {
            double* qd = static_cast<double*>(c->qd.ensure(q.size() * sizeof(double)));
            check_cuda(cudaMemcpyAsync(qd, q.data(), q.size() * sizeof(double), cudaMemcpyHostToDevice, st), "H2D");
            if (c->precision == SD_FP32) {
                float* qf = static_cast<float*>(c->qT.ensure(q.size() * sizeof(float)));
                convert_queries<float><<<unsigned((3 * Nq + 255) / 256), 256, 0, st>>>(qd, qf, 3 * Nq);
                check_cuda(cudaGetLastError(), "convert queries");
                dispatch<float>(*c, qf, Nq, *p, mode, out, st);
            } else {
                dispatch<double>(*c, qd, Nq, *p, mode, out, st);
            }
            launches += c->last_launches;
        }
        int32_t* vidx = nullptr;
        if (qpoints && Nq > 0) {
            vidx = static_cast<int32_t*>(c->out_l.ensure(size_t(Nq) * sizeof(int32_t)));
            check_cuda(cudaMemcpyAsync(vidx, qpoints, size_t(Nq) * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
        }
        const size_t wb = mesh_reduce_work_bytes(Nq);
        double* work = static_cast<double*>(c->tmp2.ensure(wb));
        double* vg = static_cast<double*>(c->out_gc.ensure(size_t(std::max<int64_t>(Vq, 1)) * 3 * sizeof(double)));
        double* dd = static_cast<double*>(c->out_c.ensure(sizeof(double) * 2));
        check_cuda(launch_mesh_reduce(out.d_hat, out.grad, Nq, vidx, 1, Vq, alpha_q, p->epsilon, work, wb, vg, dd,
                                      launches, st),
                   "mesh reduction");
        check_cuda(cudaMemcpyAsync(d_hat, dd, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        if (Vq > 0)
            check_cuda(cudaMemcpyAsync(vertex_grads, vg, size_t(Vq) * 3 * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "D2H");
        if (per_primitive && Nq > 0)
            check_cuda(cudaMemcpyAsync(per_primitive, out.d_hat, size_t(Nq) * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "D2H");
        check_cuda(cudaStreamSynchronize(st), "mesh dist");
        c->last_launches = launches;
    });
}

static void query_outputs(Ctx& c, int64_t Q, const sd_outputs* o, FinalizeOut& out) {
    out.d_hat = static_cast<double*>(c.out_d.ensure(size_t(Q) * sizeof(double)));
    if (o->grad) out.grad = static_cast<double*>(c.out_g.ensure(size_t(Q) * 3 * sizeof(double)));
    if (o->c) out.c = static_cast<double*>(c.out_c.ensure(size_t(Q) * sizeof(double)));
    if (o->grad_c) out.grad_c = static_cast<double*>(c.out_gc.ensure(size_t(Q) * 3 * sizeof(double)));
    if (o->leaves) out.leaves = static_cast<int64_t*>(c.out_l.ensure(size_t(Q) * sizeof(int64_t)));
    if (o->far_field) out.far_field = static_cast<int64_t*>(c.out_f.ensure(size_t(Q) * sizeof(int64_t)));
    if (o->decision_hash) out.hash = static_cast<uint64_t*>(c.out_h.ensure(size_t(Q) * sizeof(uint64_t)));
}

// corners / dims -> device (c.qgeom, c.qdim), validated
static void upload_simplices(Ctx& c, const double* corners, const int32_t* dims, int64_t Q, cudaStream_t st) {
    for (int64_t i = 0; i < Q; ++i)
        if (dims[i] < 0 || dims[i] > 2) throw ArgError{"query " + std::to_string(i) + ": dim must be 0, 1 or 2"};
    double* qg = static_cast<double*>(c.qgeom.ensure(size_t(Q) * 9 * sizeof(double)));
    int32_t* qd = static_cast<int32_t*>(c.qdim.ensure(size_t(Q) * sizeof(int32_t)));
    check_cuda(cudaMemcpyAsync(qg, corners, size_t(Q) * 9 * sizeof(double), cudaMemcpyHostToDevice, st), "H2D corners");
    check_cuda(cudaMemcpyAsync(qd, dims, size_t(Q) * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D dims");
}

int sd_query_simplices(sd_ctx* c, const double* corners, const int32_t* dims, int64_t Q, const sd_params* p, int mode,
                       const sd_outputs* o) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (Q < 0 || (Q > 0 && (!corners || !dims || !o || !o->d_hat))) throw ArgError{"bad query / output pointers"};
        if (Q == 0) return;
        DeviceScope ds(c->device);
        cudaStream_t st = c->stream;
        upload_simplices(*c, corners, dims, Q, st);
        FinalizeOut out;
        query_outputs(*c, Q, o, out);
        simplex_query(*c, c->qgeom.as<double>(), c->qdim.as<int32_t>(), Q, *p, mode, out, st);
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
            if (dst) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), "D2H results");
        };
        d2h(o->d_hat, out.d_hat, size_t(Q) * sizeof(double));
        d2h(o->grad, out.grad, size_t(Q) * 3 * sizeof(double));
        d2h(o->c, out.c, size_t(Q) * sizeof(double));
        d2h(o->grad_c, out.grad_c, size_t(Q) * 3 * sizeof(double));
        d2h(o->leaves, out.leaves, size_t(Q) * sizeof(int64_t));
        d2h(o->far_field, out.far_field, size_t(Q) * sizeof(int64_t));
        d2h(o->decision_hash, out.hash, size_t(Q) * sizeof(uint64_t));
        check_cuda(cudaStreamSynchronize(st), "query simplices");
    });
}

int sd_mesh_dist(sd_ctx* c, const double* qxyz, int64_t Vq, const int32_t* qsimplices, const uint8_t* qkinds,
                 int64_t Nq, const sd_params* p, double alpha_q, int mode, double* d_hat, double* vertex_grads,
                 double* per_primitive) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        check_params(p);
        check_ready(*c, mode);
        if (!(alpha_q > 0) || !std::isfinite(alpha_q)) throw ArgError{"alpha_q must be positive and finite"};
        if (Vq < 0 || Nq < 0 || (Vq > 0 && !qxyz) || (Nq > 0 && (!qsimplices || !qkinds)) || !d_hat ||
            (Vq > 0 && !vertex_grads))
            throw ArgError{"bad query mesh arrays"};
        bool points_only = true;
        std::vector<int32_t> sv(size_t(Nq) * 3, -1), pts(static_cast<size_t>(Nq));
        std::vector<double> corners(size_t(Nq) * 9, 0.0);
        std::vector<int32_t> dims(static_cast<size_t>(Nq));
        for (int64_t j = 0; j < Nq; ++j) {
            const int kind = qkinds[j];
            if (kind > SD_TRIANGLE) throw ArgError{"query simplex " + std::to_string(j) + ": bad kind"};
            points_only = points_only && kind == SD_POINT;
            dims[j] = kind;
            for (int k = 0; k <= kind; ++k) {
                const int32_t v = qsimplices[3 * j + k];
                if (v < 0 || v >= Vq)
                    throw ArgError{"query simplex " + std::to_string(j) + ": vertex index out of range"};
                sv[3 * j + k] = v;
                for (int a = 0; a < 3; ++a) corners[9 * j + 3 * k + a] = qxyz[3 * size_t(v) + a];
            }
            pts[j] = sv[3 * j];
        }
        if (points_only) {
            const int rc = sd_mesh_dist_points(c, qxyz, Vq, pts.data(), Nq, p, alpha_q, mode, d_hat, vertex_grads,
                                               per_primitive);
            if (rc != SD_OK) throw ArgError{sd_last_error()};
            return;
        }
        DeviceScope ds(c->device);
        cudaStream_t st = c->stream;
        int64_t launches = 0;
        upload_simplices(*c, corners.data(), dims.data(), Nq, st);
        FinalizeOut out;
        out.d_hat = static_cast<double*>(c->out_d.ensure(size_t(Nq) * sizeof(double)));
        out.grad = static_cast<double*>(c->out_g.ensure(size_t(Nq) * 3 * sizeof(double)));
        simplex_query(*c, c->qgeom.as<double>(), c->qdim.as<int32_t>(), Nq, *p, mode, out, st);
        launches += c->last_launches;
        int32_t* vidx = static_cast<int32_t*>(c->out_l.ensure(sv.size() * sizeof(int32_t)));
        check_cuda(cudaMemcpyAsync(vidx, sv.data(), sv.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st), "H2D");
        const size_t wb = mesh_reduce_work_bytes(Nq);
        double* work = static_cast<double*>(c->tmp2.ensure(wb));
        double* vg = static_cast<double*>(c->out_gc.ensure(size_t(std::max<int64_t>(Vq, 1)) * 3 * sizeof(double)));
        double* dd = static_cast<double*>(c->out_c.ensure(sizeof(double) * 2));
        check_cuda(launch_mesh_reduce(out.d_hat, out.grad, Nq, vidx, 3, Vq, alpha_q, p->epsilon, work, wb, vg, dd,
                                      launches, st),
                   "mesh reduction");
        check_cuda(cudaMemcpyAsync(d_hat, dd, sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
        if (Vq > 0)
            check_cuda(cudaMemcpyAsync(vertex_grads, vg, size_t(Vq) * 3 * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "D2H");
        if (per_primitive)
            check_cuda(cudaMemcpyAsync(per_primitive, out.d_hat, size_t(Nq) * sizeof(double), cudaMemcpyDeviceToHost, st),
                       "D2H");
        check_cuda(cudaStreamSynchronize(st), "mesh dist");
        c->last_launches = launches;
    });
}

int sd_render(sd_ctx* c, const sd_params* p, int mode, const sd_render_config* cfg, uint8_t* rgb, double* hit_t,
              int64_t* stats, double* seconds) {
    return guard([&] {
        if (!c || !cfg || !rgb || !hit_t) throw ArgError{"NULL argument"};
        check_params(p);
        check_ready(*c, mode);
        if (cfg->width <= 0 || cfg->height <= 0 || int64_t(cfg->width) * cfg->height > (int64_t(1) << 28))
            throw ArgError{"bad image size"};
        if (cfg->max_steps < 0 || !(cfg->fov_deg > 0 && cfg->fov_deg < 180)) throw ArgError{"bad render config"};
        DeviceScope ds(c->device);
        render_impl(*c, *p, mode, *cfg, rgb, hit_t, stats, seconds);
    });
}

int sd_grid_benchmark(sd_ctx* c, const sd_params* p, int mode, int32_t n, double* d_hat, int64_t* leaves,
                      int64_t* far_field, double* seconds) {
    return guard([&] {
        if (!c || !d_hat) throw ArgError{"NULL argument"};
        check_params(p);
        check_ready(*c, mode);
        if (n <= 0 || n > 512) throw ArgError{"resolution must be in 1..512"};
        DeviceScope ds(c->device);
        grid_impl(*c, *p, mode, n, d_hat, leaves, far_field, seconds);
    });
}

int sd_write_ppm(const uint8_t* rgb, int32_t w, int32_t h, const char* path) {
    return guard([&] {
        if (!rgb || !path || w < 0 || h < 0) throw ArgError{"bad arguments"};
        std::ofstream out(path, std::ios::binary);
        if (!out) throw ArgError{std::string("cannot open ") + path + " for writing"};
        out << "P6\n" << w << " " << h << "\n255\n";
        out.write(reinterpret_cast<const char*>(rgb), std::streamsize(size_t(w) * h * 3));
        if (!out) throw ArgError{std::string("write failed: ") + path};
    });
}

int sd_write_png(const uint8_t* rgb, int32_t w, int32_t h, const char* path) {
    return guard([&] {
        if (!rgb || !path || w < 0 || h < 0) throw ArgError{"bad arguments"};
        std::ofstream out(path, std::ios::binary);
        if (!out) throw ArgError{std::string("cannot open ") + path + " for writing"};
        auto chunk = [&](const char type[4], const uint8_t* data, uint32_t len) {
            auto be32 = [&](uint32_t v) {
                const uint8_t b[4] = {uint8_t(v >> 24), uint8_t(v >> 16), uint8_t(v >> 8), uint8_t(v)};
                out.write(reinterpret_cast<const char*>(b), 4);
            };
            be32(len);
            out.write(type, 4);
            if (len) out.write(reinterpret_cast<const char*>(data), len);
            uLong crc = crc32(0L, Z_NULL, 0);
            crc = crc32(crc, reinterpret_cast<const Bytef*>(type), 4);
            if (len) crc = crc32(crc, data, len);
            be32(uint32_t(crc));
        };
        static const uint8_t sig[8] = {137, 80, 78, 71, 13, 10, 26, 10};
        out.write(reinterpret_cast<const char*>(sig), 8);
        uint8_t ihdr[13] = {uint8_t(uint32_t(w) >> 24), uint8_t(uint32_t(w) >> 16), uint8_t(uint32_t(w) >> 8),
                            uint8_t(w), uint8_t(uint32_t(h) >> 24), uint8_t(uint32_t(h) >> 16),
                            uint8_t(uint32_t(h) >> 8), uint8_t(h), 8, 2, 0, 0, 0};
        chunk("IHDR", ihdr, 13);
        std::vector<uint8_t> raw;
        raw.reserve(size_t(h) * (1 + 3 * size_t(w)));
        for (int y = 0; y < h; ++y) {
            raw.push_back(0);
            raw.insert(raw.end(), rgb + 3 * size_t(y) * w, rgb + 3 * size_t(y + 1) * w);
        }
        uLongf comp_len = compressBound(uLong(raw.size()));
        std::vector<uint8_t> comp(comp_len);
        if (compress2(comp.data(), &comp_len, raw.data(), uLong(raw.size()), 6) != Z_OK)
            throw ArgError{std::string("zlib compression failed for ") + path};
        chunk("IDAT", comp.data(), uint32_t(comp_len));
        chunk("IEND", nullptr, 0);
        if (!out) throw ArgError{std::string("write failed: ") + path};
    });
}

int sd_write_grid_csv(const double* d, const int64_t* leaves, const int64_t* far, int32_t n, const double* slab,
                      const char* path) {
    return guard([&] {
        if (!d || !leaves || !far || !slab || !path || n <= 0) throw ArgError{"bad arguments"};
        std::ofstream out(path);
        if (!out) throw ArgError{std::string("cannot open ") + path + " for writing"};
        out << "voxel_index,d_hat,leaves_visited,far_field,slab_time_s\n";
        char buf[160];
        const size_t n3 = size_t(n) * n * n;
        for (size_t idx = 0; idx < n3; ++idx) {
            const int k = int(idx / (size_t(n) * n));
            std::snprintf(buf, sizeof buf, "%zu,%.17g,%lld,%lld,%.6g\n", idx, d[idx], static_cast<long long>(leaves[idx]),
                          static_cast<long long>(far[idx]), slab[k]);
            out << buf;
        }
        if (!out) throw ArgError{std::string("write failed: ") + path};
    });
}

int sd_query_points_async(sd_ctx* c, const double* q, int64_t Q, const sd_params* p, int mode, const sd_outputs* o,
                          int64_t* ticket) {
    return guard([&] {
        if (!c || !ticket) throw ArgError{"NULL argument"};
        check_params(p);
        check_ready(*c, mode);
        if (Q < 0 || (Q > 0 && (!q || !o || !o->d_hat))) throw ArgError{"bad query / output pointers"};
        DeviceScope ds(c->device);
        if (!c->in_stream) {
            check_cuda(cudaStreamCreateWithFlags(&c->in_stream, cudaStreamNonBlocking), "stream");
            check_cuda(cudaStreamCreateWithFlags(&c->out_stream, cudaStreamNonBlocking), "stream");
            for (auto& sl : c->slots)
                for (cudaEvent_t* e : {&sl.in, &sl.done, &sl.out})
                    check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
        }
        Ctx::AsyncSlot& sl = c->slots[c->next_ticket % 2];
        // the slot's previous batch has left the device (its buffers are free)
        if (sl.ticket >= 0) check_cuda(cudaEventSynchronize(sl.out), "wait slot");
        sl.ticket = c->next_ticket;
        *ticket = c->next_ticket++;
        if (Q == 0) {
            check_cuda(cudaEventRecord(sl.out, c->out_stream), "event");
            return;
        }
        cudaStream_t st = c->stream;
        double* qd = static_cast<double*>(sl.qd.ensure(size_t(Q) * 3 * sizeof(double)));
        check_cuda(cudaMemcpyAsync(qd, q, size_t(Q) * 3 * sizeof(double), cudaMemcpyHostToDevice, c->in_stream),
                   "H2D queries");
        check_cuda(cudaEventRecord(sl.in, c->in_stream), "event");
        check_cuda(cudaStreamWaitEvent(st, sl.in, 0), "wait");
        FinalizeOut out;
        out.d_hat = static_cast<double*>(sl.d.ensure(size_t(Q) * sizeof(double)));
        if (o->grad) out.grad = static_cast<double*>(sl.g.ensure(size_t(Q) * 3 * sizeof(double)));
        if (o->c) out.c = static_cast<double*>(sl.c.ensure(size_t(Q) * sizeof(double)));
        if (o->grad_c) out.grad_c = static_cast<double*>(sl.gc.ensure(size_t(Q) * 3 * sizeof(double)));
        if (o->leaves) out.leaves = static_cast<int64_t*>(sl.l.ensure(size_t(Q) * sizeof(int64_t)));
        if (o->far_field) out.far_field = static_cast<int64_t*>(sl.f.ensure(size_t(Q) * sizeof(int64_t)));
        if (o->decision_hash) out.hash = static_cast<uint64_t*>(sl.h.ensure(size_t(Q) * sizeof(uint64_t)));
        // the evaluation itself (stream-ordered after the previous batch's,
        // so the shared scratch -- converted queries, sort, partials -- is free)
        if (c->precision == SD_FP32) {
            float* qf = static_cast<float*>(c->qT.ensure(size_t(Q) * 3 * sizeof(float)));
            convert_queries<float><<<unsigned((3 * Q + 255) / 256), 256, 0, st>>>(qd, qf, 3 * Q);
            check_cuda(cudaGetLastError(), "convert queries");
            dispatch<float>(*c, qf, Q, *p, mode, out, st);
            c->last_launches += 1;
        } else {
            dispatch<double>(*c, qd, Q, *p, mode, out, st);
        }
        check_cuda(cudaEventRecord(sl.done, st), "event");
        check_cuda(cudaStreamWaitEvent(c->out_stream, sl.done, 0), "wait");
        auto d2h = [&](void* dst, const void* src, size_t bytes) {
            if (dst) check_cuda(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->out_stream), "D2H results");
        };
        d2h(o->d_hat, out.d_hat, size_t(Q) * sizeof(double));
        d2h(o->grad, out.grad, size_t(Q) * 3 * sizeof(double));
        d2h(o->c, out.c, size_t(Q) * sizeof(double));
        d2h(o->grad_c, out.grad_c, size_t(Q) * 3 * sizeof(double));
        d2h(o->leaves, out.leaves, size_t(Q) * sizeof(int64_t));
        d2h(o->far_field, out.far_field, size_t(Q) * sizeof(int64_t));
        d2h(o->decision_hash, out.hash, size_t(Q) * sizeof(uint64_t));
        check_cuda(cudaEventRecord(sl.out, c->out_stream), "event");
    });
}

int sd_query_wait(sd_ctx* c, int64_t ticket) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        DeviceScope ds(c->device);
        for (auto& sl : c->slots)
            if (sl.ticket >= 0 && (ticket < 0 || sl.ticket == ticket))
                check_cuda(cudaEventSynchronize(sl.out), "wait batch");
    });
}

int sd_set_exact_pruning(sd_ctx* c, double bits) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        if (!(bits >= 0) || !std::isfinite(bits)) throw ArgError{"pruning threshold must be >= 0 bits and finite"};
        if (bits > 0 && bits < 24) throw ArgError{"pruning threshold below 24 bits would show in the fp32 results"};
        c->exact_prune_bits = bits;
    });
}

int sd_set_kernel_timing(sd_ctx* c, int on) {
    return guard([&] {
        if (!c) throw ArgError{"ctx is NULL"};
        c->timing = on != 0;
    });
}

int sd_kernel_times(sd_ctx* c, double* ms, int64_t cap, int64_t* n) {
    return guard([&] {
        if (!c || !n) throw ArgError{"NULL argument"};
        DeviceScope ds(c->device);
        const int64_t k = int64_t(c->ev_pairs.size());
        *n = k;
        if (!ms) return;  // count only
        for (int64_t i = 0; i < k; ++i) {
            auto [a, b] = c->ev_pairs[size_t(i)];
            check_cuda(cudaEventSynchronize(b), "cudaEventSynchronize");
            float t = 0.f;
            check_cuda(cudaEventElapsedTime(&t, a, b), "cudaEventElapsedTime");
            if (i < cap) ms[i] = double(t);
            c->ev_pool.push_back(a);
            c->ev_pool.push_back(b);
        }
        c->ev_pairs.clear();
    });
}

int sd_last_launch_count(sd_ctx* c, int64_t* n) {
    return guard([&] {
        if (!c || !n) throw ArgError{"NULL argument"};
        *n = c->last_launches;
    });
}

}  // extern "C"
