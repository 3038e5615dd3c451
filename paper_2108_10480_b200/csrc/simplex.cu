// simplex.cu -- query SIMPLICES (points, edges, triangles) instead of query
// points: the reference's general smooth_min_dist(mesh, bvh, ws, g, params)
// and smooth_min_dist_flat(mesh, ws, g, params) (smooth.hpp:166-198) for a
// batch of SimplexGeom g, and the inner evaluations of smooth_mesh_dist
// (smooth.hpp:212-255) for edge / triangle query meshes.
//
// Geometry restated from /root/reference/proj/include/smoothdist:
//   closest_segment_segment   exact.hpp:110-141
//   simplex_distance_qp       exact.hpp:158-313 (face enumeration; the 3x3
//                             solve restates Eigen's cofactor determinant /
//                             inverse from its published algorithm)
//   simplex_distance          exact.hpp:342-367
//   box_primitive_proximity   bvh.hpp:113-180 (separating-halfspace count)
//   leaf / far-field terms    smooth.hpp:51-75 (far term: g(lambda) - y_B)
//
// Everything here is fp64 and this file is compiled with -fmad=false: every
// +, -, *, / and sqrt rounds once, in the reference's operation order, so
// the Barnes-Hut admissibility decisions (box distance vs beta) are
// bit-identical to the oracle compiled with -ffp-contract=off, with no fp32
// fast path and no re-check band. Term sums go through the same log2-domain
// accumulator as the point path (explicit fma() calls still fuse).
//
// Kernels: K3 (traverse.cuh) with SimplexVisit as the per-lane query for
// the tree path, and simplex_flat_kernel (all primitives, split over
// primitive ranges) for the exact path; K4 merges the partial states.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "traverse.cuh"

namespace sdgpu {
namespace sx {

struct D3 {
    double x, y, z;
};
__device__ __forceinline__ D3 mk(double x, double y, double z) { return D3{x, y, z}; }
__device__ __forceinline__ D3 operator+(D3 a, D3 b) { return D3{a.x + b.x, a.y + b.y, a.z + b.z}; }
__device__ __forceinline__ D3 operator-(D3 a, D3 b) { return D3{a.x - b.x, a.y - b.y, a.z - b.z}; }
__device__ __forceinline__ D3 operator-(D3 a) { return D3{-a.x, -a.y, -a.z}; }
__device__ __forceinline__ D3 operator*(double s, D3 a) { return D3{s * a.x, s * a.y, s * a.z}; }
__device__ __forceinline__ D3 operator/(D3 a, double s) { return D3{a.x / s, a.y / s, a.z / s}; }
// Eigen fixed-size reductions: (x + y) + z
__device__ __forceinline__ double dot(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ double sqnorm(D3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
__device__ __forceinline__ double co(D3 v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }
__device__ __forceinline__ void set(D3& v, int a, double x) {
    if (a == 0) v.x = x;
    else if (a == 1) v.y = x;
    else v.z = x;
}
// std::max / std::min semantics (signed zeros included)
__device__ __forceinline__ double smax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double smin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }

struct Bary {
    double c0, c1;
};
struct Geom {
    D3 c0, c1, c2;
    int dim;
    __device__ __forceinline__ D3 at(Bary b) const {  // exact.hpp:35-41
        if (dim == 0) return c0;
        if (dim == 1) return c0 + b.c0 * (c1 - c0);
        return c0 + b.c0 * (c1 - c0) + b.c1 * (c2 - c0);
    }
};
struct GPair {
    double distance;
    Bary phi, lam;
    D3 pf, pg, grad;
};
__device__ __forceinline__ void finish_pair(GPair& r) {  // exact.hpp:59-63
    const D3 diff = r.pg - r.pf;
    r.distance = sqrt(sqnorm(diff));
    r.grad = r.distance > 0.0 ? diff / r.distance : D3{0.0, 0.0, 0.0};
}

// exact.hpp:68-73
__device__ __forceinline__ double closest_on_segment(D3 a, D3 b, D3 p) {
    const D3 ab = b - a;
    const double den = sqnorm(ab);
    if (den <= 0.0) return 0.0;
    return clamp01(dot(ab, p - a) / den);
}

// exact.hpp:77-106
__device__ __forceinline__ Bary closest_on_triangle(D3 a, D3 b, D3 c, D3 p) {
    const D3 ab = b - a, ac = c - a, ap = p - a;
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return Bary{0.0, 0.0};
    const D3 bp = p - b;
    const double d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) return Bary{1.0, 0.0};
    const D3 cp = p - c;
    const double d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return Bary{0.0, 1.0};
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) return Bary{d1 / (d1 - d3), 0.0};
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) return Bary{0.0, d2 / (d2 - d6)};
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        return Bary{1.0 - t, t};
    }
    const double den = 1.0 / (va + vb + vc);
    return Bary{vb * den, vc * den};
}

// exact.hpp:317-337 (lambda = point)
__device__ __forceinline__ GPair point_geom_distance(const Geom& f, D3 q) {
    GPair r;
    r.lam = Bary{0.0, 0.0};
    r.pg = q;
    if (f.dim == 0) {
        r.phi = Bary{0.0, 0.0};
        r.pf = f.c0;
    } else if (f.dim == 1) {
        r.phi = Bary{closest_on_segment(f.c0, f.c1, q), 0.0};
        r.pf = f.at(r.phi);
    } else {
        r.phi = closest_on_triangle(f.c0, f.c1, f.c2, q);
        r.pf = f.at(r.phi);
    }
    finish_pair(r);
    return r;
}

// exact.hpp:110-141
__device__ __forceinline__ void closest_segment_segment(D3 p1, D3 q1, D3 p2, D3 q2, double& s, double& t) {
    const D3 d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
    const double a = sqnorm(d1), e = sqnorm(d2), f = dot(d2, r);
    constexpr double kTiny = 1e-30;
    if (a <= kTiny && e <= kTiny) {
        s = t = 0.0;
        return;
    }
    if (a <= kTiny) {
        s = 0.0;
        t = clamp01(f / e);
        return;
    }
    const double c = dot(d1, r);
    if (e <= kTiny) {
        t = 0.0;
        s = clamp01(-c / a);
        return;
    }
    const double b = dot(d1, d2);
    const double denom = a * e - b * b;
    s = denom > 0.0 ? clamp01((b * f - c * e) / denom) : 0.0;
    t = (b * s + f) / e;
    if (t < 0.0) {
        t = 0.0;
        s = clamp01(-c / a);
    } else if (t > 1.0) {
        t = 1.0;
        s = clamp01((b - c) / a);
    }
}

// ----------------------------------------------------- face-enumeration QP
// exact.hpp:158-313. Faces of each simplex in ascending dimension:
// base (b0, b1), directions dir[p] = (d_p0, d_p1), k parameters.
struct Face {
    double b0, b1, d00, d01, d10, d11;
    int k;
};
__device__ __forceinline__ Face face_of(int dim, int i) {
    if (dim == 1) {
        if (i == 0) return Face{0, 0, 0, 0, 0, 0, 0};
        if (i == 1) return Face{1, 0, 0, 0, 0, 0, 0};
        return Face{0, 0, 1, 0, 0, 0, 1};
    }
    switch (i) {
        case 0: return Face{0, 0, 0, 0, 0, 0, 0};
        case 1: return Face{1, 0, 0, 0, 0, 0, 0};
        case 2: return Face{0, 1, 0, 0, 0, 0, 0};
        case 3: return Face{0, 0, 1, 0, 0, 0, 1};   // edge v0-v1
        case 4: return Face{0, 0, 0, 1, 0, 0, 1};   // edge v0-v2
        case 5: return Face{1, 0, -1, 1, 0, 0, 1};  // edge v1-v2
        default: return Face{0, 0, 1, 0, 0, 1, 2};
    }
}
// bary_at: base + sum_{p < k} z_p dir_p, accumulated in p order
__device__ __forceinline__ Bary bary_at(const Face& f, double z0, double z1) {
    Bary b{f.b0, f.b1};
    if (f.k >= 1) {
        b.c0 += z0 * f.d00;
        b.c1 += z0 * f.d01;
    }
    if (f.k >= 2) {
        b.c0 += z1 * f.d10;
        b.c1 += z1 * f.d11;
    }
    return b;
}
__device__ __forceinline__ bool feasible(Bary b, int dim) {
    constexpr double tol = 1e-10;
    if (dim == 0) return true;
    if (dim == 1) return b.c0 >= -tol && b.c0 <= 1.0 + tol;
    return b.c0 >= -tol && b.c1 >= -tol && b.c0 + b.c1 <= 1.0 + tol;
}
__device__ __forceinline__ void clamp_domain(Bary& b, int dim) {
    if (dim == 0) return;
    if (dim == 1) {
        b.c0 = clamp01(b.c0);
        return;
    }
    b.c0 = smax(b.c0, 0.0);
    b.c1 = smax(b.c1, 0.0);
    const double s = b.c0 + b.c1;
    if (s > 1.0) {
        b.c0 /= s;
        b.c1 /= s;
    }
}

// One candidate of the face enumeration: face i of f against face j of g
// (the loop body of exact.hpp:196-311). Returns false when the pair is
// skipped (k > 3, singular restriction, infeasible); otherwise the clamped
// barycentrics, points and squared distance.
__device__ __forceinline__ bool qp_candidate(const Geom& f, const Geom& g, int i, int j, Bary& fb, Bary& gb, D3& pf,
                                             D3& pg, double& d2) {
    const D3 fe1 = f.c1 - f.c0, fe2 = f.c2 - f.c0;
    const D3 ge1 = g.c1 - g.c0, ge2 = g.c2 - g.c0;
    const Face Ff = face_of(f.dim, i);
    const Face Fg = face_of(g.dim, j);
    const int k = Ff.k + Fg.k;
    if (k > 3) return false;
    D3 fd0 = D3{0, 0, 0}, fd1 = D3{0, 0, 0};
    if (Ff.k >= 1) fd0 = Ff.d00 * fe1 + Ff.d01 * fe2;
    if (Ff.k >= 2) fd1 = Ff.d10 * fe1 + Ff.d11 * fe2;
    const D3 f0 = f.at(bary_at(Ff, 0.0, 0.0));
    D3 gd0 = D3{0, 0, 0}, gd1 = D3{0, 0, 0};
    if (Fg.k >= 1) gd0 = -(Fg.d00 * ge1 + Fg.d01 * ge2);
    if (Fg.k >= 2) gd1 = -(Fg.d10 * ge1 + Fg.d11 * ge2);
    // cols = [f directions..., g directions...]
    const D3 c0 = Ff.k >= 1 ? fd0 : gd0;
    const D3 c1 = Ff.k >= 2 ? fd1 : (Ff.k == 1 ? gd0 : gd1);
    const D3 c2 = Ff.k == 2 ? gd0 : gd1;
    const D3 d0 = f0 - g.at(bary_at(Fg, 0.0, 0.0));
    double z0 = 0.0, z1 = 0.0, z2 = 0.0;
    if (k == 1) {
        const double m = sqnorm(c0);
        if (m <= 0.0) return false;
        z0 = -dot(c0, d0) / m;
    } else if (k == 2) {
        const double a11 = sqnorm(c0), a22 = sqnorm(c1);
        const double a12 = dot(c0, c1);
        const double det = a11 * a22 - a12 * a12;
        if (det <= 1e-12 * a11 * a22) return false;
        const double r1 = -dot(c0, d0), r2 = -dot(c1, d0);
        z0 = (a22 * r1 - a12 * r2) / det;
        z1 = (a11 * r2 - a12 * r1) / det;
    } else if (k == 3) {
        const double m00 = dot(c0, c0), m01 = dot(c0, c1), m02 = dot(c0, c2);
        const double m10 = dot(c1, c0), m11 = dot(c1, c1), m12 = dot(c1, c2);
        const double m20 = dot(c2, c0), m21 = dot(c2, c1), m22 = dot(c2, c2);
        // Eigen determinant: first-row cofactor expansion
        const double det = m00 * (m11 * m22 - m12 * m21) - m01 * (m10 * m22 - m12 * m20) +
                           m02 * (m10 * m21 - m11 * m20);
        const double scale = m00 * m11 * m22;
        if (fabs(det) <= 1e-12 * scale) return false;
        // Eigen inverse: cofactor_3x3(i, j) = m(i1,j1) m(i2,j2) - m(i1,j2) m(i2,j1)
        const double k00 = m11 * m22 - m12 * m21, k10 = m21 * m02 - m22 * m01, k20 = m01 * m12 - m02 * m11;
        const double idet = 1.0 / (k00 * m00 + k10 * m10 + k20 * m20);
        const double r00 = k00 * idet, r01 = k10 * idet, r02 = k20 * idet;
        const double r10 = (m12 * m20 - m10 * m22) * idet;  // cofactor (0,1)
        const double r11 = (m22 * m00 - m20 * m02) * idet;  // cofactor (1,1)
        const double r12 = (m02 * m10 - m00 * m12) * idet;  // cofactor (2,1)
        const double r20 = (m10 * m21 - m11 * m20) * idet;  // cofactor (0,2)
        const double r21 = (m20 * m01 - m21 * m00) * idet;  // cofactor (1,2)
        const double r22 = (m00 * m11 - m01 * m10) * idet;  // cofactor (2,2)
        const double h0 = -dot(c0, d0), h1 = -dot(c1, d0), h2 = -dot(c2, d0);
        z0 = r00 * h0 + r01 * h1 + r02 * h2;
        z1 = r10 * h0 + r11 * h1 + r12 * h2;
        z2 = r20 * h0 + r21 * h1 + r22 * h2;
    }
    fb = bary_at(Ff, z0, z1);
    const double gz0 = Ff.k == 0 ? z0 : (Ff.k == 1 ? z1 : z2);
    const double gz1 = Ff.k == 0 ? z1 : z2;
    gb = bary_at(Fg, gz0, gz1);
    if (!feasible(fb, f.dim) || !feasible(gb, g.dim)) return false;
    clamp_domain(fb, f.dim);
    clamp_domain(gb, g.dim);
    pf = f.at(fb);
    pg = g.at(gb);
    d2 = sqnorm(pg - pf);
    return true;
}

__device__ __forceinline__ int num_faces(int dim) { return dim == 0 ? 1 : (dim == 1 ? 3 : 7); }

// exact.hpp:158-313, serial: the first strictly best candidate in
// enumeration order (f faces outer, g faces inner).
__device__ __noinline__ GPair simplex_distance_qp(const Geom& f, const Geom& g) {
    const int nf = num_faces(f.dim), ng = num_faces(g.dim);
    GPair best;
    best.phi = best.lam = Bary{0.0, 0.0};
    best.pf = best.pg = D3{0.0, 0.0, 0.0};
    double best_d2 = INFINITY;
    bool have = false;
#pragma unroll 1
    for (int i = 0; i < nf; ++i) {
#pragma unroll 1
        for (int j = 0; j < ng; ++j) {
            Bary fb, gb;
            D3 pf, pg;
            double d2;
            if (!qp_candidate(f, g, i, j, fb, gb, pf, pg, d2)) continue;
            if (!have || d2 < best_d2) {
                have = true;
                best_d2 = d2;
                best.phi = fb;
                best.lam = gb;
                best.pf = pf;
                best.pg = pg;
            }
        }
    }
    finish_pair(best);
    return best;
}

// The same QP with the candidates spread over a group of GW lanes (8, 16
// or 32; all lanes of the group hold the same f, g): the minimum over (d2,
// enumeration index) is exactly the serial scan's first strictly best
// candidate. Shuffles use the group's mask, so groups of a warp may run
// different QPs at the same time.
template <int GW>
__device__ __forceinline__ unsigned group_mask() {
    const unsigned lane = threadIdx.x & 31u;
    return GW == 32 ? 0xffffffffu : (((1u << GW) - 1u) << (lane & ~unsigned(GW - 1)));
}
template <int GW>
__device__ __noinline__ GPair simplex_distance_qp_warp(const Geom& f, const Geom& g) {
    const unsigned mask = group_mask<GW>();
    const int lane = threadIdx.x & 31, r = lane & (GW - 1), base = lane - r;
    const int nf = num_faces(f.dim), ng = num_faces(g.dim), total = nf * ng;
    double bd2 = INFINITY;
    int bidx = 0x7fffffff;
    Bary bfb{0, 0}, bgb{0, 0};
    D3 bpf{0, 0, 0}, bpg{0, 0, 0};
    for (int c = r; c < total; c += GW) {
        Bary fb, gb;
        D3 pf, pg;
        double d2;
        if (qp_candidate(f, g, c / ng, c % ng, fb, gb, pf, pg, d2) && d2 < bd2) {  // c increases per lane
            bd2 = d2;
            bidx = c;
            bfb = fb;
            bgb = gb;
            bpf = pf;
            bpg = pg;
        }
    }
    double md2 = bd2;
    int midx = bidx;
#pragma unroll
    for (int off = GW / 2; off; off >>= 1) {
        const double o = __shfl_xor_sync(mask, md2, off);
        const int oi = __shfl_xor_sync(mask, midx, off);
        if (o < md2 || (o == md2 && oi < midx)) {
            md2 = o;
            midx = oi;
        }
    }
    GPair best;
    if (midx == 0x7fffffff) {  // no candidate (not reachable: vertex pairs always qualify)
        best.phi = best.lam = Bary{0.0, 0.0};
        best.pf = best.pg = D3{0.0, 0.0, 0.0};
    } else {
        const int src = base + (midx % GW);
        auto sh = [&](double v) { return __shfl_sync(mask, v, src); };
        best.phi = Bary{sh(bfb.c0), sh(bfb.c1)};
        best.lam = Bary{sh(bgb.c0), sh(bgb.c1)};
        best.pf = D3{sh(bpf.x), sh(bpf.y), sh(bpf.z)};
        best.pg = D3{sh(bpg.x), sh(bpg.y), sh(bpg.z)};
    }
    finish_pair(best);
    return best;
}

// exact.hpp:342-367 (GW > 0: the QP spread over a group of GW lanes)
template <int GW>
__device__ GPair simplex_distance_t(const Geom& f, const Geom& g) {
    if (g.dim == 0) return point_geom_distance(f, g.c0);
    if (f.dim == 0) {
        const GPair r = point_geom_distance(g, f.c0);
        GPair out;
        out.phi = Bary{0.0, 0.0};
        out.lam = r.phi;
        out.pf = r.pg;
        out.pg = r.pf;
        finish_pair(out);
        return out;
    }
    if (f.dim == 1 && g.dim == 1) {
        double s, t;
        closest_segment_segment(f.c0, f.c1, g.c0, g.c1, s, t);
        GPair r;
        r.phi = Bary{s, 0.0};
        r.lam = Bary{t, 0.0};
        r.pf = f.at(r.phi);
        r.pg = g.at(r.lam);
        finish_pair(r);
        return r;
    }
    if constexpr (GW > 0) return simplex_distance_qp_warp<GW>(f, g);
    else return simplex_distance_qp(f, g);
}
__device__ __forceinline__ GPair simplex_distance(const Geom& f, const Geom& g) { return simplex_distance_t<0>(f, g); }

// bvh.hpp:105-111 and 113-180
struct BoxProx {
    double distance;
    D3 yb;
    Bary lam;
    bool must_descend;
};
template <int GW>
__device__ BoxProx box_primitive_proximity_t(D3 lo, D3 hi, const Geom& g) {
    BoxProx r;
    r.lam = Bary{0.0, 0.0};
    r.must_descend = false;
    if (g.dim == 0) {  // Aabb::closest_point (cwiseMax then cwiseMin)
        const D3 q = g.c0;
        r.yb = mk(smin(smax(q.x, lo.x), hi.x), smin(smax(q.y, lo.y), hi.y), smin(smax(q.z, lo.z), hi.z));
        r.distance = sqrt(sqnorm(q - r.yb));
        return r;
    }
    int out_axis[3];
    int n_out = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double h = co(hi, a), l = co(lo, a);
        bool all_hi = co(g.c0, a) >= h && co(g.c1, a) >= h;
        bool all_lo = co(g.c0, a) <= l && co(g.c1, a) <= l;
        if (g.dim == 2) {
            all_hi = all_hi && co(g.c2, a) >= h;
            all_lo = all_lo && co(g.c2, a) <= l;
        }
        out_axis[a] = all_hi ? 1 : (all_lo ? -1 : 0);
        n_out += out_axis[a] != 0;
    }
    if (n_out == 0) {
        r.must_descend = true;
        r.distance = 0.0;
        r.yb = 0.5 * (lo + hi);
        return r;
    }
    auto side = [&](int a) { return out_axis[a] > 0 ? co(hi, a) : co(lo, a); };
    Geom feat;
    if (n_out == 3) {
        feat.dim = 0;
        feat.c0 = mk(side(0), side(1), side(2));
        feat.c1 = feat.c2 = D3{0, 0, 0};
        const GPair p = simplex_distance_t<GW>(feat, g);
        r.distance = p.distance;
        r.yb = p.pf;
        r.lam = p.lam;
    } else if (n_out == 2) {
        const int fa = out_axis[0] == 0 ? 0 : (out_axis[1] == 0 ? 1 : 2);
        D3 a, b;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const double v = out_axis[ax] != 0 ? side(ax) : 0.0;
            set(a, ax, v);
            set(b, ax, v);
        }
        set(a, fa, co(lo, fa));
        set(b, fa, co(hi, fa));
        feat.dim = 1;
        feat.c0 = a;
        feat.c1 = b;
        feat.c2 = D3{0, 0, 0};
        const GPair p = simplex_distance_t<GW>(feat, g);
        r.distance = p.distance;
        r.yb = p.pf;
        r.lam = p.lam;
    } else {
        const int fa = out_axis[0] != 0 ? 0 : (out_axis[1] != 0 ? 1 : 2);
        const int u = (fa + 1) % 3, v = (fa + 2) % 3;
        const double s = side(fa);
        D3 r00, r10, r11, r01;
        set(r00, fa, s); set(r10, fa, s); set(r11, fa, s); set(r01, fa, s);
        set(r00, u, co(lo, u)); set(r00, v, co(lo, v));
        set(r10, u, co(hi, u)); set(r10, v, co(lo, v));
        set(r11, u, co(hi, u)); set(r11, v, co(hi, v));
        set(r01, u, co(lo, u)); set(r01, v, co(hi, v));
        feat.dim = 2;
        feat.c0 = r00;
        feat.c1 = r10;
        feat.c2 = r11;
        const GPair p1 = simplex_distance_t<GW>(feat, g);
        feat.c1 = r11;
        feat.c2 = r01;
        const GPair p2 = simplex_distance_t<GW>(feat, g);
        const bool first = p1.distance <= p2.distance;
        r.distance = first ? p1.distance : p2.distance;
        r.yb = first ? p1.pf : p2.pf;
        r.lam = first ? p1.lam : p2.lam;
    }
    return r;
}
__device__ __noinline__ BoxProx box_primitive_proximity(D3 lo, D3 hi, const Geom& g) {
    return box_primitive_proximity_t<0>(lo, hi, g);
}

// Leaf geometry record: corners (9), shape gradients (edge: e/|e|^2; tri:
// G1, G2), pad.
__device__ __forceinline__ Geom leaf_geom(int meta, const double* geo) {
    Geom f;
    f.dim = meta & 3;
    f.c0 = mk(geo[0], geo[1], geo[2]);
    f.c1 = mk(geo[3], geo[4], geo[5]);
    f.c2 = mk(geo[6], geo[7], geo[8]);
    return f;
}

// The weight and accumulation half of a leaf term, given the closest pair.
__device__ __forceinline__ void leaf_accumulate(const Phys<double>& ph, const Poly<double>* polys, int ne, int meta,
                                                const double* geo, const GPair& p, Acc<double>& acc) {
    const int kind = meta & 3, poly = (meta >> 2) - 1;
    const double d = p.distance;
    double lw = ph.lw_unit, kx = 0.0, ky = 0.0;
    if (kind == 1 && poly >= 0) {
        const double* c = polys[poly].c;
        const double t = p.phi.c0;
        const double base = fma(t, fma(t, fma(t, fma(t, c[4], c[3]), c[2]), c[1]), c[0]);
        const double dnum = fma(t, fma(t, fma(t, c[8], c[7]), c[6]), c[5]);
        if (base > 1e-300) {
            lw = ph.S * log2(base);
            kx = dnum / base;
        } else {
            lw = ph.lw_floor;
        }
    } else if (kind == 2 && poly >= 0) {
        double base, wx, wy;
        tri_poly(polys[ne + poly], p.phi.c0, p.phi.c1, base, wx, wy);
        if (base > 1e-300) {
            lw = ph.S * log2(base);
            kx = wx / base;
            ky = wy / base;
        } else {
            lw = ph.lw_floor;
        }
    }
    const double x = fma(ph.kappa, d, lw);
    const double xm = bump(acc, masked(ph, d, x - acc.m), [&] { return x; });
    const double e = exp2(xm);
    acc.s += e;
    double gx = e * p.grad.x, gy = e * p.grad.y, gz = e * p.grad.z;
    if (kind == 1) {
        const double ek = e * kx;
        gx -= ek * geo[9];
        gy -= ek * geo[10];
        gz -= ek * geo[11];
    } else if (kind == 2) {
        const double ex = e * kx, ey = e * ky;
        gx -= ex * geo[9] + ey * geo[12];
        gy -= ex * geo[10] + ey * geo[13];
        gz -= ex * geo[11] + ey * geo[14];
    }
    acc.gx += gx;
    acc.gy += gy;
    acc.gz += gz;
}

// One exact leaf term for query g (smooth.hpp:51-61): w and the alpha-scaled
// shape gradient at the closest point phi on f, in the log2 accumulator.
__device__ __noinline__ void leaf_term(const Phys<double>& ph, const Poly<double>* polys, int ne, int meta,
                                       const double* geo, const Geom& g, Acc<double>& acc) {
    leaf_accumulate(ph, polys, ne, meta, geo, simplex_distance(leaf_geom(meta, geo), g), acc);
}

__device__ __forceinline__ Geom load_query(const double* qg, const int32_t* qd, int64_t qi, bool valid) {
    Geom g;
    const double* c = qg + 9 * (valid ? qi : 0);
    g.c0 = mk(c[0], c[1], c[2]);
    g.c1 = mk(c[3], c[4], c[5]);
    g.c2 = mk(c[6], c[7], c[8]);
    g.dim = valid ? qd[qi] : 0;
    return g;
}

}  // namespace sx

// K3's per-lane query for simplex queries.
struct SimplexVisit {
    static constexpr bool kLeafQueue = false;  // per-lane QP leaves: no deferred leaf queues
    template <class U>
    static constexpr bool kFrame = false;
    sx::Geom g;
    __device__ __forceinline__ void load(const TraverseArgs<double>& a, int64_t qi, bool valid) {
        g = sx::load_query(a.qgeom, a.qdim, qi, valid);
    }
    // collect_contributions (smooth.hpp:114-121), bh_condition (bvh.hpp:185-187)
    template <bool HASH, class CNT>
    __device__ __forceinline__ bool far_test(const TraverseArgs<double>& a, const NodeT<double>& b, int32_t id,
                                             double lgc, bool emit, Acc<double>& acc, CNT& nfar, uint64_t& h,
                                             unsigned long long&) const {
        if (!a.use_bh) return false;
        const sx::BoxProx pr =
            sx::box_primitive_proximity(sx::mk(b.v[0], b.v[1], b.v[2]), sx::mk(b.v[4], b.v[5], b.v[6]), g);
        if (!(!pr.must_descend && pr.distance > 0.0 && a.diam64[id] < a.beta64 * pr.distance)) return false;
        if (emit) {
            const sx::D3 diff = g.at(pr.lam) - pr.yb;
            far_term(a.ph, lgc + a.lw_ff, pr.distance, 1.0 / pr.distance, diff.x, diff.y, diff.z, acc);
            ++nfar;
            if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
        }
        return true;
    }
    template <bool HASH, class CNT>
    __device__ __forceinline__ bool visit(const TraverseArgs<double>& a, const Poly<double>* polys,
                                          const NodeT<double>& b, int32_t id, double lgc, Acc<double>& acc,
                                          CNT& nleaf, CNT& nfar, uint64_t& h, unsigned long long& nre) const {
        int32_t link;
        memcpy(&link, &b.v[7], sizeof(int32_t));
        if (far_test<HASH>(a, b, id, lgc, true, acc, nfar, h, nre)) return false;
        if (link >= 0) return true;
        const int slot = -link - 1;
        sx::leaf_term(a.ph, polys, a.ne, a.leafmeta[slot], a.leafgeom + size_t(slot) * 16, g, acc);
        ++nleaf;
        if constexpr (HASH) h += decision_mix(uint64_t(id), 2);
        return false;
    }
    template <bool HASH, class CNT>
    __device__ __forceinline__ void visit_pair(const TraverseArgs<double>& a, const Poly<double>* polys,
                                               const NodeT<double>& bl, const NodeT<double>& br, int32_t lid,
                                               int32_t rid, double lgl, double lgr, Acc<double>& acc, CNT& nleaf,
                                               CNT& nfar, uint64_t& h, unsigned long long& nre, bool& dl,
                                               bool& dr) const {
        dl = visit<HASH>(a, polys, bl, lid, lgl, acc, nleaf, nfar, h, nre);
        dr = visit<HASH>(a, polys, br, rid, lgr, acc, nleaf, nfar, h, nre);
    }
};

// K3W (default for simplex queries): one warp per query simplex; its walk
// is processed 32 / GW nodes at a time (a shared-memory stack as in K3F),
// and every node test is cooperative over a group of GW lanes -- the
// face-enumeration QP of a box feature or a leaf has up to 49 independent
// candidates, which the group evaluates in parallel before a (d2, index)
// arg-min. A node is tested iff all its ancestors descended (the
// reference's visited set); each group accumulates the terms of its nodes
// and the groups' states merge in fp64 at the end. The per-lane QP of
// K3 / K3F serialises the 49 candidates and diverges between feature types
// (3.5 active lanes per instruction in the frontier kernel's profile).
// Stack bound as K3F: 2 (32 / GW) entries per level.
constexpr int kWarpThreads = 128;
template <int GW, bool HASH>
__global__ void __launch_bounds__(kWarpThreads) simplex_warp_kernel(const __grid_constant__ TraverseArgs<double> a,
                                                                    int cap) {
    constexpr int NG = 32 / GW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<double>* polys = reinterpret_cast<Poly<double>*>(smem_raw);
    int32_t* stacks = reinterpret_cast<int32_t*>(smem_raw + poly_bytes<double>(a.npoly));
    for (int t = threadIdx.x; t < a.npoly * kPolyCoefs; t += blockDim.x)
        reinterpret_cast<double*>(polys)[t] = reinterpret_cast<const double*>(a.polys)[t];
    __syncthreads();
    const int lane = threadIdx.x & 31, grp = lane / GW, r = lane % GW;
    const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // sorted position
    if (i >= a.Q) return;
    int32_t* stk = stacks + size_t(threadIdx.x >> 5) * cap;
    const int64_t qi = a.perm ? a.perm[i] : i;
    const sx::Geom g = sx::load_query(a.qgeom, a.qdim, qi, true);
    Acc<double> acc;
    acc.init();
    int32_t nleaf = 0, nfar = 0;  // per query: < 2^31 nodes
    uint64_t h = 0;
    if (lane == 0) stk[0] = 0;
    __syncwarp();
    int n = 1;
    while (n > 0) {
        const int take = n < NG ? n : NG;
        const int base = n - take;
        const int32_t id = grp < take ? stk[base + grp] : -1;
        __syncwarp();
        bool d = false;
        int32_t link = 0;
        if (id >= 0) {  // uniform within the group
            const NodeT<double> b = a.box[id];
            memcpy(&link, &b.v[7], sizeof(int32_t));
            bool far = false;
            if (a.use_bh) {  // collect_contributions (smooth.hpp:114-121), bh_condition (bvh.hpp:185-187)
                const sx::BoxProx pr = sx::box_primitive_proximity_t<GW>(sx::mk(b.v[0], b.v[1], b.v[2]),
                                                                          sx::mk(b.v[4], b.v[5], b.v[6]), g);
                if (!pr.must_descend && pr.distance > 0.0 && a.diam64[id] < a.beta64 * pr.distance) {
                    const sx::D3 diff = g.at(pr.lam) - pr.yb;
                    far_term(a.ph, a.lgcount[id] + a.lw_ff, pr.distance, 1.0 / pr.distance, diff.x, diff.y, diff.z,
                             acc);
                    ++nfar;
                    if constexpr (HASH) h += decision_mix(uint64_t(id), 1);
                    far = true;
                }
            }
            if (!far) {
                if (link < 0) {
                    const int slot = -link - 1;
                    const int meta = a.leafmeta[slot];
                    const double* geo = a.leafgeom + size_t(slot) * 16;
                    const sx::GPair p = sx::simplex_distance_t<GW>(sx::leaf_geom(meta, geo), g);
                    sx::leaf_accumulate(a.ph, polys, a.ne, meta, geo, p, acc);
                    ++nleaf;
                    if constexpr (HASH) h += decision_mix(uint64_t(id), 2);
                } else {
                    d = true;
                }
            }
        }
        const unsigned D = __ballot_sync(0xffffffffu, d && r == 0);  // one bit per descending group
        if (d && r == 0) {
            const int pos = base + 2 * __popc(D & ((1u << lane) - 1u));
            stk[pos] = link;        // right child below ...
            stk[pos + 1] = id + 1;  // ... left child on top
        }
        __syncwarp();
        n = base + 2 * __popc(D);
    }
    // merge the groups' states (fp64, anchored at the warp maximum); within a
    // group every lane holds the same state, lane r = 0 contributes it
    Tot tot;
    tot.init();
    tot.flush(acc);
    double M = r == 0 ? tot.M : -INFINITY;
    for (int off = 16; off; off >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, off));
    const double f = (r != 0 || M == -INFINITY || tot.M == -INFINITY) ? 0.0 : exp2(tot.M - M);
    double s = tot.s * f, gx = tot.gx * f, gy = tot.gy * f, gz = tot.gz * f;
    unsigned long long L = r == 0 ? (unsigned long long)nleaf : 0ull, F = r == 0 ? (unsigned long long)nfar : 0ull,
                       H = r == 0 ? h : 0ull;
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        gx += __shfl_xor_sync(0xffffffffu, gx, off);
        gy += __shfl_xor_sync(0xffffffffu, gy, off);
        gz += __shfl_xor_sync(0xffffffffu, gz, off);
        L += __shfl_xor_sync(0xffffffffu, L, off);
        F += __shfl_xor_sync(0xffffffffu, F, off);
        H += __shfl_xor_sync(0xffffffffu, H, off);
    }
    if (lane == 0) {
        a.part[i] = M;
        a.part[a.Q + i] = s;
        a.part[2 * a.Q + i] = gx;
        a.part[3 * a.Q + i] = gy;
        a.part[4 * a.Q + i] = gz;
        a.leaves[i] = int64_t(L);
        a.far[i] = int64_t(F);
        if (HASH) a.hash[i] = H;
    }
}

// Exact path: thread = query, blockIdx.y = primitive range (index order);
// partial states [split][5][Q] merged by K4.
constexpr int kFlatThreads = 128;
struct FlatArgs {
    const double* qgeom;
    const int32_t* qdim;
    int64_t Q;
    const double* primgeom;  // 16 doubles per primitive, index order
    const int32_t* primmeta;
    int64_t N, chunk;
    const Poly<double>* polys;
    int ne, npoly;
    Phys<double> ph;
    double* part;
};

__global__ void __launch_bounds__(kFlatThreads) simplex_flat_kernel(const __grid_constant__ FlatArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Poly<double>* polys = reinterpret_cast<Poly<double>*>(smem_raw);
    for (int i = threadIdx.x; i < a.npoly * kPolyCoefs; i += blockDim.x)
        reinterpret_cast<double*>(polys)[i] = reinterpret_cast<const double*>(a.polys)[i];
    __syncthreads();
    const int64_t qi = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (qi >= a.Q) return;
    const sx::Geom g = sx::load_query(a.qgeom, a.qdim, qi, true);
    const int64_t lo = int64_t(blockIdx.y) * a.chunk, hi = std::min(a.N, lo + a.chunk);
    Acc<double> acc;
    acc.init();
    Tot tot;
    tot.init();
    for (int64_t p = lo; p < hi; ++p) {
        sx::leaf_term(a.ph, polys, a.ne, a.primmeta[p], a.primgeom + size_t(p) * 16, g, acc);
        if (((p - lo) & 255) == 255) tot.flush(acc);
    }
    tot.flush(acc);
    double* part = a.part + size_t(blockIdx.y) * 5 * a.Q;
    part[qi] = tot.M;
    part[a.Q + qi] = tot.s;
    part[2 * a.Q + qi] = tot.gx;
    part[3 * a.Q + qi] = tot.gy;
    part[4 * a.Q + qi] = tot.gz;
}

// Morton keys of the query centroids (coherent packets)
__global__ void simplex_centroids(const double* qg, const int32_t* qd, int64_t Q, double* out) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= Q) return;
    const double* c = qg + 9 * i;
    const int n = qd[i] + 1;
    for (int a = 0; a < 3; ++a) {
        double s = c[a];
        if (n > 1) s += c[3 + a];
        if (n > 2) s += c[6 + a];
        out[3 * i + a] = s / n;
    }
}

// ------------------------------------------------------------------ host
// fp64 geometry record of primitive p: corners, shape gradients.
static void geo_record(const Ctx& c, int64_t p, double* out) {
    std::memset(out, 0, 16 * sizeof(double));
    const int kind = c.kind[p];
    for (int k = 0; k <= kind; ++k)
        for (int a = 0; a < 3; ++a) out[3 * k + a] = c.xyz[3 * size_t(c.sv[3 * p + k]) + a];
    if (kind == SD_POINT) return;
    double rec[kRecTri];
    build_record<double>(c, p, rec);
    if (kind == SD_EDGE) {
        for (int a = 0; a < 3; ++a) out[9 + a] = rec[7 + a];
    } else {
        for (int a = 0; a < 6; ++a) out[9 + a] = rec[16 + a];
    }
}
static int geo_meta(const Ctx& c, int64_t p) {
    const int k = c.kind[p];
    const int poly = k == SD_POINT ? -1 : c.poly_index[p];
    return k | ((poly + 1) << 2);
}

static void ensure_prims(Ctx& c) {
    if (c.sx_prim_ready) return;
    std::vector<double> geo(size_t(c.N) * 16);
    std::vector<int32_t> meta(size_t(c.N));
    for (int64_t p = 0; p < c.N; ++p) {
        geo_record(c, p, geo.data() + size_t(p) * 16);
        meta[p] = geo_meta(c, p);
    }
    check_cuda(cudaMemcpy(c.primgeom.ensure(geo.size() * sizeof(double)), geo.data(), geo.size() * sizeof(double),
                          cudaMemcpyHostToDevice),
               "upload primitive geometry");
    check_cuda(cudaMemcpy(c.primmeta.ensure(meta.size() * sizeof(int32_t)), meta.data(),
                          meta.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
               "upload primitive meta");
    c.sx_prim_ready = true;
}

// fp64 traversal layout + leaf geometry in leaf-slot (pre-order) order
static DeviceTree& ensure_tree(Ctx& c) {
    DeviceTree* t = &c.dtree;
    if (c.precision == SD_FP64) {
        if (!c.dtree_ready) tree_upload(c);
    } else {
        t = &c.dtree64;
    }
    if (!c.sx_tree_ready) {
        if (c.precision != SD_FP64) tree_upload64(c, c.dtree64);
        std::vector<double> geo;
        geo.reserve(size_t(c.N) * 16);
        for (const sd_bvh_node& nd : c.tree) {  // pre-order: leaf slots in node order
            if (nd.left >= 0) continue;
            double g[16];
            geo_record(c, nd.primitive, g);
            geo.insert(geo.end(), g, g + 16);
        }
        check_cuda(cudaMemcpy(c.leafgeom.ensure(geo.size() * sizeof(double)), geo.data(), geo.size() * sizeof(double),
                              cudaMemcpyHostToDevice),
                   "upload leaf geometry");
        c.sx_tree_ready = true;
    }
    return *t;
}

void simplex_query(Ctx& c, const double* corners, const int32_t* dims, int64_t Q, const sd_params& p, int mode,
                   const FinalizeOut& out, cudaStream_t st) {
    int64_t launches = 0;
    if (Q == 0) {
        c.last_launches = 0;
        return;
    }
    if (c.N == 0) {
        check_cuda(launch_empty_result(Q, out, st), "empty result");
        c.last_launches = 1;
        return;
    }
    const int ne = int(c.edge_a.size() / 5), nt = int(c.tri_stored.size() / 13);
    const int npoly = std::max(1, ne + nt);
    std::vector<Poly<double>> ptab(npoly);
    for (int e = 0; e < ne; ++e) ptab[e] = make_poly<double>(c, SD_EDGE, e, p);
    for (int k = 0; k < nt; ++k) ptab[ne + k] = make_poly<double>(c, SD_TRIANGLE, k, p);
    Poly<double>* dpoly = static_cast<Poly<double>*>(c.polys.ensure(ptab.size() * sizeof(Poly<double>)));
    check_cuda(cudaMemcpyAsync(dpoly, ptab.data(), ptab.size() * sizeof(Poly<double>), cudaMemcpyHostToDevice, st),
               "upload polys");
    const Phys<double> ph = make_phys<double>(c, p);

    if (mode == SD_EXACT) {
        ensure_prims(c);
        FlatArgs a;
        a.qgeom = corners;
        a.qdim = dims;
        a.Q = Q;
        a.primgeom = c.primgeom.as<double>();
        a.primmeta = c.primmeta.as<int32_t>();
        a.N = c.N;
        a.polys = dpoly;
        a.ne = ne;
        a.npoly = npoly;
        a.ph = ph;
        // enough CTAs for ~4 waves of 148 SMs, >= 64 primitives per range
        const int64_t qblocks = (Q + kFlatThreads - 1) / kFlatThreads;
        int64_t splits = std::max<int64_t>(1, (148 * 8 + qblocks - 1) / qblocks);
        splits = std::min<int64_t>({splits, std::max<int64_t>(1, c.N / 64), 65535});
        a.chunk = (c.N + splits - 1) / splits;
        splits = (c.N + a.chunk - 1) / a.chunk;
        a.part = static_cast<double*>(c.part.ensure(size_t(splits) * 5 * Q * sizeof(double)));
        const size_t smem = poly_bytes<double>(npoly);
        check_cuda(cudaFuncSetAttribute(simplex_flat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)),
                   "smem attr");
        simplex_flat_kernel<<<dim3(unsigned(qblocks), unsigned(splits)), kFlatThreads, smem, st>>>(a);
        check_cuda(cudaGetLastError(), "simplex flat kernel");
        ++launches;
        check_cuda(launch_finalize(a.part, int(splits), Q, p.alpha, p.epsilon, c.N, nullptr, nullptr, nullptr,
                                   nullptr, out, st),
                   "finalize");
        ++launches;
        c.last_launches = launches;
        return;
    }

    DeviceTree& t = ensure_tree(c);
    // Morton order of the query centroids over the root box (measured on the
    // paper-table rows against a Hilbert order over the joined boxes and the
    // input order: profiles/README.md)
    double* cen = static_cast<double*>(c.qd.ensure(size_t(Q) * 3 * sizeof(double)));
    simplex_centroids<<<unsigned((Q + 255) / 256), 256, 0, st>>>(corners, dims, Q, cen);
    check_cuda(cudaGetLastError(), "centroids");
    ++launches;
    const sd_bvh_node& root = c.tree[0];
    const int64_t* perm = sort_queries<double>(c, cen, Q, root.lo, root.hi, st, launches, false);

    double* part = static_cast<double*>(c.part.ensure(size_t(5) * Q * sizeof(double)));
    int64_t* cnt = static_cast<int64_t*>(c.counters.ensure(size_t(Q) * 3 * sizeof(int64_t) + 64));
    TraverseArgs<double> a;
    std::memset(&a, 0, sizeof(a));
    a.q = nullptr;
    a.perm = perm;
    a.Q = Q;
    a.box = t.box.as<NodeT<double>>();
    a.pairs = t.pairs.as<PairT<double>>();
    a.count = t.count.as<int32_t>();
    a.lgcount = t.lgcount.as<double>();
    a.diam64 = t.diam64.as<double>();
    a.leafrec = nullptr;
    a.leafmeta = t.leafmeta.as<int32_t>();
    a.polys = dpoly;
    a.ph = ph;
    a.lw_ff = std::log2(std::pow(std::max(c.A * c.sup_wtilde, 1e-300), p.alpha / std::max(p.alpha, p.alpha_u)));
    a.ne = ne;
    a.npoly = npoly;
    a.use_bh = p.beta > 0.0 ? 1 : 0;
    a.exact_boxes = 1;
    a.stack_depth = t.depth + 1;
    a.beta64 = p.beta;
    a.part = part;
    a.leaves = cnt;
    a.far = cnt + Q;
    a.hash = reinterpret_cast<uint64_t*>(cnt + 2 * Q);
    a.rechecks = reinterpret_cast<unsigned long long*>(cnt + 3 * Q);
    a.qgeom = corners;
    a.qdim = dims;
    a.leafgeom = c.leafgeom.as<double>();
    // SDGPU_SIMPLEX_KERNEL = warp (default: K3W) | frontier (K3F) | pair (K3)
    const char* ke = std::getenv("SDGPU_SIMPLEX_KERNEL");
    const std::string kern = ke && *ke ? ke : "warp";
    int nsplits = 1;
    if (kern == "warp") {
        // group width: lanes per node test (SDGPU_SIMPLEX_GW = 8 | 16 | 32)
        const char* ge = std::getenv("SDGPU_SIMPLEX_GW");
        // (tools/simplex_sweep.sh over the paper-table rows: 8 ~ 16 < 32)
        int gw = ge && *ge ? std::atoi(ge) : 8;
        if (gw != 16 && gw != 32) gw = 8;
        const int cap = 2 * (32 / gw) * (t.depth + 1);
        const size_t smem = poly_bytes<double>(npoly) + size_t(cap) * (kWarpThreads / 32) * sizeof(int32_t);
        using K = void (*)(TraverseArgs<double>, int);
        K kw = gw == 8 ? (out.hash ? simplex_warp_kernel<8, true> : simplex_warp_kernel<8, false>)
             : gw == 32 ? (out.hash ? simplex_warp_kernel<32, true> : simplex_warp_kernel<32, false>)
                        : (out.hash ? simplex_warp_kernel<16, true> : simplex_warp_kernel<16, false>);
        check_cuda(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
        kw<<<unsigned((Q * 32 + kWarpThreads - 1) / kWarpThreads), kWarpThreads, smem, st>>>(a, cap);
        check_cuda(cudaGetLastError(), "simplex warp kernel");
        ++launches;
    } else if (!(kern == "frontier" &&
                 launch_frontier<double, SimplexVisit>(c, t, a, out.hash != nullptr, st, launches, 32))) {
        nsplits = launch_pair_traversal<double, SimplexVisit>(c, t, a, out.hash != nullptr, st, launches, 4);
    }
    check_cuda(launch_finalize(a.part, nsplits, Q, p.alpha, p.epsilon, 0, a.leaves, a.far, a.hash, perm, out, st),
               "finalize");
    ++launches;
    c.last_launches = launches;
}

}  // namespace sdgpu
