// oracle/sdoracle.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement, in plain fp64 C++ (no Eigen), of the reference
// smooth-distance hot path of arXiv 2108.10480 (/root/reference/proj).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs may load this code; it is the checker, never the
// product. The product path (paper_2108_10480_b200/csrc) never links it.
//
// Every function cites the reference file:line it restates
// (paths relative to /root/reference/proj/include/smoothdist/).
// Deliberate reference quirks that are kept: recording-order summation,
// the -708 exponent mask, epsilon = 1e-300 in the gradient denominator,
// the padded 8x8 Horner for triangle weights and the second
// evaluate_weight call inside weight_gradient_world.
//
// Compiled with -ffp-contract=off so that the fp64 box tests used for the
// BVH admissibility decision round exactly like the GPU's explicit
// __dadd_rn/__dmul_rn sequence (decision-hash equality is a checked
// invariant).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

namespace sdo {

// ---------------------------------------------------------------- L0 types
// common.hpp:13 (Vec3 = Eigen::Vector3d; 24 B, x,y,z contiguous)
struct V3 {
    double x = 0, y = 0, z = 0;
    V3() = default;
    V3(double a, double b, double c) : x(a), y(b), z(c) {}
    double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
    double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
};
inline V3 operator+(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 operator-(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 operator-(V3 a) { return {-a.x, -a.y, -a.z}; }
inline V3 operator*(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline V3 operator/(V3 a, double s) { return {a.x / s, a.y / s, a.z / s}; }
inline V3& operator+=(V3& a, V3 b) { a = a + b; return a; }
inline bool operator==(V3 a, V3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }
// Eigen fixed-size reductions sum left to right: (x + y) + z.
inline double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline double sqnorm(V3 a) { return a.x * a.x + a.y * a.y + a.z * a.z; }
inline double norm(V3 a) { return std::sqrt(sqnorm(a)); }
inline V3 cross(V3 a, V3 b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 normalized(V3 a) {
    const double n = norm(a);
    return n > 0 ? a / n : a;
}
inline V3 vmin(V3 a, V3 b) { return {std::min(a.x, b.x), std::min(a.y, b.y), std::min(a.z, b.z)}; }
inline V3 vmax(V3 a, V3 b) { return {std::max(a.x, b.x), std::max(a.y, b.y), std::max(a.z, b.z)}; }

// common.hpp:19-48 -- empty by default (inverted bounds).
struct Aabb {
    V3 lo{INFINITY, INFINITY, INFINITY};
    V3 hi{-INFINITY, -INFINITY, -INFINITY};
    bool valid() const { return lo.x <= hi.x && lo.y <= hi.y && lo.z <= hi.z; }
    void expand(V3 p) { lo = vmin(lo, p); hi = vmax(hi, p); }
    void expand(const Aabb& b) { lo = vmin(lo, b.lo); hi = vmax(hi, b.hi); }
    V3 center() const { return 0.5 * (lo + hi); }
    V3 extent() const { return hi - lo; }
    double diagonal() const { return valid() ? norm(hi - lo) : 0.0; }          // :40
    V3 closest_point(V3 q) const {                                            // :43
        // Eigen cwiseMax then cwiseMin
        V3 t = {std::max(q.x, lo.x), std::max(q.y, lo.y), std::max(q.z, lo.z)};
        return {std::min(t.x, hi.x), std::min(t.y, hi.y), std::min(t.z, hi.z)};
    }
    bool contains(V3 p, double tol = 0) const {
        return p.x >= lo.x - tol && p.y >= lo.y - tol && p.z >= lo.z - tol && p.x <= hi.x + tol &&
               p.y <= hi.y + tol && p.z <= hi.z + tol;
    }
};

[[noreturn]] inline void fail(const std::string& m) { throw std::runtime_error(m); }  // common.hpp:50

// params.hpp:13-22
struct Params {
    double alpha = 100.0, alpha_u = 600.0, beta = 0.5, alpha_q = 100.0, epsilon = 1e-300;
    double attenuation() const { return alpha / std::max(alpha, alpha_u); }
};

// ---------------------------------------------------------------- L1 mesh
// mesh.hpp:15-50
enum Kind : std::uint8_t { POINT = 0, EDGE = 1, TRIANGLE = 2 };
struct Simplex {
    std::int32_t v[3] = {-1, -1, -1};
    std::uint8_t kind = POINT;
    int dim() const { return kind; }
    int nverts() const { return kind + 1; }
};
struct Mesh {
    std::vector<V3> vertices;
    std::vector<Simplex> simplices;
    std::size_t nv() const { return vertices.size(); }
    std::size_t ns() const { return simplices.size(); }
    std::array<V3, 3> corners(const Simplex& s) const {
        std::array<V3, 3> c{};
        for (int i = 0; i < s.nverts(); ++i) c[i] = vertices[s.v[i]];
        return c;
    }
    void add_point(int a) { Simplex s; s.v[0] = a; s.kind = POINT; simplices.push_back(s); }
    void add_edge(int a, int b) { Simplex s; s.v[0] = a; s.v[1] = b; s.kind = EDGE; simplices.push_back(s); }
    void add_tri(int a, int b, int c) {
        Simplex s; s.v[0] = a; s.v[1] = b; s.v[2] = c; s.kind = TRIANGLE; simplices.push_back(s);
    }
};

// mesh.hpp:55-87 (throws on bad indices / exactly degenerate simplices)
inline void validate(const Mesh& m) {
    const auto n = std::int64_t(m.nv());
    for (std::size_t i = 0; i < m.ns(); ++i) {
        const Simplex& s = m.simplices[i];
        if (s.kind > TRIANGLE) fail("simplex " + std::to_string(i) + ": bad kind");
        for (int a = 0; a < s.nverts(); ++a)
            if (s.v[a] < 0 || s.v[a] >= n)
                fail("simplex " + std::to_string(i) + ": vertex index out of range");
        for (int a = 0; a < s.nverts(); ++a)
            for (int b = a + 1; b < s.nverts(); ++b)
                if (s.v[a] == s.v[b] || m.vertices[s.v[a]] == m.vertices[s.v[b]])
                    fail("degenerate simplex " + std::to_string(i));
        if (s.kind == TRIANGLE) {
            auto c = m.corners(s);
            if (norm(cross(c[1] - c[0], c[2] - c[0])) == 0.0)
                fail("degenerate simplex " + std::to_string(i) + " (zero area)");
        }
    }
}

inline Aabb bounding_box(const Mesh& m) {  // mesh.hpp:89-93
    Aabb b;
    for (const V3& p : m.vertices) b.expand(p);
    return b;
}

// mesh.hpp:137-183 -- valences: vertex = incident non-point simplices,
// edge = simplices (edges and triangles) containing the undirected edge.
inline std::uint64_t edge_key(std::int32_t a, std::int32_t b) {
    if (a > b) std::swap(a, b);
    return (std::uint64_t(std::uint32_t(a)) << 32) | std::uint32_t(b);
}
struct Adjacency {
    std::vector<std::int32_t> vertex_valence;
    std::unordered_map<std::uint64_t, std::int32_t> edge_count;
    std::int32_t edge_valence(std::int32_t a, std::int32_t b) const {
        auto it = edge_count.find(edge_key(a, b));
        return it == edge_count.end() ? 0 : it->second;
    }
};
inline Adjacency build_adjacency(const Mesh& m) {
    Adjacency adj;
    adj.vertex_valence.assign(m.nv(), 0);
    adj.edge_count.reserve(m.ns() * 2);
    for (const Simplex& s : m.simplices) {
        const int nv = s.nverts();
        if (nv > 1)
            for (int a = 0; a < nv; ++a) adj.vertex_valence[s.v[a]]++;
        if (nv == 2) {
            adj.edge_count[edge_key(s.v[0], s.v[1])]++;
        } else if (nv == 3) {
            adj.edge_count[edge_key(s.v[0], s.v[1])]++;
            adj.edge_count[edge_key(s.v[1], s.v[2])]++;
            adj.edge_count[edge_key(s.v[2], s.v[0])]++;
        }
    }
    return adj;
}

// ---------------------------------------------------------------- L2 exact
// exact.hpp:13-55 -- barycentrics on the data simplex and the closest pair.
struct Bary {
    double c[2] = {0, 0};
    int dim = 0;
};
struct Pair {
    double distance = 0;
    Bary phi;
    V3 point_f, point_g, grad;
};

// exact.hpp:59-63: d = |g - f|, grad = (g - f)/d, or 0 at contact.
inline void finish_pair(Pair& r) {
    const V3 diff = r.point_g - r.point_f;
    r.distance = norm(diff);
    r.grad = r.distance > 0.0 ? diff / r.distance : V3{};
}
inline double clamp01(double x) { return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x); }  // exact.hpp:65

// exact.hpp:68-73
inline double closest_on_segment(V3 a, V3 b, V3 p) {
    const V3 ab = b - a;
    const double den = sqnorm(ab);
    if (den <= 0.0) return 0.0;
    return clamp01(dot(ab, p - a) / den);
}

// exact.hpp:77-106 -- Voronoi-region case analysis (Ericson). Returns (u, v)
// with point = a + u (b - a) + v (c - a).
inline void closest_on_triangle(V3 a, V3 b, V3 c, V3 p, double& u, double& v) {
    const V3 ab = b - a, ac = c - a, ap = p - a;
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) { u = 0; v = 0; return; }
    const V3 bp = p - b;
    const double d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) { u = 1; v = 0; return; }
    const V3 cp = p - c;
    const double d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) { u = 0; v = 1; return; }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) { u = d1 / (d1 - d3); v = 0; return; }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) { u = 0; v = d2 / (d2 - d6); return; }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        u = 1.0 - t; v = t; return;
    }
    const double den = 1.0 / (va + vb + vc);
    u = vb * den; v = vc * den;
}

// exact.hpp:317-337 -- point-query fast path; f given by its corners.
inline Pair point_simplex_distance(const std::array<V3, 3>& f, int dim, V3 q) {
    Pair r;
    r.point_g = q;
    if (dim == 0) {
        r.point_f = f[0];
    } else if (dim == 1) {
        const double t = closest_on_segment(f[0], f[1], q);
        r.phi.c[0] = t; r.phi.dim = 1;
        r.point_f = f[0] + t * (f[1] - f[0]);                       // SimplexGeom::at, exact.hpp:38
    } else {
        double u, v;
        closest_on_triangle(f[0], f[1], f[2], q, u, v);
        r.phi.c[0] = u; r.phi.c[1] = v; r.phi.dim = 2;
        r.point_f = f[0] + u * (f[1] - f[0]) + v * (f[2] - f[0]);   // exact.hpp:39
    }
    finish_pair(r);
    return r;
}

// exact.hpp:377-394 -- brute-force minimum (point queries).
struct ExactMin {
    double distance = INFINITY;
    std::size_t argmin = 0;
};
inline ExactMin exact_min_distance(const Mesh& m, V3 q) {
    ExactMin res;
    for (std::size_t i = 0; i < m.ns(); ++i) {
        const Pair p = point_simplex_distance(m.corners(m.simplices[i]), m.simplices[i].dim(), q);
        if (p.distance < res.distance) { res.distance = p.distance; res.argmin = i; }
    }
    return res;
}

// ---------------------------------------------------------------- L2 weights
// weights.hpp:33-44 -- quartic edge weight in t; a1 == 0 by construction.
struct EdgePoly {
    double a[5] = {1, 0, 0, 0, 0};
    std::int32_t valence0 = 1, valence1 = 1;
    double sup = 1.0, inf = 1.0;
    double value(double t) const { return a[0] + t * (a[1] + t * (a[2] + t * (a[3] + t * a[4]))); }
    double derivative(double t) const { return a[1] + t * (2 * a[2] + t * (3 * a[3] + t * 4 * a[4])); }
};

// weights.hpp:46-76 -- closed form of the 5x5 interpolation system.
inline EdgePoly build_edge_weight(std::int32_t n0, std::int32_t n1) {
    EdgePoly p;
    p.valence0 = n0; p.valence1 = n1;
    const double P = 1.0 / n1 - 1.0 / n0, Q = 1.0 - 1.0 / n0;
    const double a[5] = {1.0 / n0, 0.0, -5 * P + 16 * Q, 14 * P - 32 * Q, 16 * Q - 8 * P};
    std::memcpy(p.a, a, sizeof a);
    p.sup = std::max(p.value(0.0), p.value(1.0));
    p.inf = std::min(p.value(0.0), p.value(1.0));
    auto consider = [&](double t) {
        if (t > 0.0 && t < 1.0) { const double w = p.value(t); p.sup = std::max(p.sup, w); p.inf = std::min(p.inf, w); }
    };
    // interior critical points: roots of 4 a4 t^2 + 3 a3 t + 2 a2
    const double qa = 4 * p.a[4], qb = 3 * p.a[3], qc = 2 * p.a[2];
    if (std::abs(qa) > 1e-300) {
        const double disc = qb * qb - 4 * qa * qc;
        if (disc >= 0.0) {
            const double rt = std::sqrt(disc);
            consider((-qb + rt) / (2 * qa));
            consider((-qb - rt) / (2 * qa));
        }
    } else if (std::abs(qb) > 1e-300) {
        consider(-qc / qb);
    }
    return p;
}

using Grid8 = std::array<std::array<double, 8>, 8>;

// weights.hpp:103-111 -- padded 8x8 Horner (kept: it is the reference cost).
inline double tri_horner(const Grid8& m, double x, double y) {
    double acc = 0.0;
    for (int j = 7; j >= 0; --j) {
        double row = 0.0;
        for (int k = 7; k >= 0; --k) row = row * y + m[j][k];
        acc = acc * x + row;
    }
    return acc;
}

// weights.hpp:116-131 -- the 13 stored (j <= k) coefficient slots.
inline constexpr int kTriStored[13][2] = {{0, 0}, {0, 2}, {0, 3}, {0, 4}, {0, 5}, {0, 6}, {0, 7},
                                          {2, 2}, {2, 3}, {2, 4}, {2, 5}, {3, 3}, {3, 4}};

// weights.hpp:138-171
struct TriPoly {
    double stored[13] = {};
    std::int32_t vertex_valence = 1, edge_valence = 1;
    double sup = 1.0, inf = 1.0, residual = 0.0;
    Grid8 c{}, dx{}, dy{};
    double value(double x, double y) const { return tri_horner(c, x, y); }
    double deriv_x(double x, double y) const { return tri_horner(dx, x, y); }
    double deriv_y(double x, double y) const { return tri_horner(dy, x, y); }
    void expand() {  // weights.hpp:155-170
        for (auto& r : c) r.fill(0.0);
        for (int m = 0; m < 13; ++m) {
            c[kTriStored[m][0]][kTriStored[m][1]] = stored[m];
            c[kTriStored[m][1]][kTriStored[m][0]] = stored[m];
        }
        for (auto& r : dx) r.fill(0.0);
        for (auto& r : dy) r.fill(0.0);
        for (int j = 0; j <= 7; ++j)
            for (int k = 0; k + j <= 7; ++k) {
                if (j > 0) dx[j - 1][k] += j * c[j][k];
                if (k > 0) dy[j][k - 1] += k * c[j][k];
            }
    }
};

TriPoly build_tri_weight(std::int32_t vertex_valence, std::int32_t edge_valence);  // weights_build.cpp

// weights.hpp:565-579
struct WeightSet {
    double A = 1.0, sup_wtilde = 1.0;
    std::vector<EdgePoly> edge_polys;
    std::vector<TriPoly> tri_polys;
    std::vector<std::int32_t> poly_index;  // -1: point / unit weight
    double max_attenuated_weight(const Params& p) const {  // :576-578
        return std::pow(std::max(A * sup_wtilde, 1e-300), p.attenuation());
    }
};

inline WeightSet unit_weight_set(const Mesh& m) {  // weights.hpp:583-587
    WeightSet ws;
    ws.poly_index.assign(m.ns(), -1);
    return ws;
}

// Process-wide memo of triangle polynomials: the build is deterministic in
// (v, e) and costs seconds; the reference rebuilds per mesh.
TriPoly cached_tri_weight(std::int32_t v, std::int32_t e);

// weights.hpp:589-621 -- polynomials assigned in first-occurrence order.
inline WeightSet build_weight_set(const Mesh& m, const Adjacency& adj) {
    WeightSet ws;
    ws.poly_index.assign(m.ns(), -1);
    std::map<std::pair<std::int32_t, std::int32_t>, std::int32_t> ecache, tcache;
    for (std::size_t i = 0; i < m.ns(); ++i) {
        const Simplex& s = m.simplices[i];
        if (s.kind == POINT) continue;
        if (s.kind == EDGE) {
            const std::int32_t n0 = adj.vertex_valence[s.v[0]], n1 = adj.vertex_valence[s.v[1]];
            auto [it, fresh] = ecache.try_emplace({n0, n1}, std::int32_t(ws.edge_polys.size()));
            if (fresh) ws.edge_polys.push_back(build_edge_weight(n0, n1));
            ws.poly_index[i] = it->second;
            ws.A = std::max(ws.A, double(std::max(n0, n1)));
            ws.sup_wtilde = std::max(ws.sup_wtilde, ws.edge_polys[it->second].sup);
        } else {
            const std::int32_t v = std::max({adj.vertex_valence[s.v[0]], adj.vertex_valence[s.v[1]],
                                             adj.vertex_valence[s.v[2]]});
            const std::int32_t e = std::max({adj.edge_valence(s.v[0], s.v[1]), adj.edge_valence(s.v[1], s.v[2]),
                                             adj.edge_valence(s.v[2], s.v[0])});
            auto [it, fresh] = tcache.try_emplace({v, e}, std::int32_t(ws.tri_polys.size()));
            if (fresh) ws.tri_polys.push_back(cached_tri_weight(v, e));
            ws.poly_index[i] = it->second;
            ws.A = std::max(ws.A, double(v));
            ws.sup_wtilde = std::max(ws.sup_wtilde, ws.tri_polys[it->second].sup);
        }
    }
    return ws;
}

// weights.hpp:624-642
inline void evaluate_wtilde(const Mesh& m, const WeightSet& ws, std::size_t i, const Bary& phi,
                            double& value, double g[2]) {
    const Simplex& s = m.simplices[i];
    g[0] = g[1] = 0.0;
    if (s.kind == POINT || ws.poly_index[i] < 0) { value = 1.0; return; }
    if (s.kind == EDGE) {
        const EdgePoly& p = ws.edge_polys[ws.poly_index[i]];
        value = p.value(phi.c[0]);
        g[0] = p.derivative(phi.c[0]);
        return;
    }
    const TriPoly& p = ws.tri_polys[ws.poly_index[i]];
    value = p.value(phi.c[0], phi.c[1]);
    g[0] = p.deriv_x(phi.c[0], phi.c[1]);
    g[1] = p.deriv_y(phi.c[0], phi.c[1]);
}

// weights.hpp:650-666 -- w = (A w~)^S, floored at 1e-300.
inline void evaluate_weight(const Mesh& m, const WeightSet& ws, std::size_t i, const Bary& phi,
                            const Params& prm, double& w, double dw[2]) {
    double wt, g[2];
    evaluate_wtilde(m, ws, i, phi, wt, g);
    const double S = prm.attenuation();
    const double base = ws.A * wt;
    if (base <= 1e-300) {
        w = std::pow(1e-300, S);
        dw[0] = dw[1] = 0.0;
        return;
    }
    w = std::pow(base, S);
    const double chain = S * std::pow(base, S - 1.0) * ws.A;
    dw[0] = chain * g[0];
    dw[1] = chain * g[1];
}

// weights.hpp:675-697 -- world gradient with alpha-scaled shape gradients.
// Re-evaluates the weight (second evaluate_weight call, :681) as the
// reference does.
inline V3 weight_gradient_world(const Mesh& m, const WeightSet& ws, std::size_t i, const Bary& phi,
                                const Params& prm) {
    const Simplex& s = m.simplices[i];
    if (s.kind == POINT || ws.poly_index[i] < 0) return {};
    double w, dw[2];
    evaluate_weight(m, ws, i, phi, prm, w, dw);
    const auto c = m.corners(s);
    if (s.kind == EDGE) {
        const V3 e = c[1] - c[0];
        const V3 gt = e / (prm.alpha * sqnorm(e));
        return dw[0] * gt;
    }
    const V3 e1 = c[1] - c[0], e2 = c[2] - c[0];
    const V3 n2 = cross(e1, e2);
    const double den = sqnorm(n2);
    if (den <= 0.0) return {};
    const V3 g1 = cross(n2, c[0] - c[2]) / (prm.alpha * den);
    const V3 g2 = cross(n2, c[1] - c[0]) / (prm.alpha * den);
    return dw[0] * g1 + dw[1] * g2;
}

// ---------------------------------------------------------------- L2 bvh
// bvh.hpp:14-32 -- binary reference layout, 72 B per node, root 0,
// pre-order ids (left subtree immediately follows its parent).
struct BvhNode {
    Aabb box;
    std::int32_t left = -1, right = -1, primitive = -1, count = 0;
    double diameter = 0.0;
    bool is_leaf() const { return left < 0; }
};
static_assert(sizeof(BvhNode) == 72, "reference BvhNode is 72 bytes");
struct Bvh {
    std::vector<BvhNode> nodes;
    bool empty() const { return nodes.empty(); }
};

// bvh.hpp:34-91 -- longest-axis median split on bbox-centre centroids,
// (centroid, index) ordering; the partition sets are unique, so the tree
// is independent of nth_element's internal arrangement.
inline Bvh build_bvh(const Mesh& m) {
    Bvh bvh;
    const std::size_t n = m.ns();
    if (n == 0) return bvh;
    std::vector<Aabb> boxes(n);
    std::vector<V3> cent(n);
    for (std::size_t i = 0; i < n; ++i) {
        const Simplex& s = m.simplices[i];
        const auto c = m.corners(s);
        for (int k = 0; k < s.nverts(); ++k) boxes[i].expand(c[k]);
        cent[i] = boxes[i].center();
    }
    std::vector<std::int32_t> order(n);
    for (std::size_t i = 0; i < n; ++i) order[i] = std::int32_t(i);
    bvh.nodes.reserve(2 * n - 1);
    // recursion depth is ceil(log2 n) (balanced median split)
    auto build = [&](auto&& self, std::size_t first, std::size_t last) -> std::int32_t {
        const std::int32_t id = std::int32_t(bvh.nodes.size());
        bvh.nodes.emplace_back();
        if (last - first == 1) {
            BvhNode& leaf = bvh.nodes[id];
            leaf.primitive = order[first];
            leaf.count = 1;
            leaf.box = boxes[order[first]];
            leaf.diameter = leaf.box.diagonal();
            return id;
        }
        Aabb box;
        for (std::size_t i = first; i < last; ++i) box.expand(boxes[order[i]]);
        const V3 ext = box.extent();
        int axis = 0;
        if (ext.y > ext.x) axis = 1;
        if (ext.z > ext[axis]) axis = 2;
        const std::size_t mid = first + (last - first) / 2;
        std::nth_element(order.begin() + first, order.begin() + mid, order.begin() + last,
                         [&](std::int32_t a, std::int32_t b) {
                             const double ca = cent[a][axis], cb = cent[b][axis];
                             if (ca != cb) return ca < cb;
                             return a < b;
                         });
        const std::int32_t l = self(self, first, mid);
        const std::int32_t r = self(self, mid, last);
        BvhNode& node = bvh.nodes[id];
        node.left = l;
        node.right = r;
        node.count = bvh.nodes[l].count + bvh.nodes[r].count;
        node.box = bvh.nodes[l].box;
        node.box.expand(bvh.nodes[r].box);
        node.diameter = node.box.diagonal();
        return id;
    };
    build(build, 0, n);
    return bvh;
}

// bvh.hpp:98-111
struct BoxProx {
    double distance = 0.0;
    V3 y_b;
    bool must_descend = false;
};
inline BoxProx box_point_proximity(const Aabb& box, V3 q) {
    BoxProx r;
    r.y_b = box.closest_point(q);
    r.distance = norm(q - r.y_b);
    return r;
}
// bvh.hpp:185-187 (strict inequality; contact always descends)
inline bool bh_condition(const BvhNode& node, const BoxProx& p, double beta) {
    return !p.must_descend && p.distance > 0.0 && node.diameter < beta * p.distance;
}

// ---------------------------------------------------------------- L3 smooth
// smooth.hpp:20-27
struct Result {
    double d_hat = INFINITY;
    V3 grad;
    double c = 0.0;
    V3 grad_c;
    std::int64_t leaves = 0, far_field = 0;
    std::uint64_t decision_hash = 0;  // oracle-only instrumentation (see decision_mix)
};

// smooth.hpp:33-45
struct Scratch {
    std::vector<double> args, coefs, vals;
    std::vector<V3> gcoefs;
    std::vector<std::int32_t> stack;
    void clear() { args.clear(); coefs.clear(); gcoefs.clear(); }
};

// Order-independent decision fingerprint: sum (mod 2^64) over decided
// nodes of splitmix64(node_id * 4 + kind), kind 1 = far field, 2 = exact
// leaf. Shared bit-for-bit with the GPU traversal (csrc/common.cuh).
inline std::uint64_t decision_mix(std::uint64_t node, std::uint64_t kind) {
    std::uint64_t z = node * 4 + kind + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// smooth.hpp:51-61
inline void push_leaf_term(const Mesh& m, const WeightSet& ws, std::size_t prim, V3 q, const Params& prm,
                           Scratch& s) {
    const Simplex& sx = m.simplices[prim];
    const Pair p = point_simplex_distance(m.corners(sx), sx.dim(), q);
    double w, dw[2];
    evaluate_weight(m, ws, prim, p.phi, prm, w, dw);
    const V3 gw = weight_gradient_world(m, ws, prim, p.phi, prm);
    s.args.push_back(-prm.alpha * p.distance);
    s.coefs.push_back(w);
    s.gcoefs.push_back(w * p.grad - gw / prm.alpha);
}

// smooth.hpp:67-75
inline void push_far_field_term(const BvhNode& node, const BoxProx& prox, V3 q, double w_ff,
                                const Params& prm, Scratch& s) {
    const V3 diff = q - prox.y_b;
    const double scale = node.count * w_ff;
    s.args.push_back(-prm.alpha * prox.distance);
    s.coefs.push_back(scale);
    s.gcoefs.push_back((scale / prox.distance) * diff);
}

// smooth.hpp:79-93 -- recording-order sum, exp args < -708 forced to 0.
inline void finalize_terms(Scratch& s, double& c, V3& gc) {
    c = 0.0;
    gc = V3{};
    const std::size_t n = s.args.size();
    s.vals.resize(n);
    for (std::size_t i = 0; i < n; ++i) s.vals[i] = s.args[i] < -708.0 ? 0.0 : std::exp(s.args[i]);
    for (std::size_t i = 0; i < n; ++i) {
        c += s.coefs[i] * s.vals[i];
        gc += s.vals[i] * s.gcoefs[i];
    }
}

// smooth.hpp:101-131 (point queries). beta > 0 box-tests every popped node,
// leaves included; left child pops first.
inline void collect_contributions(const Mesh& m, const Bvh& bvh, const WeightSet& ws, V3 q,
                                  const Params& prm, Scratch& s, Result& st) {
    if (bvh.empty()) return;
    const double w_ff = ws.max_attenuated_weight(prm);
    const bool use_bh = prm.beta > 0.0;
    s.stack.clear();
    s.stack.push_back(0);
    while (!s.stack.empty()) {
        const std::int32_t id = s.stack.back();
        s.stack.pop_back();
        const BvhNode& node = bvh.nodes[id];
        if (use_bh) {
            const BoxProx prox = box_point_proximity(node.box, q);
            if (bh_condition(node, prox, prm.beta)) {
                push_far_field_term(node, prox, q, w_ff, prm, s);
                ++st.far_field;
                st.decision_hash += decision_mix(std::uint64_t(id), 1);
                continue;
            }
        }
        if (node.is_leaf()) {
            push_leaf_term(m, ws, std::size_t(node.primitive), q, prm, s);
            ++st.leaves;
            st.decision_hash += decision_mix(std::uint64_t(id), 2);
        } else {
            s.stack.push_back(node.right);
            s.stack.push_back(node.left);
        }
    }
}

// smooth.hpp:147-159
inline Result result_from_accum(Scratch& s, Result st, const Params& prm) {
    Result r = st;
    finalize_terms(s, r.c, r.grad_c);
    if (r.c <= 0.0) {
        r.d_hat = INFINITY;
        r.grad = V3{};
        return r;
    }
    r.d_hat = -std::log(r.c) / prm.alpha;
    r.grad = r.grad_c / (r.c + prm.epsilon);
    return r;
}

// smooth.hpp:166-184
inline Result smooth_min_dist(const Mesh& m, const Bvh& bvh, const WeightSet& ws, V3 q, const Params& prm,
                              Scratch& s) {
    s.clear();
    Result st;
    collect_contributions(m, bvh, ws, q, prm, s, st);
    return result_from_accum(s, st, prm);
}

// smooth.hpp:189-198 -- flat exact oracle over every primitive in index order.
inline Result smooth_min_dist_flat(const Mesh& m, const WeightSet& ws, V3 q, const Params& prm, Scratch& s) {
    s.clear();
    Result st;
    for (std::size_t i = 0; i < m.ns(); ++i) {
        push_leaf_term(m, ws, i, q, prm, s);
        ++st.leaves;
    }
    return result_from_accum(s, st, prm);
}

// parallel.hpp:25-44 -- static contiguous partition over std::threads.
template <class Fn>
void parallel_for(std::int64_t n, int threads, Fn&& fn);

// smooth.hpp:212-255 -- mesh-to-mesh distance: outer LogSumExp (alpha_q)
// over the inner smooth distances of the query simplices, per-vertex
// gradients by splitting each simplex's softmin mass over its vertices.
// Restated for query meshes of point simplices (the inner query is then the
// point path; edge/triangle query simplices need the QP kernels, which are
// outside this path).
struct MeshDist {
    double d_hat = INFINITY;
    std::vector<V3> vertex_grads;
    std::vector<double> per_primitive;
    std::int64_t leaves = 0, far_field = 0;
};
inline MeshDist smooth_mesh_dist_points(const Mesh& m, const Bvh* bvh, const WeightSet& ws, const Mesh& query,
                                        const Params& prm, int threads) {
    const std::size_t nq = query.ns();
    MeshDist out;
    out.vertex_grads.assign(query.nv(), V3{});
    out.per_primitive.assign(nq, INFINITY);
    if (nq == 0) return out;
    for (const Simplex& s : query.simplices)
        if (s.kind != POINT) fail("smooth_mesh_dist_points: query simplices must be points");
    std::vector<V3> inner(nq);
    std::vector<std::int64_t> leaves(nq, 0), far(nq, 0);
    parallel_for(std::int64_t(nq), threads, [&](std::int64_t b, std::int64_t e, int) {
        Scratch s;
        for (std::int64_t j = b; j < e; ++j) {
            const V3 q = query.vertices[query.simplices[std::size_t(j)].v[0]];
            const Result r = bvh ? smooth_min_dist(m, *bvh, ws, q, prm, s) : smooth_min_dist_flat(m, ws, q, prm, s);
            out.per_primitive[std::size_t(j)] = r.d_hat;
            inner[std::size_t(j)] = r.grad;
            leaves[std::size_t(j)] = r.leaves;
            far[std::size_t(j)] = r.far_field;
        }
    });
    double denom = 0.0;  // serial, primitive order (smooth.hpp:237-245)
    for (std::size_t j = 0; j < nq; ++j) {
        out.leaves += leaves[j];
        out.far_field += far[j];
        const double mass = std::exp(-prm.alpha_q * out.per_primitive[j]);
        denom += mass;
        const Simplex& s = query.simplices[j];
        const double split = mass / s.nverts();
        for (int k = 0; k < s.nverts(); ++k) out.vertex_grads[s.v[k]] += split * inner[j];
    }
    if (denom <= 0.0) {
        for (V3& g : out.vertex_grads) g = V3{};
        return out;
    }
    out.d_hat = -std::log(denom) / prm.alpha_q;
    for (V3& g : out.vertex_grads) g = g / (denom + prm.epsilon);
    return out;
}

template <class Fn>
void parallel_for(std::int64_t n, int threads, Fn&& fn) {
    if (n <= 0) return;
    if (threads < 1) threads = 1;
    if (threads == 1 || n == 1) { fn(std::int64_t{0}, n, 0); return; }
    if (threads > n) threads = int(n);
    std::vector<std::thread> pool;
    const std::int64_t chunk = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const std::int64_t b = t * chunk, e = std::min(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&fn, b, e, t] { fn(b, e, t); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace sdo
