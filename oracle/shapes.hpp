// oracle/shapes.hpp -- TEST INFRASTRUCTURE ONLY.
//
// Seeded procedural geometry: a restatement of the reference generators
// (shapes.hpp:25-265, std::mt19937_64 + libstdc++ distributions). The
// generators keep the reference's expression shapes (e.g. V3(u(rng),
// u(rng), u(rng))) because argument evaluation order decides the draw order
// and g++ (right to left) is what the reference is built with; the seeded
// test scenes are thereby reproduced draw for draw. Also holds the
// five BASELINE.json workload configs, with the interpretations frozen in
// SURVEY.md 8(d). No public dataset is involved; these synthetic inputs
// stand in for the paper's Thingi10K corpus.
#pragma once

#include "sdoracle.hpp"

#include <random>

namespace sdo {

using Rng = std::mt19937_64;

struct Mat3 {
    double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
    V3 operator*(V3 v) const {
        return {m[0][0] * v.x + m[0][1] * v.y + m[0][2] * v.z, m[1][0] * v.x + m[1][1] * v.y + m[1][2] * v.z,
                m[2][0] * v.x + m[2][1] * v.y + m[2][2] * v.z};
    }
};

// shapes.hpp:25-63 (midpoint map keyed by the sorted vertex pair; vertex
// ids follow first-creation order exactly as with the reference std::map)
inline Mesh icosphere(int subdivisions = 1, double radius = 1.0, V3 center = {}) {
    const double t = (1.0 + std::sqrt(5.0)) / 2.0;
    std::vector<V3> verts = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t},  {0, 1, t},
                             {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
    std::vector<std::array<std::int32_t, 3>> faces = {
        {0, 11, 5}, {0, 5, 1}, {0, 1, 7},  {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
        {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4},  {3, 4, 2},   {3, 2, 6}, {3, 6, 8},
        {3, 8, 9},  {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7},   {9, 8, 1}};
    for (int s = 0; s < subdivisions; ++s) {
        std::unordered_map<std::uint64_t, std::int32_t> mid_of;
        mid_of.reserve(faces.size() * 2);
        auto mid = [&](std::int32_t a, std::int32_t b) {
            auto [it, fresh] = mid_of.try_emplace(edge_key(a, b), std::int32_t(verts.size()));
            if (fresh) verts.push_back(0.5 * (verts[a] + verts[b]));
            return it->second;
        };
        std::vector<std::array<std::int32_t, 3>> next;
        next.reserve(4 * faces.size());
        for (const auto& f : faces) {
            const std::int32_t ab = mid(f[0], f[1]), bc = mid(f[1], f[2]), ca = mid(f[2], f[0]);
            next.push_back({f[0], ab, ca});
            next.push_back({f[1], bc, ab});
            next.push_back({f[2], ca, bc});
            next.push_back({ab, bc, ca});
        }
        faces.swap(next);
    }
    Mesh m;
    m.vertices.reserve(verts.size());
    for (const V3& v : verts) m.vertices.push_back(center + radius * normalized(v));
    m.simplices.reserve(faces.size());
    for (const auto& f : faces) m.add_tri(f[0], f[1], f[2]);
    return m;
}

// shapes.hpp:67-89 -- ring in x-z, tube in y; valence 6 / edge valence 2.
inline Mesh uv_torus(double major = 0.35, double minor = 0.15, int nu = 60, int nv = 60, V3 center = {}) {
    Mesh m;
    m.vertices.reserve(std::size_t(nu) * nv);
    for (int i = 0; i < nu; ++i) {
        const double u = 2 * M_PI * i / nu;
        for (int j = 0; j < nv; ++j) {
            const double v = 2 * M_PI * j / nv;
            const double ring = major + minor * std::cos(v);
            m.vertices.push_back(center + V3(ring * std::cos(u), minor * std::sin(v), ring * std::sin(u)));
        }
    }
    auto vid = [&](int i, int j) { return std::int32_t((i % nu) * nv + (j % nv)); };
    m.simplices.reserve(std::size_t(2) * nu * nv);
    for (int i = 0; i < nu; ++i)
        for (int j = 0; j < nv; ++j) {
            m.add_tri(vid(i, j), vid(i + 1, j), vid(i, j + 1));
            m.add_tri(vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1));
        }
    return m;
}

// shapes.hpp:92-110
inline Mesh grid_patch(int nx, int ny, double size = 1.0, double height_jitter = 0.0, std::uint64_t seed = 0) {
    Rng rng(seed);
    std::uniform_real_distribution<double> jit(-height_jitter, height_jitter);
    Mesh m;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i)
            m.vertices.push_back(V3(size * i / (nx - 1), size * j / (ny - 1), height_jitter > 0 ? jit(rng) : 0.0));
    auto vid = [&](int i, int j) { return std::int32_t(j * nx + i); };
    for (int j = 0; j + 1 < ny; ++j)
        for (int i = 0; i + 1 < nx; ++i) {
            m.add_tri(vid(i, j), vid(i + 1, j), vid(i, j + 1));
            m.add_tri(vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1));
        }
    return m;
}

// shapes.hpp:114-119
inline V3 random_unit(Rng& rng) {
    std::normal_distribution<double> n(0.0, 1.0);
    // same expression shape as the reference: g++ evaluates constructor
    // arguments right to left, so the draw order follows automatically
    V3 v(n(rng), n(rng), n(rng));
    while (norm(v) < 1e-8) v = V3(n(rng), n(rng), n(rng));
    return normalized(v);
}

// shapes.hpp:121-125 -- axis-angle (Rodrigues) matrix, Eigen AngleAxis layout.
inline Mat3 random_rotation(Rng& rng) {
    const V3 ax = random_unit(rng);
    std::uniform_real_distribution<double> angle(0.0, 2 * M_PI);
    const double a = angle(rng);
    const V3 sa = std::sin(a) * ax;
    const double c = std::cos(a);
    const V3 c1 = (1.0 - c) * ax;
    Mat3 r;
    double tmp = c1.x * ax.y;
    r.m[0][1] = tmp - sa.z; r.m[1][0] = tmp + sa.z;
    tmp = c1.x * ax.z;
    r.m[0][2] = tmp + sa.y; r.m[2][0] = tmp - sa.y;
    tmp = c1.y * ax.z;
    r.m[1][2] = tmp - sa.x; r.m[2][1] = tmp + sa.x;
    r.m[0][0] = c1.x * ax.x + c; r.m[1][1] = c1.y * ax.y + c; r.m[2][2] = c1.z * ax.z + c;
    return r;
}

// shapes.hpp:127-135
inline void append_mesh(Mesh& dst, const Mesh& src, const Mat3& rot, V3 shift, double scale) {
    const auto base = std::int32_t(dst.nv());
    for (const V3& v : src.vertices) dst.vertices.push_back(rot * (scale * v) + shift);
    for (Simplex s : src.simplices) {
        for (int k = 0; k < s.nverts(); ++k) s.v[k] += base;
        dst.simplices.push_back(s);
    }
}

// shapes.hpp:140-156
inline Mesh triangle_strip(int n, Rng& rng) {
    std::uniform_real_distribution<double> off(-0.15, 0.15);
    Mesh m;
    const int cols = (n + 1) / 2 + 1;
    for (int i = 0; i < cols; ++i) {
        m.vertices.push_back(V3(i * 0.4 + off(rng), off(rng), off(rng)));
        m.vertices.push_back(V3(i * 0.4 + off(rng), 0.4 + off(rng), off(rng)));
    }
    for (int k = 0; k < n; ++k) {
        const std::int32_t i = k / 2;
        if (k % 2 == 0) m.add_tri(2 * i, 2 * i + 2, 2 * i + 1);
        else m.add_tri(2 * i + 2, 2 * i + 3, 2 * i + 1);
    }
    return m;
}

// shapes.hpp:159-170
inline Mesh triangle_fan(int k, Rng& rng) {
    std::uniform_real_distribution<double> rad(0.3, 0.6), lift(-0.1, 0.1);
    Mesh m;
    m.vertices.push_back(V3(0, 0, 0));
    for (int i = 0; i <= k; ++i) {
        const double a = M_PI * 1.6 * i / k;
        const double r = rad(rng);
        m.vertices.push_back(V3(r * std::cos(a), r * std::sin(a), lift(rng)));
    }
    for (int i = 1; i <= k; ++i) m.add_tri(0, i, i + 1);
    return m;
}

// shapes.hpp:173-184
inline Mesh polyline(int n, Rng& rng) {
    std::uniform_real_distribution<double> step(0.1, 0.35);
    Mesh m;
    V3 p(0, 0, 0);
    m.vertices.push_back(p);
    for (int i = 0; i < n; ++i) {
        p += step(rng) * random_unit(rng);
        m.vertices.push_back(p);
        m.add_edge(i, i + 1);
    }
    return m;
}

// shapes.hpp:186-194
inline Mesh point_cluster(int n, Rng& rng, double spread = 0.4) {
    std::uniform_real_distribution<double> u(-spread, spread);
    Mesh m;
    for (int i = 0; i < n; ++i) {
        m.vertices.push_back(V3(u(rng), u(rng), u(rng)));
        m.add_point(i);
    }
    return m;
}

// shapes.hpp:198-240
inline Mesh random_scene(std::uint64_t seed, int max_prims = 200) {
    Rng rng(seed);
    std::uniform_int_distribution<int> npieces(1, 4), kind(0, 4);
    std::uniform_real_distribution<double> scale(0.5, 1.5), place(-1.0, 1.0);
    Mesh m;
    const int pieces = npieces(rng);
    for (int p = 0; p < pieces; ++p) {
        const int budget = max_prims - int(m.ns());
        if (budget < 2) break;
        Mesh piece;
        switch (kind(rng)) {
            case 0:
                piece = triangle_strip(std::uniform_int_distribution<int>(2, std::min(40, budget))(rng), rng);
                break;
            case 1:
                piece = triangle_fan(std::uniform_int_distribution<int>(2, std::min(8, budget))(rng), rng);
                break;
            case 2: {
                const int nx = std::uniform_int_distribution<int>(2, 5)(rng);
                const int ny = std::uniform_int_distribution<int>(2, 5)(rng);
                if (2 * (nx - 1) * (ny - 1) > budget) piece = triangle_strip(2, rng);
                else piece = grid_patch(nx, ny, 1.0, 0.15, rng());
                break;
            }
            case 3:
                piece = polyline(std::uniform_int_distribution<int>(1, std::min(30, budget))(rng), rng);
                break;
            default:
                piece = point_cluster(std::uniform_int_distribution<int>(1, std::min(30, budget))(rng), rng);
                break;
        }
        append_mesh(m, piece, random_rotation(rng), V3(place(rng), place(rng), place(rng)), scale(rng));
    }
    if (m.ns() == 0) m = point_cluster(4, rng);
    return m;
}

// shapes.hpp:243-265 -- random query simplex (all kinds drawn, so the RNG
// stream matches the reference; only dim-0 queries are on the hot path).
struct QuerySimplex {
    std::array<V3, 3> c{};
    int dim = 0;
};
inline QuerySimplex random_query(Rng& rng, const Aabb& box, double size_scale = 0.3) {
    std::uniform_int_distribution<int> kind(0, 2);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    const V3 ext = box.extent();
    const V3 pad = 0.5 * vmax(ext, V3(0.2, 0.2, 0.2));
    const V3 lo = box.lo - pad, hi = box.hi + pad;
    auto sample = [&] {
        return V3(lo.x + u(rng) * (hi.x - lo.x), lo.y + u(rng) * (hi.y - lo.y), lo.z + u(rng) * (hi.z - lo.z));
    };
    QuerySimplex q;
    const V3 a = sample();
    q.c[0] = a;
    switch (kind(rng)) {
        case 0: q.dim = 0; break;
        case 1: q.dim = 1; q.c[1] = a + size_scale * random_unit(rng); break;
        default: {
            const V3 e1 = size_scale * random_unit(rng);
            V3 e2 = size_scale * random_unit(rng);
            while (norm(cross(e1, e2)) < 1e-6) e2 = size_scale * random_unit(rng);
            q.dim = 2; q.c[1] = a + e1; q.c[2] = a + e2;
        }
    }
    return q;
}

// ------------------------------------------------ BASELINE.json configs
inline double mean_unique_edge_length(const Mesh& m) {
    std::unordered_map<std::uint64_t, char> seen;
    seen.reserve(m.ns() * 2);
    double sum = 0.0;
    std::int64_t n = 0;
    for (const Simplex& s : m.simplices) {
        const int nv = s.nverts();
        if (nv < 2) continue;
        for (int a = 0; a < nv; ++a) {
            const int b = (a + 1) % nv;
            if (nv == 2 && a == 1) break;
            if (seen.emplace(edge_key(s.v[a], s.v[b]), 1).second) {
                sum += norm(m.vertices[s.v[a]] - m.vertices[s.v[b]]);
                ++n;
            }
        }
    }
    return n ? sum / double(n) : 0.0;
}

inline void jitter_vertices(Mesh& m, double sigma, Rng& rng) {
    std::normal_distribution<double> n(0.0, sigma);
    for (V3& v : m.vertices) {
        const double a = n(rng), b = n(rng), c = n(rng);
        v = v + V3(a, b, c);
    }
}

// cfg3 mesh: uv_torus(1, 0.3, 512, 256) with N(0, (0.1 * mean edge)^2) jitter.
inline Mesh cfg3_torus(std::uint64_t seed = 3001) {
    Mesh m = uv_torus(1.0, 0.3, 512, 256);
    const double sigma = 0.1 * mean_unique_edge_length(m);
    Rng rng(seed);
    jitter_vertices(m, sigma, rng);
    return m;
}

// uniform sample on a triangle of the mesh (uniform triangle index,
// uniform barycentric via the square-root map) and its unit normal
inline V3 surface_sample(const Mesh& m, std::int64_t tri_begin, std::int64_t tri_end, Rng& rng, V3* normal_out) {
    std::uniform_int_distribution<std::int64_t> pick(tri_begin, tri_end - 1);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    const Simplex& s = m.simplices[pick(rng)];
    const double r1 = u(rng), r2 = u(rng);
    const double sr = std::sqrt(r1);
    const double b0 = 1.0 - sr, b1 = sr * (1.0 - r2), b2 = sr * r2;
    const auto c = m.corners(s);
    if (normal_out) *normal_out = normalized(cross(c[1] - c[0], c[2] - c[0]));
    return b0 * c[0] + b1 * c[1] + b2 * c[2];
}

inline Mesh config_mesh(int cfg) {
    switch (cfg) {
        case 1: {  // 4096 unit-sphere points
            Rng rng(1001);
            Mesh m;
            for (int i = 0; i < 4096; ++i) { m.vertices.push_back(random_unit(rng)); m.add_point(i); }
            return m;
        }
        case 2: {  // helix polyline, 20,000 edges, N(0, 1e-3^2) jitter
            Mesh m;
            const int K = 20000;
            for (int k = 0; k <= K; ++k) {
                const double t = 40.0 * M_PI * k / K;
                m.vertices.push_back(V3(std::cos(t), std::sin(t), 0.05 * t));
            }
            Rng rng(2001);
            jitter_vertices(m, 1e-3, rng);
            for (int k = 0; k < K; ++k) m.add_edge(k, k + 1);
            return m;
        }
        case 3:
            return cfg3_torus();
        case 4: {  // icosphere(9) with radial displacement
            Mesh m = icosphere(9);
            for (V3& v : m.vertices) {
                const double r = norm(v);
                const double th = std::acos(v.z / r), ph = std::atan2(v.y, v.x);
                v = (1.0 + 0.05 * std::sin(8 * th) * std::cos(8 * ph)) * v;
            }
            return m;
        }
        case 5: {  // 64 rotated tori + 1M edges + 1M points
            const Mesh torus = cfg3_torus();
            const double mel = mean_unique_edge_length(torus);
            Mesh m;
            m.vertices.reserve(64 * torus.nv() + 3000000);
            m.simplices.reserve(64 * torus.ns() + 2000000);
            Rng rng(5001);
            std::uniform_real_distribution<double> c(-10.0, 10.0);
            for (int i = 0; i < 64; ++i) {
                const Mat3 rot = random_rotation(rng);
                const double x = c(rng), y = c(rng), z = c(rng);
                append_mesh(m, torus, rot, V3(x, y, z), 1.0);
            }
            const std::int64_t ntri = std::int64_t(m.ns());
            Rng r3(5003);
            for (int i = 0; i < 1000000; ++i) {  // standalone edges along the surface
                V3 n;
                const V3 p = surface_sample(m, 0, ntri, r3, &n);
                V3 t = random_unit(r3);
                t = normalized(t - dot(t, n) * n);
                const auto base = std::int32_t(m.nv());
                m.vertices.push_back(p);
                m.vertices.push_back(p + mel * t);
                m.add_edge(base, base + 1);
            }
            for (int i = 0; i < 1000000; ++i) {  // isolated points on the surface
                const V3 p = surface_sample(m, 0, ntri, r3, nullptr);
                m.vertices.push_back(p);
                m.add_point(std::int32_t(m.nv()) - 1);
            }
            return m;
        }
    }
    fail("unknown config " + std::to_string(cfg));
}

// First nq queries of the config's seeded query stream (cfg4: nq/2 from
// each half, so subsets are prefixes of both halves).
inline std::vector<V3> config_queries(int cfg, const Mesh& m, std::int64_t nq) {
    std::vector<V3> q;
    q.reserve(std::size_t(nq));
    auto uniform_box = [&](V3 lo, V3 hi, std::uint64_t seed, std::int64_t n) {
        Rng rng(seed);
        std::uniform_real_distribution<double> ux(lo.x, hi.x), uy(lo.y, hi.y), uz(lo.z, hi.z);
        for (std::int64_t i = 0; i < n; ++i) {
            const double x = ux(rng), y = uy(rng), z = uz(rng);
            q.push_back(V3(x, y, z));
        }
    };
    const Aabb box = bounding_box(m);
    switch (cfg) {
        case 1: uniform_box(V3(-2, -2, -2), V3(2, 2, 2), 1002, nq); break;
        case 2: {
            const V3 c = box.center(), h = 0.6 * box.extent();  // AABB scaled x1.2 about its centre
            uniform_box(c - h, c + h, 2002, nq);
            break;
        }
        case 3: uniform_box(box.lo - V3(0.5, 0.5, 0.5), box.hi + V3(0.5, 0.5, 0.5), 3002, nq); break;
        case 4: {
            const std::int64_t h1 = nq / 2, h2 = nq - h1;
            uniform_box(V3(-1.5, -1.5, -1.5), V3(1.5, 1.5, 1.5), 4001, h1);
            Rng rng(4002);
            std::normal_distribution<double> off(0.0, 0.01);
            for (std::int64_t i = 0; i < h2; ++i) {
                V3 n;
                const V3 p = surface_sample(m, 0, std::int64_t(m.ns()), rng, &n);
                const double d = std::min(0.02, std::max(-0.02, off(rng)));
                q.push_back(p + d * n);
            }
            break;
        }
        case 5: uniform_box(box.lo, box.hi, 5002, nq); break;
        default: fail("unknown config " + std::to_string(cfg));
    }
    return q;
}

}  // namespace sdo
