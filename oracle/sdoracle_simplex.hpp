// oracle/sdoracle_simplex.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement (plain fp64, -ffp-contract=off) of the reference's
// SIMPLEX-query path: edge / triangle query primitives g instead of points.
// Same rules as sdoracle.hpp: only tests/, smoke() and bench.py's CPU legs
// load it; the product (paper_2108_10480_b200/csrc/simplex.cu) never does.
//
//   exact.hpp:13-55      SimplexGeom::at, Barycentric, ClosestPair
//   exact.hpp:110-141    closest_segment_segment
//   exact.hpp:143-313    simplex_distance_qp (face enumeration)
//   exact.hpp:342-367    simplex_distance dispatch
//   bvh.hpp:113-180      box_primitive_proximity (halfspace classification)
//   smooth.hpp:51-75     leaf / far-field terms for a query simplex
//   smooth.hpp:101-131   collect_contributions
//   smooth.hpp:166-198   smooth_min_dist / smooth_min_dist_flat
//   smooth.hpp:212-255   smooth_mesh_dist (any query mesh)
//
// The 3x3 normal-equation solve goes through Eigen's Matrix3d::determinant
// and ::inverse in the reference (exact.hpp:275-285). Eigen is not vendored
// (SURVEY 8c); its published fixed-size algorithms are restated: the
// determinant as the cofactor expansion along the first row (Eigen
// Determinant.h, bruteforce_det3_helper), the inverse as the cofactor
// transpose times 1/det (InverseImpl.h, compute_inverse_size3_helper), and
// the matrix-vector product summed left to right. The low bits of the 3x3
// path are therefore pinned to this restatement, not to an Eigen build.
#pragma once

#include "sdoracle.hpp"

namespace sdo {

// exact.hpp:24-41 -- a simplex by its corners; at() = c0 + b0 (c1 - c0) [+ b1 (c2 - c0)].
struct Geom {
    std::array<V3, 3> c{};
    int dim = 0;
    V3 at(const Bary& b) const {
        if (dim == 0) return c[0];
        if (dim == 1) return c[0] + b.c[0] * (c[1] - c[0]);
        return c[0] + b.c[0] * (c[1] - c[0]) + b.c[1] * (c[2] - c[0]);
    }
    static Geom point(V3 a) { Geom g; g.c[0] = a; return g; }
    static Geom edge(V3 a, V3 b) { Geom g; g.c[0] = a; g.c[1] = b; g.dim = 1; return g; }
    static Geom triangle(V3 a, V3 b, V3 c) { Geom g; g.c[0] = a; g.c[1] = b; g.c[2] = c; g.dim = 2; return g; }
    static Geom from_mesh(const Mesh& m, const Simplex& s) {
        Geom g;
        g.c = m.corners(s);
        g.dim = s.dim();
        return g;
    }
};

// exact.hpp:48-55 (both barycentrics kept)
struct GPair {
    double distance = 0;
    Bary phi, lambda;
    V3 point_f, point_g, grad;
};
inline void finish_pair(GPair& r) {  // exact.hpp:59-63
    const V3 diff = r.point_g - r.point_f;
    r.distance = norm(diff);
    r.grad = r.distance > 0.0 ? diff / r.distance : V3{};
}

// exact.hpp:317-337 with lambda = point
inline GPair point_geom_distance(const Geom& f, V3 q) {
    const Pair p = point_simplex_distance(f.c, f.dim, q);
    GPair r;
    r.distance = p.distance;
    r.phi = p.phi;
    r.point_f = p.point_f;
    r.point_g = p.point_g;
    r.grad = p.grad;
    return r;
}

// exact.hpp:110-141
inline void closest_segment_segment(V3 p1, V3 q1, V3 p2, V3 q2, double& s, double& t) {
    const V3 d1 = q1 - p1, d2 = q2 - p2, r = p1 - p2;
    const double a = sqnorm(d1), e = sqnorm(d2), f = dot(d2, r);
    constexpr double kTiny = 1e-30;
    if (a <= kTiny && e <= kTiny) { s = t = 0.0; return; }
    if (a <= kTiny) { s = 0.0; t = clamp01(f / e); return; }
    const double c = dot(d1, r);
    if (e <= kTiny) { t = 0.0; s = clamp01(-c / a); return; }
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

// exact.hpp:158-313 -- minimise |f(phi) - g(lambda)|^2 over the joint domain
// by enumerating the faces (active sets) of both simplices, vertices ->
// edges -> interior, keeping the first strictly best feasible candidate.
struct QpFace {
    double base[2];
    double dir[2][2];  // dir[param][bary coord]
    int k;
};
inline constexpr QpFace kQpPoint[] = {{{0, 0}, {{0, 0}, {0, 0}}, 0}};
inline constexpr QpFace kQpEdge[] = {
    {{0, 0}, {{0, 0}, {0, 0}}, 0},
    {{1, 0}, {{0, 0}, {0, 0}}, 0},
    {{0, 0}, {{1, 0}, {0, 0}}, 1},
};
inline constexpr QpFace kQpTri[] = {
    {{0, 0}, {{0, 0}, {0, 0}}, 0},  {{1, 0}, {{0, 0}, {0, 0}}, 0},  {{0, 1}, {{0, 0}, {0, 0}}, 0},
    {{0, 0}, {{1, 0}, {0, 0}}, 1},  {{0, 0}, {{0, 1}, {0, 0}}, 1},  {{1, 0}, {{-1, 1}, {0, 0}}, 1},
    {{0, 0}, {{1, 0}, {0, 1}}, 2},
};

inline Bary qp_bary_at(const QpFace& fc, const double* z, int dim) {
    Bary b;
    b.dim = dim;
    b.c[0] = fc.base[0];
    b.c[1] = fc.base[1];
    for (int p = 0; p < fc.k; ++p) {
        b.c[0] += z[p] * fc.dir[p][0];
        b.c[1] += z[p] * fc.dir[p][1];
    }
    return b;
}
inline bool qp_feasible(const Bary& b) {
    constexpr double tol = 1e-10;
    if (b.dim == 0) return true;
    if (b.dim == 1) return b.c[0] >= -tol && b.c[0] <= 1.0 + tol;
    return b.c[0] >= -tol && b.c[1] >= -tol && b.c[0] + b.c[1] <= 1.0 + tol;
}
inline void qp_clamp(Bary& b) {
    if (b.dim == 0) return;
    if (b.dim == 1) { b.c[0] = clamp01(b.c[0]); return; }
    b.c[0] = std::max(b.c[0], 0.0);
    b.c[1] = std::max(b.c[1], 0.0);
    const double s = b.c[0] + b.c[1];
    if (s > 1.0) { b.c[0] /= s; b.c[1] /= s; }
}

// Eigen Matrix3d::determinant / ::inverse (see the header comment).
inline double det3(const double M[3][3]) {
    auto h = [&](int a, int b, int c) { return M[0][a] * (M[1][b] * M[2][c] - M[1][c] * M[2][b]); };
    return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
}
inline void inverse3(const double M[3][3], double R[3][3]) {
    auto cof = [&](int i, int j) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        return M[i1][j1] * M[i2][j2] - M[i1][j2] * M[i2][j1];
    };
    const double c0[3] = {cof(0, 0), cof(1, 0), cof(2, 0)};
    const double det = c0[0] * M[0][0] + c0[1] * M[1][0] + c0[2] * M[2][0];
    const double inv = 1.0 / det;
    R[1][0] = cof(0, 1) * inv;
    R[1][1] = cof(1, 1) * inv;
    R[2][0] = cof(0, 2) * inv;
    R[1][2] = cof(2, 1) * inv;
    R[2][1] = cof(1, 2) * inv;
    R[2][2] = cof(2, 2) * inv;
    R[0][0] = c0[0] * inv;
    R[0][1] = c0[1] * inv;
    R[0][2] = c0[2] * inv;
}

inline GPair simplex_distance_qp(const Geom& f, const Geom& g) {
    auto faces_of = [](int dim, const QpFace*& ptr, int& n) {
        if (dim == 0) { ptr = kQpPoint; n = 1; }
        else if (dim == 1) { ptr = kQpEdge; n = 3; }
        else { ptr = kQpTri; n = 7; }
    };
    static constexpr double kOrigin[3] = {0, 0, 0};
    const QpFace *ff, *gf;
    int nf, ng;
    faces_of(f.dim, ff, nf);
    faces_of(g.dim, gf, ng);
    const V3 fe1 = f.c[1] - f.c[0], fe2 = f.c[2] - f.c[0];
    const V3 ge1 = g.c[1] - g.c[0], ge2 = g.c[2] - g.c[0];
    GPair best;
    double best_d2 = INFINITY;
    bool have = false;
    for (int i = 0; i < nf; ++i) {
        const QpFace& Ff = ff[i];
        V3 fdir[2];
        for (int p = 0; p < Ff.k; ++p) fdir[p] = Ff.dir[p][0] * fe1 + Ff.dir[p][1] * fe2;
        const V3 f0 = f.at(qp_bary_at(Ff, kOrigin, f.dim));
        for (int j = 0; j < ng; ++j) {
            const QpFace& Fg = gf[j];
            const int k = Ff.k + Fg.k;
            if (k > 3) continue;
            V3 cols[3];
            for (int p = 0; p < Ff.k; ++p) cols[p] = fdir[p];
            for (int p = 0; p < Fg.k; ++p) cols[Ff.k + p] = -(Fg.dir[p][0] * ge1 + Fg.dir[p][1] * ge2);
            const V3 d0 = f0 - g.at(qp_bary_at(Fg, kOrigin, g.dim));
            double z[3] = {0, 0, 0};
            bool solved = true;
            if (k == 1) {
                const double m = sqnorm(cols[0]);
                if (m <= 0.0) solved = false;
                else z[0] = -dot(cols[0], d0) / m;
            } else if (k == 2) {
                const double a11 = sqnorm(cols[0]), a22 = sqnorm(cols[1]);
                const double a12 = dot(cols[0], cols[1]);
                const double det = a11 * a22 - a12 * a12;
                if (det <= 1e-12 * a11 * a22) {
                    solved = false;
                } else {
                    const double r1 = -dot(cols[0], d0), r2 = -dot(cols[1], d0);
                    z[0] = (a22 * r1 - a12 * r2) / det;
                    z[1] = (a11 * r2 - a12 * r1) / det;
                }
            } else if (k == 3) {
                double M[3][3];
                for (int r = 0; r < 3; ++r)
                    for (int c = 0; c < 3; ++c) M[r][c] = dot(cols[r], cols[c]);
                const double det = det3(M);
                const double scale = M[0][0] * M[1][1] * M[2][2];
                if (std::abs(det) <= 1e-12 * scale) {
                    solved = false;
                } else {
                    double rhs[3], R[3][3];
                    for (int r = 0; r < 3; ++r) rhs[r] = -dot(cols[r], d0);
                    inverse3(M, R);
                    for (int r = 0; r < 3; ++r) z[r] = R[r][0] * rhs[0] + R[r][1] * rhs[1] + R[r][2] * rhs[2];
                }
            }
            if (!solved && k > 0) continue;
            Bary fb = qp_bary_at(Ff, z, f.dim);
            Bary gb = qp_bary_at(Fg, z + Ff.k, g.dim);
            if (!qp_feasible(fb) || !qp_feasible(gb)) continue;
            qp_clamp(fb);
            qp_clamp(gb);
            const V3 pf = f.at(fb), pg = g.at(gb);
            const double d2 = sqnorm(pg - pf);
            if (!have || d2 < best_d2) {
                have = true;
                best_d2 = d2;
                best.phi = fb;
                best.lambda = gb;
                best.point_f = pf;
                best.point_g = pg;
            }
        }
    }
    finish_pair(best);
    return best;
}

// exact.hpp:342-367
inline GPair simplex_distance(const Geom& f, const Geom& g) {
    if (g.dim == 0) return point_geom_distance(f, g.c[0]);
    if (f.dim == 0) {
        const GPair r = point_geom_distance(g, f.c[0]);
        GPair out;
        out.lambda = r.phi;
        out.point_f = r.point_g;
        out.point_g = r.point_f;
        finish_pair(out);
        return out;
    }
    if (f.dim == 1 && g.dim == 1) {
        double s, t;
        closest_segment_segment(f.c[0], f.c[1], g.c[0], g.c[1], s, t);
        GPair r;
        r.phi.c[0] = s; r.phi.dim = 1;
        r.lambda.c[0] = t; r.lambda.dim = 1;
        r.point_f = f.at(r.phi);
        r.point_g = g.at(r.lambda);
        finish_pair(r);
        return r;
    }
    return simplex_distance_qp(f, g);
}

// bvh.hpp:113-180 -- count the box face halfspaces containing g entirely:
// 3 -> corner, 2 -> box edge, 1 -> face (two triangles), 0 -> must descend.
struct GBoxProx {
    double distance = 0.0;
    V3 y_b;
    Bary lambda;
    bool must_descend = false;
};
inline GBoxProx box_primitive_proximity(const Aabb& box, const Geom& g) {
    GBoxProx r;
    if (g.dim == 0) {
        const BoxProx p = box_point_proximity(box, g.c[0]);
        r.distance = p.distance;
        r.y_b = p.y_b;
        return r;
    }
    auto lo = [&](int a) { return a == 0 ? box.lo.x : (a == 1 ? box.lo.y : box.lo.z); };
    auto hi = [&](int a) { return a == 0 ? box.hi.x : (a == 1 ? box.hi.y : box.hi.z); };
    auto co = [](V3 v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); };
    auto set = [](V3& v, int a, double x) { (a == 0 ? v.x : (a == 1 ? v.y : v.z)) = x; };
    int out_axis[3];
    int n_out = 0;
    for (int a = 0; a < 3; ++a) {
        out_axis[a] = 0;
        bool all_hi = true, all_lo = true;
        for (int k = 0; k <= g.dim; ++k) {
            all_hi = all_hi && co(g.c[k], a) >= hi(a);
            all_lo = all_lo && co(g.c[k], a) <= lo(a);
        }
        if (all_hi) out_axis[a] = 1, ++n_out;
        else if (all_lo) out_axis[a] = -1, ++n_out;
    }
    if (n_out == 0) {
        r.must_descend = true;
        r.y_b = box.center();
        return r;
    }
    auto side = [&](int a) { return out_axis[a] > 0 ? hi(a) : lo(a); };
    if (n_out == 3) {
        const GPair p = simplex_distance(Geom::point(V3(side(0), side(1), side(2))), g);
        r.distance = p.distance;
        r.y_b = p.point_f;
        r.lambda = p.lambda;
    } else if (n_out == 2) {
        int free_axis = 0;
        while (out_axis[free_axis] != 0) ++free_axis;
        V3 a, b;
        for (int ax = 0; ax < 3; ++ax) {
            const double v = out_axis[ax] != 0 ? side(ax) : 0.0;
            set(a, ax, v);
            set(b, ax, v);
        }
        set(a, free_axis, lo(free_axis));
        set(b, free_axis, hi(free_axis));
        const GPair p = simplex_distance(Geom::edge(a, b), g);
        r.distance = p.distance;
        r.y_b = p.point_f;
        r.lambda = p.lambda;
    } else {
        int fa = 0;
        while (out_axis[fa] == 0) ++fa;
        const int u = (fa + 1) % 3, v = (fa + 2) % 3;
        V3 r00, r10, r11, r01;
        const double s = side(fa);
        set(r00, fa, s); set(r10, fa, s); set(r11, fa, s); set(r01, fa, s);
        set(r00, u, lo(u)); set(r00, v, lo(v));
        set(r10, u, hi(u)); set(r10, v, lo(v));
        set(r11, u, hi(u)); set(r11, v, hi(v));
        set(r01, u, lo(u)); set(r01, v, hi(v));
        const GPair p1 = simplex_distance(Geom::triangle(r00, r10, r11), g);
        const GPair p2 = simplex_distance(Geom::triangle(r00, r11, r01), g);
        const GPair& p = p1.distance <= p2.distance ? p1 : p2;
        r.distance = p.distance;
        r.y_b = p.point_f;
        r.lambda = p.lambda;
    }
    return r;
}

// smooth.hpp:51-61 for a query simplex
inline void push_leaf_term(const Mesh& m, const WeightSet& ws, std::size_t prim, const Geom& g, const Params& prm,
                           Scratch& s) {
    const Geom f = Geom::from_mesh(m, m.simplices[prim]);
    const GPair p = simplex_distance(f, g);
    double w, dw[2];
    evaluate_weight(m, ws, prim, p.phi, prm, w, dw);
    const V3 gw = weight_gradient_world(m, ws, prim, p.phi, prm);
    s.args.push_back(-prm.alpha * p.distance);
    s.coefs.push_back(w);
    s.gcoefs.push_back(w * p.grad - gw / prm.alpha);
}

// smooth.hpp:67-75 for a query simplex: diff = g(lambda) - y_B
inline void push_far_field_term(const BvhNode& node, const GBoxProx& prox, const Geom& g, double w_ff,
                                const Params& prm, Scratch& s) {
    const V3 diff = g.at(prox.lambda) - prox.y_b;
    const double scale = node.count * w_ff;
    s.args.push_back(-prm.alpha * prox.distance);
    s.coefs.push_back(scale);
    s.gcoefs.push_back((scale / prox.distance) * diff);
}

// smooth.hpp:101-131 for a query simplex
inline void collect_contributions(const Mesh& m, const Bvh& bvh, const WeightSet& ws, const Geom& g,
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
            const GBoxProx prox = box_primitive_proximity(node.box, g);
            if (!prox.must_descend && prox.distance > 0.0 && node.diameter < prm.beta * prox.distance) {
                push_far_field_term(node, prox, g, w_ff, prm, s);
                ++st.far_field;
                st.decision_hash += decision_mix(std::uint64_t(id), 1);
                continue;
            }
        }
        if (node.is_leaf()) {
            push_leaf_term(m, ws, std::size_t(node.primitive), g, prm, s);
            ++st.leaves;
            st.decision_hash += decision_mix(std::uint64_t(id), 2);
        } else {
            s.stack.push_back(node.right);
            s.stack.push_back(node.left);
        }
    }
}

// smooth.hpp:166-184 / 189-198 for a query simplex
inline Result smooth_min_dist(const Mesh& m, const Bvh& bvh, const WeightSet& ws, const Geom& g, const Params& prm,
                              Scratch& s) {
    s.clear();
    Result st;
    collect_contributions(m, bvh, ws, g, prm, s, st);
    return result_from_accum(s, st, prm);
}
inline Result smooth_min_dist_flat(const Mesh& m, const WeightSet& ws, const Geom& g, const Params& prm, Scratch& s) {
    s.clear();
    Result st;
    for (std::size_t i = 0; i < m.ns(); ++i) {
        push_leaf_term(m, ws, i, g, prm, s);
        ++st.leaves;
    }
    return result_from_accum(s, st, prm);
}

// smooth.hpp:212-255 for any query mesh (points, edges, triangles)
inline MeshDist smooth_mesh_dist(const Mesh& m, const Bvh* bvh, const WeightSet& ws, const Mesh& query,
                                 const Params& prm, int threads) {
    const std::size_t nq = query.ns();
    MeshDist out;
    out.vertex_grads.assign(query.nv(), V3{});
    out.per_primitive.assign(nq, INFINITY);
    if (nq == 0) return out;
    std::vector<V3> inner(nq);
    std::vector<std::int64_t> leaves(nq, 0), far(nq, 0);
    parallel_for(std::int64_t(nq), threads, [&](std::int64_t b, std::int64_t e, int) {
        Scratch s;
        for (std::int64_t j = b; j < e; ++j) {
            const Geom g = Geom::from_mesh(query, query.simplices[std::size_t(j)]);
            const Result r = bvh ? smooth_min_dist(m, *bvh, ws, g, prm, s) : smooth_min_dist_flat(m, ws, g, prm, s);
            out.per_primitive[std::size_t(j)] = r.d_hat;
            inner[std::size_t(j)] = r.grad;
            leaves[std::size_t(j)] = r.leaves;
            far[std::size_t(j)] = r.far_field;
        }
    });
    double denom = 0.0;
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
        for (V3& gk : out.vertex_grads) gk = V3{};
        return out;
    }
    out.d_hat = -std::log(denom) / prm.alpha_q;
    for (V3& gk : out.vertex_grads) gk = gk / (denom + prm.epsilon);
    return out;
}

}  // namespace sdo

// ------------------------------------------------------ reference caches
// (kept in this header: oracle-side interchange with the product's
// sd_save_* / sd_load_* entry points)
#include <fstream>

namespace sdo {

// bvh.hpp:190-236 (SDBV0001)
inline void save_bvh_cache(const Bvh& bvh, const std::string& path) {
    static const char magic[8] = {'S', 'D', 'B', 'V', '0', '0', '0', '1'};
    std::ofstream out(path, std::ios::binary);
    if (!out) fail("cannot open " + path + " for writing");
    out.write(magic, 8);
    const std::uint64_t n = bvh.nodes.size();
    out.write(reinterpret_cast<const char*>(&n), sizeof(n));
    for (const BvhNode& node : bvh.nodes) {
        const double lo[3] = {node.box.lo.x, node.box.lo.y, node.box.lo.z};
        const double hi[3] = {node.box.hi.x, node.box.hi.y, node.box.hi.z};
        out.write(reinterpret_cast<const char*>(lo), sizeof lo);
        out.write(reinterpret_cast<const char*>(hi), sizeof hi);
        out.write(reinterpret_cast<const char*>(&node.left), sizeof(node.left));
        out.write(reinterpret_cast<const char*>(&node.right), sizeof(node.right));
        out.write(reinterpret_cast<const char*>(&node.primitive), sizeof(node.primitive));
        out.write(reinterpret_cast<const char*>(&node.count), sizeof(node.count));
        out.write(reinterpret_cast<const char*>(&node.diameter), sizeof(node.diameter));
    }
    if (!out) fail("write failed: " + path);
}
inline Bvh load_bvh_cache(const std::string& path) {
    static const char magic[8] = {'S', 'D', 'B', 'V', '0', '0', '0', '1'};
    std::ifstream in(path, std::ios::binary);
    if (!in) fail("cannot open " + path);
    char m[8];
    in.read(m, 8);
    if (!in || std::memcmp(m, magic, 8) != 0) fail(path + ": not a BVH cache (bad magic)");
    std::uint64_t n = 0;
    in.read(reinterpret_cast<char*>(&n), sizeof(n));
    Bvh bvh;
    bvh.nodes.resize(n);
    for (BvhNode& node : bvh.nodes) {
        double lo[3], hi[3];
        in.read(reinterpret_cast<char*>(lo), sizeof lo);
        in.read(reinterpret_cast<char*>(hi), sizeof hi);
        node.box.lo = V3(lo[0], lo[1], lo[2]);
        node.box.hi = V3(hi[0], hi[1], hi[2]);
        in.read(reinterpret_cast<char*>(&node.left), sizeof(node.left));
        in.read(reinterpret_cast<char*>(&node.right), sizeof(node.right));
        in.read(reinterpret_cast<char*>(&node.primitive), sizeof(node.primitive));
        in.read(reinterpret_cast<char*>(&node.count), sizeof(node.count));
        in.read(reinterpret_cast<char*>(&node.diameter), sizeof(node.diameter));
    }
    if (!in) fail(path + ": truncated BVH cache");
    return bvh;
}

// weights.hpp:700-781 (SDWT0001)
inline void save_weight_cache(const WeightSet& ws, const std::string& path) {
    static const char magic[8] = {'S', 'D', 'W', 'T', '0', '0', '0', '1'};
    std::ofstream out(path, std::ios::binary);
    if (!out) fail("cannot open " + path + " for writing");
    auto pod = [&](const auto& v) { out.write(reinterpret_cast<const char*>(&v), sizeof(v)); };
    out.write(magic, 8);
    pod(ws.A);
    pod(ws.sup_wtilde);
    pod(std::uint64_t(ws.edge_polys.size()));
    pod(std::uint64_t(ws.tri_polys.size()));
    pod(std::uint64_t(ws.poly_index.size()));
    for (const EdgePoly& p : ws.edge_polys) {
        pod(p.valence0);
        pod(p.valence1);
        for (double a : p.a) pod(a);
        pod(p.sup);
        pod(p.inf);
    }
    for (const TriPoly& p : ws.tri_polys) {
        pod(p.vertex_valence);
        pod(p.edge_valence);
        for (double a : p.stored) pod(a);
        pod(p.sup);
        pod(p.inf);
        pod(p.residual);
    }
    out.write(reinterpret_cast<const char*>(ws.poly_index.data()),
              std::streamsize(ws.poly_index.size() * sizeof(std::int32_t)));
    if (!out) fail("write failed: " + path);
}
inline WeightSet load_weight_cache(const std::string& path) {
    static const char magic[8] = {'S', 'D', 'W', 'T', '0', '0', '0', '1'};
    std::ifstream in(path, std::ios::binary);
    if (!in) fail("cannot open " + path);
    auto pod = [&](auto& v) { in.read(reinterpret_cast<char*>(&v), sizeof(v)); };
    char m[8];
    in.read(m, 8);
    if (!in || std::memcmp(m, magic, 8) != 0) fail(path + ": not a weight cache (bad magic)");
    WeightSet ws;
    std::uint64_t ne, nt, np;
    pod(ws.A);
    pod(ws.sup_wtilde);
    pod(ne);
    pod(nt);
    pod(np);
    ws.edge_polys.resize(ne);
    for (EdgePoly& p : ws.edge_polys) {
        pod(p.valence0);
        pod(p.valence1);
        for (double& a : p.a) pod(a);
        pod(p.sup);
        pod(p.inf);
    }
    ws.tri_polys.resize(nt);
    for (TriPoly& p : ws.tri_polys) {
        pod(p.vertex_valence);
        pod(p.edge_valence);
        for (double& a : p.stored) pod(a);
        pod(p.sup);
        pod(p.inf);
        pod(p.residual);
        p.expand();
    }
    ws.poly_index.resize(np);
    in.read(reinterpret_cast<char*>(ws.poly_index.data()), std::streamsize(np * sizeof(std::int32_t)));
    if (!in) fail(path + ": truncated weight cache");
    return ws;
}

}  // namespace sdo
