// oracle/capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" surface of the CPU oracle for ctypes (oracle/__init__.py).
// Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU
// baseline legs. Opaque handles own oracle meshes / weight tables / trees;
// every entry returns 0 on success and -1 with sdo_last_error() set.
#include "shapes.hpp"
#include "sdoracle_simplex.hpp"
#include "sdoracle_callers.hpp"

#include <chrono>

using namespace sdo;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
Geom geom_from(const double* c, int dim) {
    if (dim < 0 || dim > 2) fail("query simplex dim must be 0, 1 or 2");
    Geom g;
    g.dim = dim;
    for (int k = 0; k <= dim; ++k) g.c[std::size_t(k)] = V3(c[3 * k], c[3 * k + 1], c[3 * k + 2]);
    return g;
}
Params params_from(const double* p) {
    Params prm;
    prm.alpha = p[0];
    prm.alpha_u = p[1];
    prm.beta = p[2];
    prm.epsilon = p[3];
    return prm;
}
}  // namespace

extern "C" {

const char* sdo_last_error() { return g_err.c_str(); }

// ------------------------------------------------------------------ meshes
void* sdo_mesh_create(const double* xyz, std::int64_t V, const std::int32_t* sv, const std::uint8_t* kind,
                      std::int64_t N) {
    auto* m = new Mesh;
    m->vertices.resize(std::size_t(V));
    std::memcpy(m->vertices.data(), xyz, sizeof(double) * 3 * std::size_t(V));
    m->simplices.resize(std::size_t(N));
    for (std::int64_t i = 0; i < N; ++i) {
        Simplex& s = m->simplices[std::size_t(i)];
        s.kind = kind[i];
        for (int k = 0; k < 3; ++k) s.v[k] = sv[3 * i + k];
    }
    return m;
}
void sdo_mesh_free(void* h) { delete static_cast<Mesh*>(h); }
std::int64_t sdo_mesh_nv(void* h) { return std::int64_t(static_cast<Mesh*>(h)->nv()); }
std::int64_t sdo_mesh_ns(void* h) { return std::int64_t(static_cast<Mesh*>(h)->ns()); }
void sdo_mesh_export(void* h, double* xyz, std::int32_t* sv, std::uint8_t* kind) {
    const Mesh& m = *static_cast<Mesh*>(h);
    std::memcpy(xyz, m.vertices.data(), sizeof(double) * 3 * m.nv());
    for (std::size_t i = 0; i < m.ns(); ++i) {
        const Simplex& s = m.simplices[i];
        kind[i] = s.kind;
        for (int k = 0; k < 3; ++k) sv[3 * i + k] = k < s.nverts() ? s.v[k] : -1;
    }
}
int sdo_mesh_validate(void* h) { return guard([&] { validate(*static_cast<Mesh*>(h)); }); }
double sdo_mesh_mean_edge(void* h) { return mean_unique_edge_length(*static_cast<Mesh*>(h)); }

// shapes (shapes.hpp) and configs
void* sdo_gen_config_mesh(int cfg) {
    void* out = nullptr;
    guard([&] { out = new Mesh(config_mesh(cfg)); });
    return out;
}
int sdo_gen_config_queries(int cfg, void* mesh, std::int64_t nq, double* out) {
    return guard([&] {
        const auto q = config_queries(cfg, *static_cast<Mesh*>(mesh), nq);
        std::memcpy(out, q.data(), sizeof(double) * 3 * q.size());
    });
}
void* sdo_gen_random_scene(std::uint64_t seed, int max_prims) { return new Mesh(random_scene(seed, max_prims)); }
void* sdo_gen_point_cluster(int n, std::uint64_t seed, double spread) {
    Rng rng(seed);
    return new Mesh(point_cluster(n, rng, spread));
}
void* sdo_gen_icosphere(int sub) { return new Mesh(icosphere(sub)); }
void* sdo_gen_uv_torus(double major, double minor, int nu, int nv) { return new Mesh(uv_torus(major, minor, nu, nv)); }
void* sdo_gen_triangle_fan(int k, std::uint64_t seed) {
    Rng rng(seed);
    return new Mesh(triangle_fan(k, rng));
}
void* sdo_gen_polyline(int n, std::uint64_t seed) {
    Rng rng(seed);
    return new Mesh(polyline(n, rng));
}
// n random query simplices from one mt19937_64(seed) stream over the
// mesh's bounding box (shapes.hpp:243-265); corners n x 9, dims n.
void sdo_gen_random_queries(std::uint64_t seed, void* mesh, int n, double* corners, std::int32_t* dims) {
    Rng rng(seed);
    const Aabb box = bounding_box(*static_cast<Mesh*>(mesh));
    for (int i = 0; i < n; ++i) {
        const QuerySimplex q = random_query(rng, box);
        for (int k = 0; k < 3; ++k) {
            corners[9 * i + 3 * k + 0] = q.c[k].x;
            corners[9 * i + 3 * k + 1] = q.c[k].y;
            corners[9 * i + 3 * k + 2] = q.c[k].z;
        }
        dims[i] = q.dim;
    }
}

void sdo_gen_random_queries_scaled(std::uint64_t seed, void* mesh, int n, double scale, double* corners,
                                   std::int32_t* dims) {
    Rng rng(seed);
    const Aabb box = bounding_box(*static_cast<Mesh*>(mesh));
    for (int i = 0; i < n; ++i) {
        const QuerySimplex q = random_query(rng, box, scale);
        for (int k = 0; k < 3; ++k) {
            corners[9 * i + 3 * k + 0] = q.c[k].x;
            corners[9 * i + 3 * k + 1] = q.c[k].y;
            corners[9 * i + 3 * k + 2] = q.c[k].z;
        }
        dims[i] = q.dim;
    }
}

// A persistent mt19937_64 so several random_query draws can share one
// stream across scenes, as the reference tests do (e.g. test_smooth.cpp:143-175).
void* sdo_rng_new(std::uint64_t seed) { return new Rng(seed); }
void sdo_rng_free(void* r) { delete static_cast<Rng*>(r); }
void sdo_rng_random_queries(void* rng, void* mesh, int n, double* corners, std::int32_t* dims) {
    Rng& g = *static_cast<Rng*>(rng);
    const Aabb box = bounding_box(*static_cast<Mesh*>(mesh));
    for (int i = 0; i < n; ++i) {
        const QuerySimplex q = random_query(g, box);
        for (int k = 0; k < 3; ++k) {
            corners[9 * i + 3 * k + 0] = q.c[k].x;
            corners[9 * i + 3 * k + 1] = q.c[k].y;
            corners[9 * i + 3 * k + 2] = q.c[k].z;
        }
        dims[i] = q.dim;
    }
}

// ----------------------------------------------------------------- weights
void* sdo_weights_build(void* mesh) {
    void* out = nullptr;
    guard([&] {
        const Mesh& m = *static_cast<Mesh*>(mesh);
        out = new WeightSet(build_weight_set(m, build_adjacency(m)));
    });
    return out;
}
void* sdo_weights_unit(void* mesh) { return new WeightSet(unit_weight_set(*static_cast<Mesh*>(mesh))); }
void sdo_weights_free(void* h) { delete static_cast<WeightSet*>(h); }
void sdo_weights_info(void* h, double* A, double* sup, std::int32_t* ne, std::int32_t* nt, std::int64_t* npi) {
    const WeightSet& w = *static_cast<WeightSet*>(h);
    *A = w.A;
    *sup = w.sup_wtilde;
    *ne = std::int32_t(w.edge_polys.size());
    *nt = std::int32_t(w.tri_polys.size());
    *npi = std::int64_t(w.poly_index.size());
}
// edge: a[5], (v0, v1), (sup, inf); tri: stored[13], (v, e), (sup, inf, residual)
void sdo_weights_export(void* h, double* edge_a, std::int32_t* edge_val, double* edge_si, double* tri_stored,
                        std::int32_t* tri_val, double* tri_sir, std::int32_t* poly_index) {
    const WeightSet& w = *static_cast<WeightSet*>(h);
    for (std::size_t i = 0; i < w.edge_polys.size(); ++i) {
        const EdgePoly& p = w.edge_polys[i];
        for (int k = 0; k < 5; ++k) edge_a[5 * i + k] = p.a[k];
        edge_val[2 * i] = p.valence0;
        edge_val[2 * i + 1] = p.valence1;
        edge_si[2 * i] = p.sup;
        edge_si[2 * i + 1] = p.inf;
    }
    for (std::size_t i = 0; i < w.tri_polys.size(); ++i) {
        const TriPoly& p = w.tri_polys[i];
        for (int k = 0; k < 13; ++k) tri_stored[13 * i + k] = p.stored[k];
        tri_val[2 * i] = p.vertex_valence;
        tri_val[2 * i + 1] = p.edge_valence;
        tri_sir[3 * i] = p.sup;
        tri_sir[3 * i + 1] = p.inf;
        tri_sir[3 * i + 2] = p.residual;
    }
    std::memcpy(poly_index, w.poly_index.data(), sizeof(std::int32_t) * w.poly_index.size());
}
void* sdo_weights_from_arrays(double A, double sup, std::int32_t ne, const double* edge_a, std::int32_t nt,
                              const double* tri_stored, std::int64_t npi, const std::int32_t* poly_index) {
    auto* w = new WeightSet;
    w->A = A;
    w->sup_wtilde = sup;
    for (std::int32_t i = 0; i < ne; ++i) {
        EdgePoly p;
        for (int k = 0; k < 5; ++k) p.a[k] = edge_a[5 * i + k];
        w->edge_polys.push_back(p);
    }
    for (std::int32_t i = 0; i < nt; ++i) {
        TriPoly p;
        for (int k = 0; k < 13; ++k) p.stored[k] = tri_stored[13 * i + k];
        p.expand();
        w->tri_polys.push_back(p);
    }
    w->poly_index.assign(poly_index, poly_index + npi);
    return w;
}
double sdo_weights_max_attenuated(void* h, const double* params) {
    return static_cast<WeightSet*>(h)->max_attenuated_weight(params_from(params));
}
// w, dw[2] and the world gradient gw[3] of primitive i at barycentric phi
void sdo_weights_eval(void* mesh, void* ws, std::int64_t i, const double* phi, int dim, const double* params,
                      double* w, double* dw, double* gw) {
    const Mesh& m = *static_cast<Mesh*>(mesh);
    const WeightSet& s = *static_cast<WeightSet*>(ws);
    Bary b;
    b.c[0] = phi[0];
    b.c[1] = phi[1];
    b.dim = dim;
    const Params prm = params_from(params);
    evaluate_weight(m, s, std::size_t(i), b, prm, *w, dw);
    const V3 g = weight_gradient_world(m, s, std::size_t(i), b, prm);
    gw[0] = g.x; gw[1] = g.y; gw[2] = g.z;
}
void sdo_edge_weight(std::int32_t v0, std::int32_t v1, double* a5, double* supinf) {
    const EdgePoly p = build_edge_weight(v0, v1);
    for (int k = 0; k < 5; ++k) a5[k] = p.a[k];
    supinf[0] = p.sup;
    supinf[1] = p.inf;
}
void sdo_tri_weight(std::int32_t v, std::int32_t e, double* stored13, double* sir3) {
    const TriPoly p = cached_tri_weight(v, e);
    for (int k = 0; k < 13; ++k) stored13[k] = p.stored[k];
    sir3[0] = p.sup;
    sir3[1] = p.inf;
    sir3[2] = p.residual;
}
// value / d/dx / d/dy of the polynomial with the given stored coefficients
// at n points (x, y), via the padded Horner of weights.hpp:103-111
void sdo_tri_poly_eval(const double* stored13, int n, const double* xy, double* val, double* dx, double* dy) {
    TriPoly p;
    for (int k = 0; k < 13; ++k) p.stored[k] = stored13[k];
    p.expand();
    for (int i = 0; i < n; ++i) {
        val[i] = p.value(xy[2 * i], xy[2 * i + 1]);
        dx[i] = p.deriv_x(xy[2 * i], xy[2 * i + 1]);
        dy[i] = p.deriv_y(xy[2 * i], xy[2 * i + 1]);
    }
}
void sdo_tri_poly_grid(const double* stored13, double* c64) {
    TriPoly p;
    for (int k = 0; k < 13; ++k) p.stored[k] = stored13[k];
    p.expand();
    for (int j = 0; j < 8; ++j)
        for (int k = 0; k < 8; ++k) c64[8 * j + k] = p.c[j][k];
}

// --------------------------------------------------------------------- bvh
void* sdo_bvh_build(void* mesh) { return new Bvh(build_bvh(*static_cast<Mesh*>(mesh))); }
void* sdo_bvh_from_nodes(const void* nodes, std::int64_t n) {
    auto* b = new Bvh;
    b->nodes.resize(std::size_t(n));
    std::memcpy(b->nodes.data(), nodes, sizeof(BvhNode) * std::size_t(n));
    return b;
}
void sdo_bvh_free(void* h) { delete static_cast<Bvh*>(h); }
std::int64_t sdo_bvh_size(void* h) { return std::int64_t(static_cast<Bvh*>(h)->nodes.size()); }
void sdo_bvh_export(void* h, void* nodes) {
    const Bvh& b = *static_cast<Bvh*>(h);
    std::memcpy(nodes, b.nodes.data(), sizeof(BvhNode) * b.nodes.size());
}
// box proximity of n points to one box: distance, y_b[3]
void sdo_box_point_proximity(const double* lo, const double* hi, int n, const double* q, double* dist, double* yb) {
    Aabb box;
    box.lo = V3(lo[0], lo[1], lo[2]);
    box.hi = V3(hi[0], hi[1], hi[2]);
    for (int i = 0; i < n; ++i) {
        const BoxProx p = box_point_proximity(box, V3(q[3 * i], q[3 * i + 1], q[3 * i + 2]));
        dist[i] = p.distance;
        yb[3 * i] = p.y_b.x; yb[3 * i + 1] = p.y_b.y; yb[3 * i + 2] = p.y_b.z;
    }
}
int sdo_bh_condition(double diameter, double distance, int must_descend, double beta) {
    BvhNode node;
    node.diameter = diameter;
    BoxProx p;
    p.distance = distance;
    p.must_descend = must_descend != 0;
    return bh_condition(node, p, beta) ? 1 : 0;
}

// ------------------------------------------------------------------- exact
// pair distance of point q to a simplex given by corners[9] and dim;
// out: distance, phi[2], point_f[3], grad[3]
void sdo_point_simplex(const double* corners, int dim, const double* q, double* out) {
    std::array<V3, 3> f;
    for (int k = 0; k < 3; ++k) f[k] = V3(corners[3 * k], corners[3 * k + 1], corners[3 * k + 2]);
    const Pair p = point_simplex_distance(f, dim, V3(q[0], q[1], q[2]));
    out[0] = p.distance;
    out[1] = p.phi.c[0];
    out[2] = p.phi.c[1];
    out[3] = p.point_f.x; out[4] = p.point_f.y; out[5] = p.point_f.z;
    out[6] = p.grad.x; out[7] = p.grad.y; out[8] = p.grad.z;
}
void sdo_exact_min(void* mesh, std::int64_t Q, const double* q, double* dist, std::int64_t* argmin, int threads) {
    const Mesh& m = *static_cast<Mesh*>(mesh);
    parallel_for(Q, threads, [&](std::int64_t b, std::int64_t e, int) {
        for (std::int64_t i = b; i < e; ++i) {
            const ExactMin r = exact_min_distance(m, V3(q[3 * i], q[3 * i + 1], q[3 * i + 2]));
            dist[i] = r.distance;
            argmin[i] = std::int64_t(r.argmin);
        }
    });
}

// ------------------------------------------------------------------ smooth
// Batched point queries through the restated evaluator. bvh == NULL runs
// smooth_min_dist_flat (smooth.hpp:189-198); otherwise smooth_min_dist
// (smooth.hpp:166-184) on the given tree. params = {alpha, alpha_u, beta,
// epsilon}. Optional outputs may be NULL. Returns wall seconds in *secs.
int sdo_query(void* mesh, void* ws, void* bvh, const double* q, std::int64_t Q, const double* params, int threads,
              double* d_hat, double* grad, double* c, double* grad_c, std::int64_t* leaves, std::int64_t* far,
              std::uint64_t* hash, double* secs) {
    return guard([&] {
        const Mesh& m = *static_cast<Mesh*>(mesh);
        const WeightSet& w = *static_cast<WeightSet*>(ws);
        const Bvh* b = static_cast<Bvh*>(bvh);
        const Params prm = params_from(params);
        if (w.poly_index.size() != m.ns()) fail("weight table does not match the mesh");
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(Q, threads, [&](std::int64_t lo, std::int64_t hi, int) {
            Scratch s;
            for (std::int64_t i = lo; i < hi; ++i) {
                const V3 qi(q[3 * i], q[3 * i + 1], q[3 * i + 2]);
                const Result r = b ? smooth_min_dist(m, *b, w, qi, prm, s) : smooth_min_dist_flat(m, w, qi, prm, s);
                d_hat[i] = r.d_hat;
                if (grad) { grad[3 * i] = r.grad.x; grad[3 * i + 1] = r.grad.y; grad[3 * i + 2] = r.grad.z; }
                if (c) c[i] = r.c;
                if (grad_c) { grad_c[3 * i] = r.grad_c.x; grad_c[3 * i + 1] = r.grad_c.y; grad_c[3 * i + 2] = r.grad_c.z; }
                if (leaves) leaves[i] = r.leaves;
                if (far) far[i] = r.far_field;
                if (hash) hash[i] = r.decision_hash;
            }
        });
        if (secs) secs[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// Query simplices (points, edges, triangles): corners n x 9, dims n
// (smooth.hpp:166-198 with a SimplexGeom g).
int sdo_query_simplices(void* mesh, void* ws, void* bvh, const double* corners, const std::int32_t* dims,
                        std::int64_t Q, const double* params, int threads, double* d_hat, double* grad, double* c,
                        double* grad_c, std::int64_t* leaves, std::int64_t* far, std::uint64_t* hash, double* secs) {
    return guard([&] {
        const Mesh& m = *static_cast<Mesh*>(mesh);
        const WeightSet& w = *static_cast<WeightSet*>(ws);
        const Bvh* b = static_cast<Bvh*>(bvh);
        const Params prm = params_from(params);
        if (w.poly_index.size() != m.ns()) fail("weight table does not match the mesh");
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(Q, threads, [&](std::int64_t lo, std::int64_t hi, int) {
            Scratch s;
            for (std::int64_t i = lo; i < hi; ++i) {
                const Geom g = geom_from(corners + 9 * i, dims[i]);
                const Result r = b ? smooth_min_dist(m, *b, w, g, prm, s) : smooth_min_dist_flat(m, w, g, prm, s);
                d_hat[i] = r.d_hat;
                if (grad) { grad[3 * i] = r.grad.x; grad[3 * i + 1] = r.grad.y; grad[3 * i + 2] = r.grad.z; }
                if (c) c[i] = r.c;
                if (grad_c) { grad_c[3 * i] = r.grad_c.x; grad_c[3 * i + 1] = r.grad_c.y; grad_c[3 * i + 2] = r.grad_c.z; }
                if (leaves) leaves[i] = r.leaves;
                if (far) far[i] = r.far_field;
                if (hash) hash[i] = r.decision_hash;
            }
        });
        if (secs) secs[0] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// exact.hpp:342-367 / 158-313: out = distance, phi[2], lambda[2],
// point_f[3], point_g[3], grad[3]
static void put_pair(const GPair& r, double* out) {
    const double v[14] = {r.distance, r.phi.c[0], r.phi.c[1], r.lambda.c[0], r.lambda.c[1],
                          r.point_f.x, r.point_f.y, r.point_f.z, r.point_g.x, r.point_g.y, r.point_g.z,
                          r.grad.x, r.grad.y, r.grad.z};
    std::memcpy(out, v, sizeof(v));
}
int sdo_simplex_distance(const double* f, int fdim, const double* g, int gdim, int qp, double* out) {
    return guard([&] {
        const Geom F = geom_from(f, fdim), G = geom_from(g, gdim);
        put_pair(qp ? simplex_distance_qp(F, G) : simplex_distance(F, G), out);
    });
}
// bvh.hpp:113-180: out = distance, y_b[3], lambda[2], must_descend
int sdo_box_primitive_proximity(const double* lo, const double* hi, const double* g, int gdim, double* out) {
    return guard([&] {
        Aabb box;
        box.lo = V3(lo[0], lo[1], lo[2]);
        box.hi = V3(hi[0], hi[1], hi[2]);
        const GBoxProx p = box_primitive_proximity(box, geom_from(g, gdim));
        const double v[7] = {p.distance, p.y_b.x, p.y_b.y, p.y_b.z, p.lambda.c[0], p.lambda.c[1],
                             p.must_descend ? 1.0 : 0.0};
        std::memcpy(out, v, sizeof(v));
    });
}

// Mesh-to-mesh distance for any query mesh (smooth.hpp:212-255).
// params = {alpha, alpha_u, beta, epsilon, alpha_q}; bvh NULL = flat inner sums.
int sdo_mesh_dist(void* mesh, void* ws, void* bvh, void* query, const double* params, int threads, double* d_hat,
                  double* vertex_grads, double* per_primitive, std::int64_t* counters) {
    return guard([&] {
        Params prm = params_from(params);
        prm.alpha_q = params[4];
        const Mesh& q = *static_cast<Mesh*>(query);
        const MeshDist r = smooth_mesh_dist(*static_cast<Mesh*>(mesh), static_cast<Bvh*>(bvh),
                                            *static_cast<WeightSet*>(ws), q, prm, threads);
        *d_hat = r.d_hat;
        for (std::size_t k = 0; k < q.nv(); ++k) {
            vertex_grads[3 * k] = r.vertex_grads[k].x;
            vertex_grads[3 * k + 1] = r.vertex_grads[k].y;
            vertex_grads[3 * k + 2] = r.vertex_grads[k].z;
        }
        for (std::size_t j = 0; j < q.ns(); ++j) per_primitive[j] = r.per_primitive[j];
        counters[0] = r.leaves;
        counters[1] = r.far_field;
    });
}

// reference caches (bvh.hpp:190-236, weights.hpp:700-781)
int sdo_save_bvh_cache(void* bvh, const char* path) {
    return guard([&] { save_bvh_cache(*static_cast<Bvh*>(bvh), path); });
}
void* sdo_load_bvh_cache(const char* path) {
    try {
        return new Bvh(load_bvh_cache(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
int sdo_save_weight_cache(void* ws, const char* path) {
    return guard([&] { save_weight_cache(*static_cast<WeightSet*>(ws), path); });
}
void* sdo_load_weight_cache(const char* path) {
    try {
        return new WeightSet(load_weight_cache(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// render (render.hpp:77-134): cfg = origin[3] target[3] up[3] fov width height
// threshold max_steps (12 doubles); stats = leaves, far_field, rays, hits
int sdo_render(void* mesh, void* ws, void* bvh, const double* params, const double* cfg, int threads,
               std::uint8_t* rgb, double* hit_t, std::int64_t* stats, double* seconds) {
    return guard([&] {
        RenderConfig rc;
        rc.origin = V3(cfg[0], cfg[1], cfg[2]);
        rc.target = V3(cfg[3], cfg[4], cfg[5]);
        rc.up = V3(cfg[6], cfg[7], cfg[8]);
        rc.fov_deg = cfg[9];
        rc.width = int(cfg[10]);
        rc.height = int(cfg[11]);
        rc.threshold = cfg[12];
        rc.max_steps = int(cfg[13]);
        const RenderOut r = render(*static_cast<Mesh*>(mesh), *static_cast<Bvh*>(bvh), *static_cast<WeightSet*>(ws),
                                   params_from(params), rc, threads);
        std::memcpy(rgb, r.rgb.data(), r.rgb.size());
        std::memcpy(hit_t, r.hit_t.data(), r.hit_t.size() * sizeof(double));
        stats[0] = r.leaves;
        stats[1] = r.far_field;
        stats[2] = r.rays;
        stats[3] = r.hits;
        *seconds = r.seconds;
    });
}
int sdo_write_ppm(const std::uint8_t* rgb, int w, int h, const char* path) {
    return guard([&] { write_ppm(std::vector<std::uint8_t>(rgb, rgb + 3 * std::size_t(w) * h), w, h, path); });
}
// grid_benchmark (bench.hpp:29-70) and write_grid_csv (:75-88)
int sdo_grid_benchmark(void* mesh, void* ws, void* bvh, const double* params, int n, int threads, double* d,
                       std::int64_t* leaves, std::int64_t* far) {
    return guard([&] {
        const GridOut r = grid_benchmark(*static_cast<Mesh*>(mesh), *static_cast<Bvh*>(bvh),
                                         *static_cast<WeightSet*>(ws), params_from(params), n, threads);
        std::memcpy(d, r.d_hat.data(), r.d_hat.size() * sizeof(double));
        std::memcpy(leaves, r.leaves.data(), r.leaves.size() * sizeof(std::int64_t));
        std::memcpy(far, r.far_field.data(), r.far_field.size() * sizeof(std::int64_t));
    });
}
int sdo_write_grid_csv(const double* d, const std::int64_t* leaves, const std::int64_t* far, int n,
                       const double* slab_seconds, const char* path) {
    return guard([&] {
        const std::size_t n3 = std::size_t(n) * n * n;
        GridOut r;
        r.d_hat.assign(d, d + n3);
        r.leaves.assign(leaves, leaves + n3);
        r.far_field.assign(far, far + n3);
        write_grid_csv(r, n, std::vector<double>(slab_seconds, slab_seconds + n), path);
    });
}

std::uint64_t sdo_decision_mix(std::uint64_t node, std::uint64_t kind) { return decision_mix(node, kind); }
int sdo_hardware_threads() {
    const unsigned n = std::thread::hardware_concurrency();
    return n ? int(n) : 1;
}

}  // extern "C"
