// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (oracle/_ref).
//
// extern "C" surface over the REFERENCE's own headers, compiled unmodified
// from /root/reference/proj/include (never copied into this repo) with the
// Eigen-subset shim of oracle/eigen_shim (Eigen is absent from the image).
// Built by `make -C oracle ref` into oracle/_ref/libsdref.so when the
// reference is present; the .so travels to the GPU box with the snapshot.
// Loaded only by tests/ and bench.py's reference / cpu-baseline legs.
//
// A scene handle owns a smoothdist::SimplexMesh, a WeightSet (fed in as a
// table: the triangle-polynomial SVD construction is not reproduced by the
// shim) and optionally a Bvh (fed in, or built by the reference's
// build_bvh). Queries run the reference's own entry points
// (smooth_min_dist / smooth_min_dist_flat, smooth.hpp:166-198) batched by
// its own parallel_for (parallel.hpp:25-44) with one EvalScratch per worker.
#include <smoothdist/smooth.hpp>

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

using namespace smoothdist;

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

struct Node72 {  // sd_bvh_node / the reference BvhNode field set (bvh.hpp:14-22)
    double lo[3], hi[3];
    std::int32_t left, right, primitive, count;
    double diameter;
};
static_assert(sizeof(Node72) == 72, "node layout");

struct Scene {
    SimplexMesh mesh;
    WeightSet ws;
    Bvh bvh;
};

SmoothParams params_from(const double* p) {
    SmoothParams prm;
    prm.alpha = p[0];
    prm.alpha_u = p[1];
    prm.beta = p[2];
    prm.epsilon = p[3];
    prm.alpha_q = p[4];
    return prm;
}

SimplexMesh mesh_from(const double* xyz, std::int64_t V, const std::int32_t* sv, const std::uint8_t* kind,
                      std::int64_t N) {
    SimplexMesh m;
    m.vertices.resize(std::size_t(V));
    for (std::int64_t i = 0; i < V; ++i) m.vertices[std::size_t(i)] = Vec3(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    m.simplices.resize(std::size_t(N));
    for (std::int64_t i = 0; i < N; ++i) {
        Simplex& s = m.simplices[std::size_t(i)];
        s.kind = static_cast<SimplexKind>(kind[i]);
        for (int k = 0; k < 3; ++k) s.v[std::size_t(k)] = k <= int(kind[i]) ? sv[3 * i + k] : -1;
    }
    return m;
}
}  // namespace

extern "C" {

const char* sdr_last_error() { return g_err.c_str(); }

// Scene: mesh + WeightSet table (A, sup_wtilde, ne x 5 edge coefficients,
// nt x 13 stored triangle coefficients, poly_index) + optional tree.
void* sdr_scene_create(const double* xyz, std::int64_t V, const std::int32_t* sv, const std::uint8_t* kind,
                       std::int64_t N, double A, double sup_wtilde, std::int32_t ne, const double* edge_a,
                       std::int32_t nt, const double* tri_stored, const std::int32_t* poly_index) {
    Scene* out = nullptr;
    guard([&] {
        auto sc = std::make_unique<Scene>();
        sc->mesh = mesh_from(xyz, V, sv, kind, N);
        validate(sc->mesh);
        sc->ws.A = A;
        sc->ws.sup_wtilde = sup_wtilde;
        sc->ws.edge_polys.resize(std::size_t(ne));
        for (int k = 0; k < ne; ++k)
            for (int j = 0; j < 5; ++j) sc->ws.edge_polys[std::size_t(k)].a[std::size_t(j)] = edge_a[5 * k + j];
        sc->ws.tri_polys.resize(std::size_t(nt));
        for (int k = 0; k < nt; ++k) {
            TriWeightPoly& p = sc->ws.tri_polys[std::size_t(k)];
            for (int j = 0; j < 13; ++j) p.stored[std::size_t(j)] = tri_stored[13 * k + j];
            p.expand();
        }
        sc->ws.poly_index.assign(poly_index, poly_index + N);
        out = sc.release();
    });
    return out;
}

void sdr_scene_free(void* h) { delete static_cast<Scene*>(h); }

// Install a tree in the reference layout, or (nodes == NULL) build it with
// the reference's build_bvh (bvh.hpp:34-91).
int sdr_scene_set_bvh(void* h, const void* nodes, std::int64_t n) {
    return guard([&] {
        Scene& sc = *static_cast<Scene*>(h);
        if (!nodes) {
            sc.bvh = build_bvh(sc.mesh);
            return;
        }
        const Node72* in = static_cast<const Node72*>(nodes);
        sc.bvh.nodes.resize(std::size_t(n));
        for (std::int64_t i = 0; i < n; ++i) {
            BvhNode& o = sc.bvh.nodes[std::size_t(i)];
            o.box.lo = Vec3(in[i].lo[0], in[i].lo[1], in[i].lo[2]);
            o.box.hi = Vec3(in[i].hi[0], in[i].hi[1], in[i].hi[2]);
            o.left = in[i].left;
            o.right = in[i].right;
            o.primitive = in[i].primitive;
            o.count = in[i].count;
            o.diameter = in[i].diameter;
        }
    });
}

std::int64_t sdr_scene_bvh_size(void* h) { return std::int64_t(static_cast<Scene*>(h)->bvh.nodes.size()); }

int sdr_scene_export_bvh(void* h, void* out) {
    return guard([&] {
        const Scene& sc = *static_cast<Scene*>(h);
        Node72* o = static_cast<Node72*>(out);
        for (std::size_t i = 0; i < sc.bvh.nodes.size(); ++i) {
            const BvhNode& b = sc.bvh.nodes[i];
            for (int a = 0; a < 3; ++a) {
                o[i].lo[a] = b.box.lo(a);
                o[i].hi[a] = b.box.hi(a);
            }
            o[i].left = b.left;
            o[i].right = b.right;
            o[i].primitive = b.primitive;
            o[i].count = b.count;
            o[i].diameter = b.diameter;
        }
    });
}

// Batched point (dims == NULL) or simplex queries (corners Q x 9, dims Q):
// mode 0 = smooth_min_dist_flat, 1 = smooth_min_dist on the scene's tree.
// Outputs (any may be NULL except d_hat): SmoothResult fields
// (smooth.hpp:20-27). *seconds = wall time of the batched evaluation.
int sdr_query(void* h, const double* q, const std::int32_t* dims, std::int64_t Q, const double* prm, int mode,
              int threads, double* d_hat, double* grad, double* c, double* grad_c, std::int64_t* leaves,
              std::int64_t* far_field, double* seconds) {
    return guard([&] {
        const Scene& sc = *static_cast<Scene*>(h);
        const SmoothParams params = params_from(prm);
        if (mode == 1 && sc.bvh.empty() && sc.mesh.num_simplices() > 0) fail("no tree");
        const int nt = std::max(1, threads);
        std::vector<EvalScratch> scratch(static_cast<std::size_t>(nt));
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(Q, nt, [&](std::int64_t b, std::int64_t e, int w) {
            for (std::int64_t i = b; i < e; ++i) {
                SimplexGeom g;
                if (dims) {
                    const double* cc = q + 9 * i;
                    const Vec3 c0(cc[0], cc[1], cc[2]), c1(cc[3], cc[4], cc[5]), c2(cc[6], cc[7], cc[8]);
                    g = dims[i] == 0 ? SimplexGeom::point(c0)
                                     : (dims[i] == 1 ? SimplexGeom::edge(c0, c1) : SimplexGeom::triangle(c0, c1, c2));
                } else {
                    g = SimplexGeom::point(Vec3(q[3 * i], q[3 * i + 1], q[3 * i + 2]));
                }
                const SmoothResult r = mode == 1 ? smooth_min_dist(sc.mesh, sc.bvh, sc.ws, g, params,
                                                                   scratch[std::size_t(w)])
                                                 : smooth_min_dist_flat(sc.mesh, sc.ws, g, params);
                d_hat[i] = r.d_hat;
                if (grad)
                    for (int a = 0; a < 3; ++a) grad[3 * i + a] = r.grad(a);
                if (c) c[i] = r.c;
                if (grad_c)
                    for (int a = 0; a < 3; ++a) grad_c[3 * i + a] = r.grad_c(a);
                if (leaves) leaves[i] = r.leaves;
                if (far_field) far_field[i] = r.far_field;
            }
        });
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// The reference's adjacency (mesh.hpp:163-183) and, for meshes without
// triangles, its whole build_weight_set (weights.hpp:589-621; edge
// polynomials are closed form, weights.hpp:46-76). valence: V vertex
// valences. poly_index: N. edge_a: capacity ne_cap x 5.
int sdr_build_weights_no_tris(const double* xyz, std::int64_t V, const std::int32_t* sv, const std::uint8_t* kind,
                              std::int64_t N, std::int32_t* valence, double* A, double* sup_wtilde, std::int32_t* ne,
                              double* edge_a, std::int32_t ne_cap, std::int32_t* poly_index) {
    return guard([&] {
        const SimplexMesh m = mesh_from(xyz, V, sv, kind, N);
        const Adjacency adj = build_adjacency(m);
        for (std::int64_t v = 0; v < V; ++v) valence[v] = adj.vertex_valence[std::size_t(v)];
        for (const Simplex& s : m.simplices)
            if (s.kind == SimplexKind::Triangle) fail("triangles need the SVD construction (not in the shim)");
        const WeightSet ws = build_weight_set(m, adj);
        *A = ws.A;
        *sup_wtilde = ws.sup_wtilde;
        *ne = std::int32_t(ws.edge_polys.size());
        if (*ne > ne_cap) fail("edge table capacity");
        for (std::size_t k = 0; k < ws.edge_polys.size(); ++k)
            for (int j = 0; j < 5; ++j) edge_a[5 * k + std::size_t(j)] = ws.edge_polys[k].a[std::size_t(j)];
        std::memcpy(poly_index, ws.poly_index.data(), sizeof(std::int32_t) * std::size_t(N));
    });
}

}  // extern "C"
