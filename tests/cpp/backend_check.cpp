// tests/cpp/backend_check.cpp -- TEST INFRASTRUCTURE: the reference-typed
// drop-in (include/smoothdist_gpu_backend.hpp) compiled against the
// reference's own headers (/root/reference/proj/include, with the Eigen
// shim of oracle/eigen_shim) and checked against the reference's own CPU
// evaluator in the same process. Built by `make -C oracle ref` into
// oracle/_ref/backend_check; run by tests/test_gpu_backend_header.py.
//
//   backend_check mesh.obj weights.sdwt queries.bin precision alpha beta
//
// The mesh comes through the reference's load_mesh (mesh_io.hpp:260), the
// WeightSet through its load_weight_cache (weights.hpp:744-781), the tree
// from its build_bvh (bvh.hpp:34-91). Exit 0 iff every comparison holds.
#include "smoothdist_gpu_backend.hpp"

#include <smoothdist/mesh_io.hpp>

#include <cstdio>
#include <fstream>

using namespace smoothdist;

static int g_fail = 0;
static void check(bool ok, const char* what, double v) {
    std::printf("%-44s %s (%.3g)\n", what, ok ? "ok" : "FAIL", v);
    if (!ok) ++g_fail;
}

int main(int argc, char** argv) {
    if (argc != 7) {
        std::fprintf(stderr, "usage: %s mesh.obj weights.sdwt queries.bin precision alpha beta\n", argv[0]);
        return 2;
    }
    const SimplexMesh mesh = load_mesh(argv[1]);
    validate(mesh);
    const WeightSet ws = load_weight_cache(argv[2]);
    const Bvh bvh = build_bvh(mesh);
    std::vector<Vec3> q;
    {
        std::ifstream in(argv[3], std::ios::binary);
        double x[3];
        while (in.read(reinterpret_cast<char*>(x), sizeof x)) q.emplace_back(x[0], x[1], x[2]);
    }
    const int prec = std::atoi(argv[4]);
    SmoothParams p;
    p.alpha = std::atof(argv[5]);
    p.beta = std::atof(argv[6]);
    const double td = prec == SD_FP64 ? 1e-10 : 1e-5, tg = prec == SD_FP64 ? 1e-9 : 1e-4;

    gpu::Backend gpu(0, prec);
    gpu.upload(mesh, ws, &bvh);
    const Bvh back = gpu.tree();
    check(back.nodes.size() == bvh.nodes.size() &&
              std::memcmp(back.nodes.data(), bvh.nodes.data(), bvh.nodes.size() * sizeof(BvhNode)) == 0,
          "uploaded tree round-trips (BvhNode layout)", double(back.nodes.size()));

    // point queries: tree path and flat path against the reference per query
    const auto gt = gpu.smooth_min_dist(q, p);
    const auto ge = gpu.smooth_min_dist_flat(q, p);
    double ed = 0, eg = 0, edx = 0, egx = 0;
    bool counters = true, inf_ok = true;
    for (std::size_t i = 0; i < q.size(); ++i) {
        const SmoothResult r = smooth_min_dist(mesh, bvh, ws, q[i], p);
        const SmoothResult re = smooth_min_dist_flat(mesh, ws, SimplexGeom::point(q[i]), p);
        counters &= gt[i].leaves == r.leaves && gt[i].far_field == r.far_field &&
                    ge[i].leaves == std::int64_t(mesh.num_simplices());
        auto acc = [&](const SmoothResult& a, const SmoothResult& b, double& e1, double& e2) {
            if (std::isfinite(b.d_hat) != std::isfinite(a.d_hat)) inf_ok = false;
            if (!std::isfinite(b.d_hat)) return;
            e1 = std::max(e1, std::abs(a.d_hat - b.d_hat) / std::max(1.0, std::abs(b.d_hat)));
            e2 = std::max(e2, (a.grad - b.grad).norm() / std::max(1.0, b.grad.norm()));
        };
        acc(gt[i], r, ed, eg);
        acc(ge[i], re, edx, egx);
    }
    check(counters, "tree counters = reference, exact leaves = N", double(q.size()));
    {  // pipelined submission: the same results as the blocking batch
        std::vector<double> d0(q.size()), g0(3 * q.size()), d1(q.size()), g1(3 * q.size());
        const std::int64_t t0 = gpu.submit(q, p, d0.data(), g0.data());
        const std::int64_t t1 = gpu.submit(q, p, d1.data(), g1.data(), true);
        gpu.wait(t0);
        gpu.wait(t1);
        bool same = true;
        for (std::size_t i = 0; i < q.size(); ++i) {
            same &= (d0[i] == gt[i].d_hat || (std::isnan(d0[i]) && std::isnan(gt[i].d_hat))) && d1[i] == ge[i].d_hat;
            for (int a = 0; a < 3; ++a) same &= g0[3 * i + a] == gt[i].grad(a) && g1[3 * i + a] == ge[i].grad(a);
        }
        check(same, "submit / wait = the blocking batches", 0.0);
    }
    check(inf_ok, "+inf agrees", 0.0);
    check(ed <= td && eg <= tg, "smooth_min_dist (tree) d_hat / grad", std::max(ed, eg));
    check(edx <= td && egx <= tg, "smooth_min_dist_flat d_hat / grad", std::max(edx, egx));
    {  // pruned exact evaluation against the reference's flat sum, same tolerances
        gpu.set_exact_pruning(prec == SD_FP64 ? 64.0 : 48.0);
        const auto gp = gpu.smooth_min_dist_flat(q, p);
        gpu.set_exact_pruning(0.0);
        double epd = 0, epg = 0;
        bool pinf = true;
        for (std::size_t i = 0; i < q.size(); ++i) {
            const SmoothResult re = smooth_min_dist_flat(mesh, ws, SimplexGeom::point(q[i]), p);
            if (std::isfinite(re.d_hat) != std::isfinite(gp[i].d_hat)) pinf = false;
            if (!std::isfinite(re.d_hat)) continue;
            epd = std::max(epd, std::abs(gp[i].d_hat - re.d_hat) / std::max(1.0, std::abs(re.d_hat)));
            epg = std::max(epg, (gp[i].grad - re.grad).norm() / std::max(1.0, re.grad.norm()));
        }
        check(pinf && epd <= td && epg <= tg, "pruned smooth_min_dist_flat d_hat / grad", std::max(epd, epg));
    }

    // query simplices (edges / triangles from consecutive query points): fp64 path
    std::vector<SimplexGeom> g;
    for (std::size_t i = 0; i + 2 < q.size() && g.size() < 64; i += 3) {
        g.push_back(g.size() % 2 ? SimplexGeom::edge(q[i], q[i + 1]) : SimplexGeom::triangle(q[i], q[i + 1], q[i + 2]));
    }
    const auto gs = gpu.smooth_min_dist(g, p);
    double es = 0;
    bool scount = true;
    for (std::size_t i = 0; i < g.size(); ++i) {
        const SmoothResult r = smooth_min_dist(mesh, bvh, ws, g[i], p);
        scount &= gs[i].leaves == r.leaves && gs[i].far_field == r.far_field;
        if (std::isfinite(r.d_hat)) es = std::max(es, std::abs(gs[i].d_hat - r.d_hat) / std::max(1.0, std::abs(r.d_hat)));
    }
    check(scount, "simplex queries: counters = reference", double(g.size()));
    check(es <= 1e-10, "simplex queries: d_hat (fp64 path)", es);

    // mesh-to-mesh: the first simplices of the mesh, shifted, as the query mesh
    SimplexMesh qm;
    for (std::size_t i = 0; i < std::min<std::size_t>(40, mesh.num_simplices()); ++i) {
        Simplex s = mesh.simplices[i];
        for (int k = 0; k < s.nverts(); ++k) {
            qm.vertices.push_back(mesh.vertices[std::size_t(s.v[std::size_t(k)])] + Vec3(0.02, -0.01, 0.015));
            s.v[std::size_t(k)] = std::int32_t(qm.vertices.size() - 1);
        }
        qm.simplices.push_back(s);
    }
    const MeshDistResult mg = gpu.smooth_mesh_dist(qm, p);
    const MeshDistResult mr = smooth_mesh_dist(mesh, bvh, ws, qm, p);
    check(std::abs(mg.d_hat - mr.d_hat) <= td * std::max(1.0, std::abs(mr.d_hat)), "smooth_mesh_dist d_hat",
          std::abs(mg.d_hat - mr.d_hat));
    std::printf("%s\n", g_fail ? "BACKEND CHECK FAILED" : "BACKEND CHECK OK");
    return g_fail ? 1 : 0;
}
