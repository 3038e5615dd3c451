"""GPU parity: the CUDA path (through the C ABI of include/sdgpu.h) against
the CPU oracle on the same seeded inputs and the same WeightSet table.

Tolerances (BASELINE.json north_star):
  fp32: |d - d_ref| <= 1e-5 max(1, |d_ref|),  |g - g_ref| <= 1e-4 max(1, |g_ref|)
  fp64: |d - d_ref| <= 1e-10 max(1, |d_ref|), |g - g_ref| <= 1e-9 max(1, |g_ref|)
  +inf must agree except in the tie band |alpha d_min - 708| < 1e-3.
fp32 inputs (vertices, queries) are rounded to float before either side
sees them, so parity measures arithmetic, not input rounding.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = {0: (1e-5, 1e-4), 1: (1e-10, 1e-9)}


def engine_for(sd, O, mesh, weights, prec, tree=None):
    e = sd.Engine(0, prec)
    e.set_geometry(mesh.vertices, mesh.simplices, mesh.kinds)
    e.set_weight_table(weights.table)
    if tree is not None:
        e.set_bvh(tree.nodes())
    return e


def prep(O, mesh, q, prec):
    if prec == 0:
        mesh = mesh.quantized()
        q = np.asarray(q, np.float32).astype(np.float64)
    return mesh, np.ascontiguousarray(q, np.float64)


def assert_close(got, ref, prec, alpha=None, what=""):
    td, tg = TOL[prec]
    fin = np.isfinite(ref.d_hat)
    bad_inf = np.isfinite(got.d_hat) != fin
    if bad_inf.any():
        # allowed only in the -708 tie band
        assert alpha is not None, f"{what}: inf mismatch at {np.nonzero(bad_inf)[0][:5]}"
        band = np.abs(-np.log(np.maximum(ref.c, 1e-320)) - 708.0) < 1e-2
        assert (band | ~bad_inf).all(), f"{what}: inf mismatch outside the tie band"
    both = fin & np.isfinite(got.d_hat)
    err = np.abs(got.d_hat[both] - ref.d_hat[both]) / np.maximum(1.0, np.abs(ref.d_hat[both]))
    assert err.size == 0 or err.max() <= td, f"{what}: d_hat err {err.max():.3g} > {td}"
    gref = ref.grad[both]
    gerr = np.linalg.norm(got.grad[both] - gref, axis=1) / np.maximum(1.0, np.linalg.norm(gref, axis=1))
    assert gerr.size == 0 or gerr.max() <= tg, f"{what}: grad err {gerr.max():.3g} > {tg}"
    assert not got.grad[~np.isfinite(got.d_hat)].any(), f"{what}: nonzero gradient at +inf"


# -------------------------------------------------------- known answers
@pytest.mark.parametrize("prec", [0, 1])
def test_known_answers_on_gpu(sd, oracle, prec):
    O = oracle
    # SinglePointClosedForm (test_smooth.cpp:40-55)
    m = O.Mesh.from_arrays([[0, 0, 0]], [[0, -1, -1]], [0])
    q = np.array([[0.3, -0.2, 0.6]])
    e = engine_for(sd, O, m, O.Weights.build(m), prec)
    r = e.smooth_min_dist_flat(q.astype(np.float32).astype(float) if prec == 0 else q,
                               sd.SmoothParams(alpha=50.0, beta=0.0))
    qq = q.astype(np.float32).astype(float) if prec == 0 else q
    tol = 1e-6 if prec == 0 else 1e-12
    assert abs(r.d_hat[0] - np.linalg.norm(qq)) < tol
    assert np.abs(r.grad[0] - qq[0] / np.linalg.norm(qq)).max() < tol
    assert r.leaves[0] == 1 and r.far_field[0] == 0
    # CoincidentPointsShiftByLogCount (:57-72)
    p = [0.1, 0.2, 0.3]
    m = O.Mesh.from_arrays([p, p], [[0, -1, -1], [1, -1, -1]], [0, 0])
    with pytest.raises(sd.SdError):  # coincident corners are only rejected within a simplex
        sd.Engine(0, prec).set_geometry([[0, 0, 0], [0, 0, 0]], [[0, 1, -1]], [1])
    e = engine_for(sd, O, m, O.Weights.build(m), prec)
    r = e.smooth_min_dist_flat([[1.0, 0.0, 0.0]], sd.SmoothParams(alpha=80.0, beta=0.0))
    pp = np.array(p, np.float32).astype(float) if prec == 0 else np.array(p)
    d = np.linalg.norm(np.array([1.0, 0, 0]) - pp)
    assert abs(r.d_hat[0] - (d - math.log(2.0) / 80.0)) < tol
    # FarQueryUnderflowsToInfinity (:201-219)
    m = O.point_cluster(20, 2, 0.05)
    e = engine_for(sd, O, m, O.Weights.build(m), prec)
    r = e.smooth_min_dist_flat([[3.0, 0.0, 0.0]], sd.SmoothParams(alpha=400.0, beta=0.0))
    assert r.c[0] == 0.0 and math.isinf(r.d_hat[0]) and not r.grad.any()
    r = e.smooth_min_dist_flat([[3.0, 0.0, 0.0]], sd.SmoothParams(alpha=200.0, beta=0.0))
    assert math.isfinite(r.d_hat[0]) and abs(np.linalg.norm(r.grad[0]) - 1.0) < 1e-3


@pytest.mark.parametrize("prec", [0, 1])
def test_far_cluster_collapses_on_gpu(sd, oracle, prec):  # test_smooth.cpp:74-90
    O = oracle
    m = O.point_cluster(4, 3, 1e-3)
    mq, q = prep(O, m, [[2.0, 0.4, -0.3]], prec)
    t = O.Tree.build(mq)
    e = engine_for(sd, O, mq, O.Weights.build(mq), prec, tree=t)
    r = e.smooth_min_dist(q, sd.SmoothParams(alpha=100.0, beta=0.9))
    assert r.far_field[0] == 1 and r.leaves[0] == 0
    root = t.nodes()[0]
    d, _ = O.box_point_proximity(root["lo"], root["hi"], q)
    assert abs(r.d_hat[0] - (d[0] - math.log(4.0) / 100.0)) < (1e-6 if prec == 0 else 1e-12)


# ------------------------------------------------------ seeded scenes
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("seed", list(range(1, 13)))
def test_random_scene_exact(sd, oracle, prec, seed):
    O = oracle
    m0 = O.random_scene(seed, 200)
    qs = O.QueryStream(1000 + seed).draw_points(m0, 300)
    m, q = prep(O, m0, qs, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    for alpha, alpha_u in ((100.0, 600.0), (20.0, 600.0), (900.0, 600.0)):
        p = O.Params(alpha=alpha, alpha_u=alpha_u, beta=0.0)
        ref = O.query(m, w, q, p)
        got = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=alpha, alpha_u=alpha_u, beta=0.0))
        assert_close(got, ref, prec, alpha, f"seed {seed} alpha {alpha}")
        assert (got.leaves == m.num_simplices).all() and not got.far_field.any()


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("seed", list(range(1, 9)))
def test_random_scene_tree_decisions(sd, oracle, prec, seed):
    """BVH path on the reference median tree: identical far-field / leaf
    decisions (per-query counters and decision hash) and parity of d_hat."""
    O = oracle
    m0 = O.random_scene(seed, 200)
    qs = O.QueryStream(2000 + seed).draw_points(m0, 300)
    m, q = prep(O, m0, qs, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    for beta in (0.3, 0.5, 0.9):
        p = O.Params(alpha=100.0, beta=beta)
        ref = O.query(m, w, q, p, tree=t)
        got = e.smooth_min_dist(q, sd.SmoothParams(alpha=100.0, beta=beta))
        assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
        assert (got.decision_hash == ref.decision_hash).all()
        assert_close(got, ref, prec, 100.0, f"seed {seed} beta {beta}")


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("split", ["0", "1", "3", "6", "", "frontier", "frontier32",
                                   "q3", "q16", "noq", "coop3", "coop24", "lanes40"])
def test_split_traversal_decisions(sd, oracle, prec, split, monkeypatch):
    """The few-query traversal modes visit exactly the oracle's nodes:
    the slot split (one warp per (packet, depth-k slot) after re-testing the
    slot's ancestors, merged in fp64) at every depth k, none ("0"), the
    automatic choice (""), and the node-parallel frontier kernel: counters
    and decision hash identical.
    "qL": the unsplit walk with per-lane deferred queues of L exact leaves
    (K3Q; small queues force many flushes); "noq": leaf terms inline;
    "coopL" / "lanesL": the warp-cooperative flush / per-lane rounds."""
    O = oracle
    if split.startswith("coop") or split.startswith("lanes"):
        monkeypatch.setenv("SDGPU_FRONTIER", "0")
        monkeypatch.setenv("SDGPU_SPLIT", "0")
        monkeypatch.setenv("SDGPU_LEAF_QUEUE", "1")
        monkeypatch.setenv("SDGPU_LEAF_COOP", "1" if split.startswith("coop") else "0")
        monkeypatch.setenv("SDGPU_LEAFQ", split.lstrip("coplanes"))
    elif split.startswith("q") or split == "noq":
        monkeypatch.setenv("SDGPU_FRONTIER", "0")
        monkeypatch.setenv("SDGPU_SPLIT", "0")
        monkeypatch.setenv("SDGPU_LEAF_QUEUE", "0" if split == "noq" else "1")
        monkeypatch.setenv("SDGPU_LEAFQ", split[1:] if split != "noq" else "16")
    elif split.startswith("frontier"):
        monkeypatch.setenv("SDGPU_FRONTIER", "1")
        monkeypatch.setenv("SDGPU_FRONTIER_G", split[8:] or "4")
    else:
        monkeypatch.setenv("SDGPU_FRONTIER", "0")
        monkeypatch.setenv("SDGPU_SPLIT", split)
    m0 = O.random_scene(7, 400)
    qs = O.QueryStream(4242).draw_points(m0, 777)  # ragged last packet
    m, q = prep(O, m0, qs, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    for beta in (0.2, 0.6):
        p = O.Params(alpha=150.0, beta=beta)
        ref = O.query(m, w, q, p, tree=t)
        got = e.smooth_min_dist(q, sd.SmoothParams(alpha=150.0, beta=beta))
        assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
        assert (got.decision_hash == ref.decision_hash).all()
        assert_close(got, ref, prec, 150.0, f"split {split!r} beta {beta}")


@pytest.mark.parametrize("prec", [0, 1])
def test_gpu_median_build_matches_reference_tree(sd, oracle, prec):
    O = oracle
    for seed in (1, 5, 9):
        m, _ = prep(O, O.random_scene(seed, 200), np.zeros((1, 3)), prec)
        e = engine_for(sd, O, m, O.Weights.build(m), prec)
        e.build_bvh(sd.SD_BVH_MEDIAN)
        got, ref = e.export_bvh(), O.Tree.build(m).nodes()
        assert got.tobytes() == ref.tobytes()


def check_tree_structure(nodes, n):
    """bvh.hpp invariants (T/test_bvh.cpp:27-59) + the pre-order layout."""
    assert len(nodes) == 2 * n - 1 and nodes[0]["count"] == n
    leaf = nodes["left"] < 0
    assert sorted(nodes["primitive"][leaf].tolist()) == list(range(n))
    assert (nodes["count"][leaf] == 1).all()
    idx = np.nonzero(~leaf)[0]
    assert (nodes["left"][idx] == idx + 1).all()
    l, r = nodes[nodes["left"][idx]], nodes[nodes["right"][idx]]
    assert (nodes["count"][idx] == l["count"] + r["count"]).all()
    assert (nodes["lo"][idx] == np.minimum(l["lo"], r["lo"])).all()
    assert (nodes["hi"][idx] == np.maximum(l["hi"], r["hi"])).all()
    e = nodes["hi"] - nodes["lo"]
    diag = np.sqrt((e[:, 0] * e[:, 0] + e[:, 1] * e[:, 1]) + e[:, 2] * e[:, 2])
    assert (nodes["diameter"] == diag).all()


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 11, 12])
def test_lbvh_structure_and_decisions(sd, oracle, prec, seed):
    """GPU-built LBVH, exported in the reference layout: structure
    invariants, and the oracle traversing the exported tree makes exactly
    the GPU's far-field / leaf decisions."""
    O = oracle
    m0 = O.random_scene(seed, 200)
    qs = O.QueryStream(3000 + seed).draw_points(m0, 200)
    m, q = prep(O, m0, qs, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    e.build_bvh(sd.SD_BVH_LBVH)
    nodes = e.export_bvh()
    check_tree_structure(nodes, m.num_simplices)
    t = O.Tree.from_nodes(nodes)
    for beta in (0.3, 0.7):
        ref = O.query(m, w, q, O.Params(alpha=100.0, beta=beta), tree=t)
        got = e.smooth_min_dist(q, sd.SmoothParams(alpha=100.0, beta=beta))
        assert (got.decision_hash == ref.decision_hash).all()
        assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
        assert_close(got, ref, prec, 100.0, f"lbvh seed {seed} beta {beta}")


def test_lbvh_tiny_meshes(sd, oracle):
    O = oracle
    for verts, simp, kinds in (([[0, 0, 0]], [[0, -1, -1]], [0]),
                               ([[0, 0, 0], [1, 0, 0]], [[0, -1, -1], [1, -1, -1]], [0, 0]),
                               ([[0, 0, 0], [1, 0, 0], [0, 1, 0]], [[0, 1, 2]], [2])):
        m = O.Mesh.from_arrays(verts, simp, kinds)
        e = engine_for(sd, O, m, O.Weights.build(m), 1)
        e.build_bvh(sd.SD_BVH_LBVH)
        check_tree_structure(e.export_bvh(), m.num_simplices)
        r = e.smooth_min_dist([[3.0, 0.5, 0.25]], sd.SmoothParams(alpha=50.0, beta=0.5))
        assert np.isfinite(r.d_hat).all()


# --------------------------------------------------- BASELINE configs
def _cfg(O, cfg, nq, prec):
    m = O.config_mesh(cfg)
    q = O.config_queries(cfg, m, nq)
    return prep(O, m, q, prec)


@pytest.mark.parametrize("cfg,prec,alphas,nq", [
    (1, 1, (50.0,), 2048),
    (2, 0, (100.0,), 1024),
    (2, 1, (100.0,), 512),
    (3, 0, (10.0, 100.0, 1000.0), 256),
])
def test_config_exact_parity(sd, oracle, cfg, prec, alphas, nq):
    O = oracle
    m, q = _cfg(O, cfg, nq, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    for alpha in alphas:
        p = O.Params(alpha=alpha, alpha_u=600.0, beta=0.0)
        ref = O.query(m, w, q, p)
        got = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=alpha, beta=0.0))
        assert_close(got, ref, prec, alpha, f"cfg{cfg} alpha {alpha}")


@pytest.mark.parametrize("builder,kernel", [("median", "K3F"), ("lbvh", "K3F"), ("lbvh", "K3"), ("median", "K3"),
                                            ("median", "K3NQ"), ("median", "K3L")])
def test_config4_tree_parity_subset(sd, oracle, builder, kernel, monkeypatch):
    """cfg4 (icosphere(9), 5.2M triangles, beta 0.5, alpha 200) on a query
    subset (both halves of the query distribution): decisions identical to
    the oracle on the same tree -- the reference median tree, or the GPU
    LBVH exported to the oracle -- and the Barnes-Hut field below the exact
    one (acceptance [1]); both traversal kernels (K3F is the default for
    this batch size, K3 the one the full-size bench runs)."""
    O = oracle
    monkeypatch.setenv("SDGPU_FRONTIER", "1" if kernel == "K3F" else "0")
    if kernel in ("K3", "K3NQ", "K3L"):
        # the unsplit packet walk of the full-size batch: K3 = the default
        # K3Q (deferred leaf queues, cooperative flush in fp32), K3NQ =
        # inline leaf terms, K3L = per-lane leaf rounds
        monkeypatch.setenv("SDGPU_SPLIT", "0")
        monkeypatch.setenv("SDGPU_LEAF_QUEUE", "0" if kernel == "K3NQ" else "1")
        monkeypatch.setenv("SDGPU_LEAF_COOP", "0" if kernel == "K3L" else "1")
    m, q = _cfg(O, 4, 512, 0)
    w = O.Weights.build(m)
    if builder == "median":
        t = O.Tree.build(m)
        e = engine_for(sd, O, m, w, 0, tree=t)
    else:
        e = engine_for(sd, O, m, w, 0)
        e.build_bvh(sd.SD_BVH_LBVH)
        nodes = e.export_bvh()
        check_tree_structure(nodes, m.num_simplices)
        t = O.Tree.from_nodes(nodes)
    p = O.Params(alpha=200.0, beta=0.5)
    ref = O.query(m, w, q, p, tree=t)
    got = e.smooth_min_dist(q, sd.SmoothParams(alpha=200.0, beta=0.5))
    assert (got.decision_hash == ref.decision_hash).all()
    assert_close(got, ref, 0, 200.0, "cfg4 bvh")
    ex = e.smooth_min_dist_flat(q[:64], sd.SmoothParams(alpha=200.0, beta=0.0))
    assert (got.d_hat[:64] <= ex.d_hat + 1e-5).all()


@pytest.mark.parametrize("kernel", ["K3", "K3F"])
def test_config4_parity_65536_queries(sd, oracle, kernel, monkeypatch):
    """cfg4 at the scale BASELINE configs[3] names for its exact comparison:
    65,536 queries (32,768 from each half of the distribution), the median
    tree built on the GPU and exported to the oracle. Every query's decision
    hash and counters equal the oracle's; d_hat / grad within the fp32
    tolerance in both forms (max(1, |ref|) and the strict relative form
    with a 1/alpha floor); Barnes-Hut below exact + 1e-5 on every query
    (acceptance [1], T/acceptance.cpp:76-115). K3 = the packet walk of the
    full-size batch, K3F = the node-parallel kernel this batch size picks
    by default."""
    O = oracle
    monkeypatch.setenv("SDGPU_FRONTIER", "1" if kernel == "K3F" else "0")
    monkeypatch.setenv("SDGPU_SPLIT", "0")
    m = O.config_mesh(4).quantized()
    qa = O.config_queries(4, m, 1 << 17)
    q = np.concatenate([qa[:32768], qa[65536:65536 + 32768]]).astype(np.float32).astype(np.float64)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, 0)
    e.build_bvh(sd.SD_BVH_MEDIAN)
    t = O.Tree.from_nodes(e.export_bvh())
    P = sd.SmoothParams(alpha=200.0, beta=0.5)
    got = e.smooth_min_dist(q, P)
    ref = O.query(m, w, q, O.Params(alpha=200.0, beta=0.5), tree=t)
    assert (got.decision_hash == ref.decision_hash).all()
    assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
    assert_close(got, ref, 0, 200.0, "cfg4 65536")
    fin = np.isfinite(ref.d_hat)
    strict = np.abs(got.d_hat[fin] - ref.d_hat[fin]) / np.maximum(np.abs(ref.d_hat[fin]), 1.0 / 200.0)
    assert strict.max() <= 1e-5, strict.max()
    gs = np.linalg.norm(got.grad[fin] - ref.grad[fin], axis=1) / np.maximum(np.linalg.norm(ref.grad[fin], axis=1), 1e-3)
    assert gs.max() <= 1e-4, gs.max()
    ex = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=200.0, beta=0.0))
    both = np.isfinite(ex.d_hat) & fin
    assert (got.d_hat[both] <= ex.d_hat[both] + 1e-5).all()


def test_config4_whole_batch_fp32_against_fp64(sd):
    """The whole cfg4 batch (4,194,304 queries, the bench's BVH leg): the
    fp32 tree path (K3Q + the K3C near-contact correction) against the fp64
    tree path, which matches the compiled reference to ~1e-13 (bench parity,
    test_config4_parity_65536_queries at fp64). Same decisions and counters
    on every query; d_hat within 1e-5 and grad within 1e-4 in the STRICT
    relative forms (floors 1/alpha and 1e-3). Without K3C, 110 queries
    within ~1e-6 of a face failed the gradient bound (up to 2e-2 relative:
    their fp32 face offsets are rounding noise in direction)."""
    from paper_2108_10480_b200 import configs
    w, q = configs.cfg4()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
    res = {}
    for prec in (sd.SD_FP32, sd.SD_FP64):
        e = sd.Engine(0, prec)
        e.set_geometry(v, w.simplices, w.kinds)
        e.build_weights()
        e.build_bvh(sd.SD_BVH_MEDIAN)
        res[prec] = e.smooth_min_dist(q, P)
        e.close()
    a, b = res[sd.SD_FP32], res[sd.SD_FP64]
    assert (a.decision_hash == b.decision_hash).all()
    assert (a.leaves == b.leaves).all() and (a.far_field == b.far_field).all()
    fin = np.isfinite(b.d_hat)
    assert (np.isfinite(a.d_hat) == fin).all()
    dd = np.abs(a.d_hat[fin] - b.d_hat[fin]) / np.maximum(np.abs(b.d_hat[fin]), 1.0 / w.alpha)
    assert dd.max() <= 1e-5, dd.max()
    gn = np.linalg.norm(b.grad[fin], axis=1)
    gs = np.linalg.norm(a.grad[fin] - b.grad[fin], axis=1) / np.maximum(gn, 1e-3)
    assert gs.max() <= 1e-4, (gs.max(), int((gs > 1e-4).sum()))


@pytest.mark.parametrize("kernel", ["K3Q", "K3F"])
def test_exact_gradient_finite_at_contact(sd, oracle, kernel, monkeypatch):
    """A query within ~1e-9 of a face (cfg4 has ~100 such queries): the fp32
    exact kernel's tile shift allows terms up to 2^H, and with r = 1/d ~ 4e8
    the gradient product overflowed to -inf at H = 100 (exact.cu); it must
    stay finite; the tree path must resolve the offset direction like the
    fp64 path (tri_contact: K3Q + K3C or K3F inline)."""
    O = oracle
    monkeypatch.setenv("SDGPU_FRONTIER", "1" if kernel == "K3F" else "0")
    monkeypatch.setenv("SDGPU_SPLIT", "0")
    m = O.icosphere(4).quantized()
    w = O.Weights.build(m)
    V = m.vertices
    f = m.simplices[7]
    p = (V[f[0]] + V[f[1]] + V[f[2]]) / 3.0
    n = np.cross(V[f[1]] - V[f[0]], V[f[2]] - V[f[0]])
    n /= np.linalg.norm(n)
    q = np.array([p + t * n for t in (2e-9, -3e-9, 1e-7, 5e-6)], np.float32).astype(np.float64)
    out = {}
    for prec in (0, 1):
        e = engine_for(sd, O, m, w, prec)
        e.build_bvh(sd.SD_BVH_MEDIAN)
        out[prec, "exact"] = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=200.0, beta=0.0))
        out[prec, "tree"] = e.query_points(q, sd.SmoothParams(alpha=200.0, beta=0.5), sd.SD_BVH, want_c=True)
    for mode in ("exact", "tree"):
        g32, g64 = out[0, mode].grad, out[1, mode].grad
        assert np.isfinite(g32).all(), (mode, g32)
        gs = np.linalg.norm(g32 - g64, axis=1) / np.maximum(np.linalg.norm(g64, axis=1), 1e-3)
        # strict parity on the tree path (K3Q + K3C, or K3F inline); K1 keeps
        # the cancelling offset form (DESIGN: near-contact faces): finite only
        if mode == "tree":
            assert gs.max() <= 1e-4, (mode, gs)


# ---------------------------------------------- full-size properties
def test_config3_full_size_properties(sd, oracle):
    """cfg3 at the BASELINE size (1,048,576 queries x 262,144 triangles):
    properties that need no oracle -- finite/inf consistent with the -708
    rule, translation invariance under a float-exact shift, and exact
    parity on a strided sample."""
    O = oracle
    m, q = _cfg(O, 3, 1 << 20, 0)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, 0)
    P = sd.SmoothParams(alpha=100.0, beta=0.0)
    r = e.query_points(q, P, sd.SD_EXACT)
    assert np.isfinite(r.d_hat).mean() > 0.5
    shift = np.array([0.5, -0.25, 1.0])
    e2 = engine_for(sd, O, O.Mesh.from_arrays(m.vertices + shift, m.simplices, m.kinds), w, 0)
    r2 = e2.query_points(q + shift, P, sd.SD_EXACT)
    fin = np.isfinite(r.d_hat)
    assert (np.isfinite(r2.d_hat) == fin).all()
    assert np.abs(r2.d_hat[fin] - r.d_hat[fin]).max() < 1e-4
    idx = np.arange(0, len(q), 4099)[:128]
    ref = O.query(m, w, q[idx], O.Params(alpha=100.0, beta=0.0))
    sub = type(r)(r.d_hat[idx], r.grad[idx])
    assert_close(sub, ref, 0, 100.0, "cfg3 strided")


# --------------------------------------------------------- edge cases
def test_edge_cases(sd, oracle):
    O = oracle
    e = sd.Engine(0, sd.SD_FP32)
    e.set_geometry(np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros(0, np.uint8))
    e.set_weights(1.0, 1.0, np.zeros((0, 5)), np.zeros((0, 13)), np.zeros(0, np.int32))
    r = e.query_points([[1, 2, 3]], sd.SmoothParams(beta=0.0), sd.SD_EXACT, want_c=True, want_counters=True)
    assert math.isinf(r.d_hat[0]) and not r.grad.any() and r.c[0] == 0.0
    m = O.random_scene(3, 200)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m.quantized(), w, 0)
    r = e.query_points(np.zeros((0, 3)), sd.SmoothParams(beta=0.0))
    assert r.d_hat.shape == (0,)
    # query exactly on a vertex: contact term, zero distance gradient
    mq = m.quantized()
    v = mq.vertices[mq.simplices[0, 0]][None, :]
    ref = O.query(mq, w, v, O.Params(beta=0.0))
    got = e.query_points(v, sd.SmoothParams(beta=0.0))
    assert_close(got, ref, 0, 100.0, "on-vertex")
    with pytest.raises(sd.SdError):
        e.query_points(v, sd.SmoothParams(alpha=-1.0))
    with pytest.raises(sd.SdError):
        e.query_points(v, sd.SmoothParams(beta=0.5), sd.SD_BVH)  # no tree yet
    with pytest.raises(sd.SdError):
        sd.Engine(0, sd.SD_FP32).set_geometry([[0, 0, 0], [1, 0, 0], [2, 0, 0]], [[0, 1, 2]], [2])  # zero area
    with pytest.raises(sd.SdError):
        sd.Engine(0, sd.SD_FP32).set_geometry([[0, 0, 0]], [[0, 5, -1]], [1])  # index out of range


# ------------------------------------------------- host weight build
@pytest.mark.parametrize("case", ["scenes", "cfg2", "cfg3", "cfg4", "valences"])
def test_build_weights_matches_oracle(sd, oracle, case):
    """sd_build_weights (pivoted-QR construction) against the oracle's
    restated build_weight_set (Jacobi-SVD construction): identical valence
    bookkeeping (poly_index, A, edge polynomials). Triangle polynomials are
    only defined up to ties of the null-space LP (weights.hpp:277-334,
    which vertex wins depends on the SVD basis), so each product polynomial
    is checked for the construction's defining properties instead: the
    interpolation targets (test_weights.cpp:56-67), exact symmetry and zero
    normal derivative on the legs (:69-88), and a domain minimum no worse
    than the oracle's (the LP objective)."""
    O = oracle
    if case == "scenes":
        meshes = [O.random_scene(s, 200) for s in range(1, 16)]
    elif case == "valences":
        meshes = [O.triangle_fan(k, 40 + k) for k in range(2, 9)] + [O.random_scene(s, 200) for s in (21, 22, 23)]
    else:
        meshes = [O.config_mesh(int(case[-1]))]
    g = np.array([[i / 64, j / 64] for i in range(65) for j in range(65 - i)])
    for m in meshes:
        e = sd.Engine(0, sd.SD_FP64)
        e.set_geometry(m.vertices, m.simplices, m.kinds)
        got = e.build_weights()
        ref = O.Weights.build(m).table
        assert got.A == ref.A
        assert np.array_equal(got.poly_index, ref.poly_index)
        assert np.array_equal(got.edge_a, ref.edge_a)
        assert got.tri_stored.shape == ref.tri_stored.shape
        for p, (v, ev) in enumerate(ref.tri_val):
            st = got.tri_stored[p]
            targets = [(0, 0, 1 / v), (1, 0, 1 / v), (0, 1, 1 / v), (1 / 3, 0, 1 / ev), (2 / 3, 0, 1 / ev),
                       (1 / 3, 2 / 3, 1 / ev), (1 / 3, 1 / 3, (v - 1) / v)]
            val, _, _ = O.tri_poly_eval(st, [[x, y] for x, y, _ in targets])
            assert np.abs(val - [t for *_, t in targets]).max() < 1e-7, (v, ev)
            grid = O.tri_poly_grid(st)
            assert np.array_equal(grid, grid.T) and not grid[1].any()
            mg = O.tri_poly_eval(st, g)[0].min()
            mo = O.tri_poly_eval(ref.tri_stored[p], g)[0].min()
            assert mg >= mo - 1e-6, (v, ev, mg, mo)


# ------------------------------------- primitive sharding on one device
@pytest.mark.parametrize("prec,beta", [(1, 0.0), (0, 0.0), (0, 0.5)])
def test_virtual_primitive_shards(sd, oracle, prec, beta):
    """cfg5 merge path with 3 virtual shards on one GPU: each shard's engine
    writes its unshifted fp64 partials (c, grad_c), they are summed (the
    all_reduce of the multi-GPU run) and sd_finalize_device finishes. Must
    equal the oracle on the whole mesh (beta = 0), or the oracle on the same
    per-shard trees (beta > 0)."""
    import torch
    from paper_2108_10480_b200 import sharding
    O = oracle
    m0 = O.random_scene(6, 200)
    q0 = O.QueryStream(60).draw_points(m0, 400)
    m, q = prep(O, m0, q0, prec)
    wt = O.Weights.build(m).table
    shards = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, wt.poly_index, 3)
    P = sd.SmoothParams(alpha=100.0, beta=beta)
    c_sum, g_sum = np.zeros(len(q)), np.zeros((len(q), 3))
    ref_c, ref_g = np.zeros(len(q)), np.zeros((len(q), 3))
    for s in shards:
        e = sd.Engine(0, prec)
        e.set_geometry(s.vertices, s.simplices, s.kinds)
        e.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index)
        sm = O.Mesh.from_arrays(s.vertices, s.simplices, s.kinds)
        sw = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index))
        tree = None
        if beta > 0:
            e.build_bvh(sd.SD_BVH_LBVH)
            tree = O.Tree.from_nodes(e.export_bvh())
        r = e.query_points(q, P, sd.SD_BVH if beta > 0 else sd.SD_EXACT, want_c=True)
        c_sum += r.c
        g_sum += r.grad_c
        rr = O.query(sm, sw, q, O.Params(alpha=100.0, beta=beta), tree=tree)
        ref_c += rr.c
        ref_g += rr.grad_c
    dev = torch.device("cuda", 0)
    c_d = torch.tensor(c_sum, device=dev)
    g_d = torch.tensor(g_sum, device=dev)
    d_d = torch.empty(len(q), dtype=torch.float64, device=dev)
    gr_d = torch.empty(len(q), 3, dtype=torch.float64, device=dev)
    e.finalize_device(c_d.data_ptr(), g_d.data_ptr(), len(q), P, d_d.data_ptr(), gr_d.data_ptr())
    torch.cuda.synchronize()
    got = sd.SmoothResults(d_d.cpu().numpy(), gr_d.cpu().numpy())
    rd, rg = sharding.finalize(ref_c, ref_g, 100.0)
    ref = sd.SmoothResults(rd, rg)
    ref.c = ref_c
    assert_close(got, ref, prec, 100.0, "virtual shards")
    if beta == 0.0:
        whole = O.query(m, O.Weights.from_table(wt), q, O.Params(alpha=100.0, beta=0.0))
        fin = np.isfinite(whole.d_hat)
        assert np.abs(rd[fin] - whole.d_hat[fin]).max() < 1e-12


def test_config5_primitive_sharded_parity(sd, oracle):
    """BASELINE configs[4] (64 tori + 1M edges + 1M points, 18.8M
    primitives) in 4 Morton primitive shards, one GPU LBVH per shard, the
    global WeightSet: per-shard fp64 partials summed and finalised
    (sd_finalize_device) must match the oracle run on the same per-shard
    trees (beta = 0.5) and the oracle's flat sum over the whole mesh
    (beta = 0, on fewer queries)."""
    import torch
    from paper_2108_10480_b200 import sharding
    O = oracle
    m, q = _cfg(O, 5, 256, 0)
    wt = O.Weights.build(m).table
    shards = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, wt.poly_index, 4)
    dev = torch.device("cuda", 0)
    for beta, nq in ((0.5, 256), (0.0, 24)):
        qq = q[:nq]
        P = sd.SmoothParams(alpha=100.0, beta=beta)
        cs, gs = np.zeros(nq), np.zeros((nq, 3))
        rc, rg = np.zeros(nq), np.zeros((nq, 3))
        for s in shards:
            e = sd.Engine(0, sd.SD_FP32)
            e.set_geometry(s.vertices, s.simplices, s.kinds)
            e.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index)
            sm = O.Mesh.from_arrays(s.vertices, s.simplices, s.kinds)
            sw = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index))
            tree = None
            if beta > 0:
                e.build_bvh(sd.SD_BVH_LBVH)
                tree = O.Tree.from_nodes(e.export_bvh())
            r = e.query_points(qq, P, sd.SD_BVH if beta > 0 else sd.SD_EXACT, want_c=True, want_counters=True)
            rr = O.query(sm, sw, qq, O.Params(alpha=100.0, beta=beta), tree=tree)
            if beta > 0:
                assert (r.decision_hash == rr.decision_hash).all()
            cs += r.c
            gs += r.grad_c
            rc += rr.c
            rg += rr.grad_c
        d_d = torch.empty(nq, dtype=torch.float64, device=dev)
        g_d = torch.empty(nq, 3, dtype=torch.float64, device=dev)
        c_t, gc_t = torch.tensor(cs, device=dev), torch.tensor(gs, device=dev)
        e.finalize_device(c_t.data_ptr(), gc_t.data_ptr(), nq, P, d_d.data_ptr(), g_d.data_ptr())
        torch.cuda.synchronize()
        got = sd.SmoothResults(d_d.cpu().numpy(), g_d.cpu().numpy())
        rd, rgd = sharding.finalize(rc, rg, 100.0)
        ref = sd.SmoothResults(rd, rgd)
        ref.c = rc
        assert_close(got, ref, 0, 100.0, f"cfg5 beta {beta}")
        if beta == 0.0:
            whole = O.query(m, O.Weights.from_table(wt), qq, O.Params(alpha=100.0, beta=0.0))
            fin = np.isfinite(whole.d_hat)
            assert np.abs(rd[fin] - whole.d_hat[fin]).max() < 1e-10


# ------------------------------------------------------ weight regimes
@pytest.mark.parametrize("prec", [0, 1])
def test_unit_weight_tables(sd, oracle, prec):
    """unit_weight_set (weights.hpp:583-587): every primitive w = 1."""
    O = oracle
    m0 = O.random_scene(10, 200)
    m, q = prep(O, m0, O.QueryStream(77).draw_points(m0, 200), prec)
    w = O.Weights.unit(m)
    e = engine_for(sd, O, m, w, prec, tree=O.Tree.build(m))
    for beta in (0.0, 0.5):
        ref = O.query(m, w, q, O.Params(alpha=150.0, beta=beta), tree=O.Tree.build(m) if beta else None)
        got = (e.smooth_min_dist if beta else e.smooth_min_dist_flat)(q, sd.SmoothParams(alpha=150.0, beta=beta))
        assert_close(got, ref, prec, 150.0, f"unit weights beta {beta}")


@pytest.mark.parametrize("prec", [0, 1])
def test_floored_out_of_model_weights(sd, oracle, prec):
    """A polynomial that is negative on the domain triggers the reference's
    1e-300 floor (weights.hpp:657-661; test_weights.cpp:171-192): w =
    1e-300^S, dw = 0 -- finite, on the non-certified kernel path."""
    O = oracle
    m = O.Mesh.from_arrays([[0, 0, 0], [1, 0, 0], [0, 1, 0], [3, 0, 0], [4, 0, 0]],
                           [[0, 1, 2], [3, 4, -1]], [2, 1])
    stored = np.zeros((1, 13))
    stored[0, 0] = -2.0
    edge = np.array([[-1.0, 0, 0, 0, 0]])
    t = O.WeightTable(1.0, 1.0, edge, stored, np.array([0, 0], np.int32))
    w = O.Weights.from_table(t)
    q = np.array([[0.2, 0.3, 0.5], [3.5, 0.4, 0.0], [10.0, 10.0, 10.0]])
    mq, q = prep(O, m, q, prec)
    e = engine_for(sd, O, mq, w, prec)
    for alpha in (20.0, 100.0):
        ref = O.query(mq, w, q, O.Params(alpha=alpha, beta=0.0))
        got = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=alpha, beta=0.0))
        assert np.isfinite(ref.d_hat[:2]).all()
        assert_close(got, ref, prec, alpha, f"floored alpha {alpha}")


@pytest.mark.parametrize("prec", [0, 1])
def test_tree_path_at_beta_zero_equals_flat(sd, oracle, prec):
    """smooth_min_dist with beta = 0 walks the whole tree (every leaf exact,
    test_smooth.cpp:221-241): leaves = N, no far field, same field."""
    O = oracle
    m0 = O.random_scene(6, 200)
    m, q = prep(O, m0, O.QueryStream(31).draw_points(m0, 100), prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    e.build_bvh(sd.SD_BVH_LBVH)
    got = e.query_points(q, sd.SmoothParams(alpha=100.0, beta=0.0), sd.SD_BVH, want_c=True, want_counters=True)
    ref = O.query(m, w, q, O.Params(alpha=100.0, beta=0.0))
    assert (got.leaves == m.num_simplices).all() and not got.far_field.any()
    assert_close(got, ref, prec, 100.0, "tree beta 0")


# ------------------------------------------------- mesh-to-mesh (points)
@pytest.mark.parametrize("prec", [0, 1])
def test_mesh_dist_single_point_matches_point_field(sd, oracle, prec):  # test_smooth.cpp:263-280
    O = oracle
    m = O.icosphere(1)
    mq, q = prep(O, m, [[1.4, -0.2, 0.3]], prec)
    w = O.Weights.build(mq)
    e = engine_for(sd, O, mq, w, prec)
    P = sd.SmoothParams(beta=0.0)
    md = e.smooth_mesh_dist(q, P)
    pt = e.smooth_min_dist_flat(q, P)
    assert abs(md.d_hat - pt.d_hat[0]) < 1e-12 and md.per_primitive[0] == pt.d_hat[0]
    assert np.abs(md.vertex_grads[0] - pt.grad[0]).max() < 1e-12


@pytest.mark.parametrize("prec,beta", [(0, 0.0), (1, 0.0), (0, 0.5), (1, 0.5)])
def test_mesh_dist_point_cloud_parity(sd, oracle, prec, beta):
    """d_hat(M, cloud), per-point values and vertex gradients vs the oracle's
    smooth_mesh_dist restatement; softmin identity and bounds
    (test_smooth.cpp:282-304); shared vertices accumulate."""
    O = oracle
    m0 = O.random_scene(12, 200)
    cloud0 = O.point_cluster(64, 5, 0.6)
    m, _ = prep(O, m0, np.zeros((1, 3)), prec)
    cv = cloud0.vertices + np.array([0.3, -0.2, 0.4])
    if prec == 0:
        cv = cv.astype(np.float32).astype(np.float64)
    pts = np.concatenate([np.arange(64), [3, 3, 7]]).astype(np.int32)  # vertices 3, 7 carry extra points
    cloud = O.Mesh.from_arrays(cv, np.stack([pts, -np.ones_like(pts), -np.ones_like(pts)], 1), np.zeros(len(pts)))
    w = O.Weights.build(m)
    t = O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    P = sd.SmoothParams(alpha=100.0, beta=beta, alpha_q=40.0)
    got = e.smooth_mesh_dist(cv, P, query_points=pts)
    ref = O.mesh_dist(m, w, cloud, O.Params(alpha=100.0, beta=beta, alpha_q=40.0), tree=t if beta else None)
    td, tg = TOL[prec]
    assert abs(got.d_hat - ref.d_hat) <= td * max(1.0, abs(ref.d_hat))
    fin = np.isfinite(ref.per_primitive)
    assert np.abs(got.per_primitive[fin] - ref.per_primitive[fin]).max() <= td * max(1.0, np.abs(ref.per_primitive[fin]).max())
    assert np.abs(got.vertex_grads - ref.vertex_grads).max() <= tg * max(1.0, np.abs(ref.vertex_grads).max())
    mass = np.exp(-40.0 * (got.per_primitive - got.d_hat))
    assert abs(mass.sum() - 1.0) < 1e-6
    dmin = got.per_primitive.min()
    assert got.d_hat <= dmin + 1e-9 and got.d_hat >= dmin - np.log(len(pts)) / 40.0 - 1e-9


def test_mesh_dist_far_cloud_underflows(sd, oracle):
    """every inner distance +inf -> denom 0 -> d_hat +inf, zero gradients."""
    O = oracle
    m = O.point_cluster(20, 2, 0.05)
    e = engine_for(sd, O, m, O.Weights.build(m), 1)
    md = e.smooth_mesh_dist([[3.0, 0, 0], [0, 4.0, 0]], sd.SmoothParams(alpha=400.0, beta=0.0, alpha_q=20.0))
    assert np.isinf(md.d_hat) and not md.vertex_grads.any()


@pytest.mark.parametrize("case", ["cfg3", "cfg5_mixed_subset", "ties"])
def test_gpu_median_build_equals_host_build(sd, oracle, case, monkeypatch):
    """The device median build (median.cu: segmented reductions + stable
    segmented sorts per level) emits the host restatement's tree byte for
    byte -- at 262k triangles, on a mixed point/edge/triangle scene, and on
    a grid with exactly tied centroids (index tie-break)."""
    O = oracle
    if case == "cfg3":
        m = O.config_mesh(3)
    elif case == "cfg5_mixed_subset":
        m = O.random_scene(17, 5000)
    else:
        g = np.stack(np.meshgrid(np.arange(12.0), np.arange(9.0), np.arange(7.0), indexing="ij"), -1).reshape(-1, 3)
        g = np.concatenate([g, g])  # duplicated points: equal centroids everywhere
        m = O.Mesh.from_arrays(g, np.stack([np.arange(len(g)), -np.ones(len(g)), -np.ones(len(g))], 1), np.zeros(len(g)))
    e = sd.Engine(0, sd.SD_FP64)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.build_bvh(sd.SD_BVH_MEDIAN)
    gpu = e.export_bvh()
    monkeypatch.setenv("SDGPU_MEDIAN_HOST", "1")
    e.build_bvh(sd.SD_BVH_MEDIAN)
    assert gpu.tobytes() == e.export_bvh().tobytes()
    if case != "cfg3":
        assert gpu.tobytes() == O.Tree.build(m).nodes().tobytes()


def test_auto_tree_picks_the_smaller_surface_area_cost(sd, oracle):
    """SD_BVH_AUTO keeps whichever device tree (median split or LBVH) has
    the smaller sum of internal box areas; the result is one of the two
    exactly and traverses to the oracle's decisions."""
    O = oracle
    m = O.random_scene(19, 3000)
    e = sd.Engine(0, sd.SD_FP64)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.set_weight_table(O.Weights.build(m).table)
    trees = {}
    for k in (sd.SD_BVH_MEDIAN, sd.SD_BVH_LBVH, sd.SD_BVH_AUTO):
        e.build_bvh(k)
        trees[k] = e.export_bvh()

    def cost(t):
        ext = np.maximum(t["hi"] - t["lo"], 0)
        a = 2 * (ext[:, 0] * ext[:, 1] + ext[:, 1] * ext[:, 2] + ext[:, 0] * ext[:, 2])
        return a[t["left"] >= 0].sum() / a[0]
    best = sd.SD_BVH_MEDIAN if cost(trees[sd.SD_BVH_MEDIAN]) < cost(trees[sd.SD_BVH_LBVH]) else sd.SD_BVH_LBVH
    assert trees[sd.SD_BVH_AUTO].tobytes() == trees[best].tobytes()
    q = O.random_point_queries(5, m, 300)
    t = O.Tree.from_nodes(trees[sd.SD_BVH_AUTO])
    ref = O.query(m, O.Weights.build(m), q, O.Params(beta=0.5), tree=t)
    got = e.smooth_min_dist(q, sd.SmoothParams(beta=0.5))
    assert (got.decision_hash == ref.decision_hash).all()



def test_peer_exchange_with_virtual_ranks(sd, oracle):
    """The peer-memory merge of the primitive-sharded path (sd_scatter_partials
    + sd_reduce_owned) with 4 virtual ranks on one GPU: each rank's engine
    stores its partials into the four owners' buffers through a device
    pointer table, exactly as over NVLink, then every owner finalises its
    block. Equal to summing the partials and finalising (the all-reduce
    path), and to the oracle on the whole mesh."""
    import torch
    from paper_2108_10480_b200 import sharding
    O = oracle
    m = O.random_scene(11, 400)
    q = O.QueryStream(61).draw_points(m, 700)
    wt = O.Weights.build(m).table
    world = 4
    shards = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, wt.poly_index, world)
    P = sd.SmoothParams(alpha=100.0, beta=0.0)
    dev = torch.device("cuda", 0)
    n = len(q)
    per, counts = sharding.owner_blocks(n, world)
    sbufs = [torch.zeros(world * 4 * per, dtype=torch.float64, device=dev) for _ in range(world)]
    table = torch.tensor([b.data_ptr() for b in sbufs], dtype=torch.int64, device=dev)
    qd = torch.tensor(q, dtype=torch.float64, device=dev)
    partials = []
    for r, s in enumerate(shards):
        e = sd.Engine(0, sd.SD_FP64)
        e.set_geometry(s.vertices, s.simplices, s.kinds)
        e.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index)
        c = torch.empty(n, dtype=torch.float64, device=dev)
        g = torch.empty(n, 3, dtype=torch.float64, device=dev)
        d = torch.empty(n, dtype=torch.float64, device=dev)
        e.query_points_device(qd.data_ptr(), n, P, sd.SD_EXACT, d.data_ptr(), c_ptr=c.data_ptr(),
                              grad_c_ptr=g.data_ptr())
        e.scatter_partials(c.data_ptr(), g.data_ptr(), n, table.data_ptr(), world, r, per)
        torch.cuda.synchronize()
        partials.append((c.cpu().numpy(), g.cpu().numpy()))
    expect = sharding.exchange_reference(partials, per)
    d_all = np.zeros(n)
    for o in range(world):
        sb = sbufs[o].cpu().numpy().reshape(world, 4, per)
        lo = o * per
        for r in range(world):  # rank r's contribution landed in owner o's slot r
            assert np.array_equal(sb[r, 0, :counts[o]], partials[r][0][lo:lo + counts[o]])
            assert np.array_equal(sb[r, 1:, :counts[o]].T, partials[r][1][lo:lo + counts[o]])
        dd = torch.empty(max(1, counts[o]), dtype=torch.float64, device=dev)
        gg = torch.empty(max(1, counts[o]), 3, dtype=torch.float64, device=dev)
        e.reduce_owned(sbufs[o].data_ptr(), per, counts[o], world, P, dd.data_ptr(), gg.data_ptr())
        torch.cuda.synchronize()
        rd, rg = sharding.finalize(expect[o][0], expect[o][1], 100.0)
        got = dd.cpu().numpy()[:counts[o]]
        fin = np.isfinite(rd)
        assert (np.isfinite(got) == fin).all()
        assert np.abs(got[fin] - rd[fin]).max(initial=0.0) <= 1e-14 * max(1.0, np.abs(rd[fin]).max(initial=0.0))
        d_all[lo:lo + counts[o]] = got
    whole = O.query(m, O.Weights.from_table(wt), q, O.Params(alpha=100.0, beta=0.0))
    fin = np.isfinite(whole.d_hat)
    assert np.abs(d_all[fin] - whole.d_hat[fin]).max() < 1e-10


@pytest.mark.parametrize("seed", [1, 5, 9])
def test_fp64_kernel_math_is_near_ulp(sd, oracle, seed):
    """The fp64 path's branch-free exp2 / log2 / rsqrt / rcp (device_common.cuh
    Math<double>) keep d_hat and the gradient within a few hundred ulp of the
    oracle's libm results -- far inside the 1e-10 / 1e-9 parity bar -- on mixed
    scenes, at small and large alpha, at contact (queries on vertices: d_hat
    only -- the distance gradient is discontinuous there, and a closest point
    one rounding away from the query turns the term's gradient into an
    arbitrary unit vector on either side) and for masked (-708) terms."""
    O = oracle
    m = O.random_scene(seed, 300)
    q = O.QueryStream(3000 + seed).draw_points(m, 400)
    q = np.concatenate([q, m.vertices[:16]])  # distance 0 to some primitive
    w = O.Weights.build(m)
    t = O.Tree.build(m)
    e = engine_for(sd, O, m, w, 1, tree=t)
    worst_d = worst_g = 0.0
    for alpha, beta in ((10.0, 0.0), (100.0, 0.0), (900.0, 0.0), (100.0, 0.5)):
        p = O.Params(alpha=alpha, alpha_u=600.0, beta=beta)
        ref = O.query(m, w, q, p, tree=t if beta > 0 else None)
        sp = sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=beta)
        got = e.smooth_min_dist(q, sp) if beta > 0 else e.smooth_min_dist_flat(q, sp)
        fin = np.isfinite(ref.d_hat)
        assert (np.isfinite(got.d_hat) == fin).all()
        worst_d = max(worst_d, float((np.abs(got.d_hat[fin] - ref.d_hat[fin]) /
                                      np.maximum(1.0, np.abs(ref.d_hat[fin]))).max(initial=0.0)))
        gm = fin.copy()
        gm[-16:] = False
        worst_g = max(worst_g, float((np.linalg.norm(got.grad[gm] - ref.grad[gm], axis=1) /
                                      np.maximum(1.0, np.linalg.norm(ref.grad[gm], axis=1))).max(initial=0.0)))
    print(f"fp64 worst relative error: d_hat {worst_d:.3g}, grad {worst_g:.3g}")
    assert worst_d <= 1e-14 and worst_g <= 1e-13, (worst_d, worst_g)


@pytest.mark.parametrize("prec", [0, 1])
def test_host_chunk_pipeline_matches_unpipelined(sd, oracle, prec, monkeypatch):
    """sd_query_points' optional chunk pipeline (SDGPU_PIPELINE=1: four
    chunks, H2D / compute / D2H overlapped on two streams) returns exactly
    the unpipelined results for a ragged batch above its 2^17-query
    threshold, exact and BVH: decisions (counters, hash) identical, values
    within the parity tolerance (a chunk is a smaller batch, so the kernel
    choice and with it the summation order may differ)."""
    O = oracle
    m0 = O.random_scene(4, 300)
    rng = np.random.default_rng(17)
    lo, hi = m0.vertices.min(0), m0.vertices.max(0)
    q0 = rng.uniform(lo - 0.2, hi + 0.2, size=((1 << 17) + 4097, 3))
    m, q = prep(O, m0, q0, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    for mode, beta in ((sd.SD_EXACT, 0.0), (sd.SD_BVH, 0.5)):
        p = sd.SmoothParams(alpha=120.0, beta=beta)
        monkeypatch.delenv("SDGPU_PIPELINE", raising=False)
        a = e.query_points(q, p, mode, want_c=True, want_counters=True)
        monkeypatch.setenv("SDGPU_PIPELINE", "1")
        b = e.query_points(q, p, mode, want_c=True, want_counters=True)
        for f in ("leaves", "far_field", "decision_hash"):
            assert np.array_equal(getattr(a, f), getattr(b, f)), (mode, f)
        assert_close(b, a, prec, 120.0, f"pipeline mode {mode}")


@pytest.mark.parametrize("prec,beta", [(1, 0.0), (0, 0.0), (1, 0.5), (0, 0.5)])
def test_fused_evaluate_and_scatter_with_virtual_ranks(sd, oracle, prec, beta):
    """sd_query_points_scatter: the finalize epilogue stores every query's
    unshifted partials straight into its owner's buffer (4 virtual ranks, one
    GPU, a device pointer table as over NVLink). Bit-equal to the unfused
    query_points_device (c, grad_c) + scatter_partials, including an empty
    shard, exact and BVH; the owners' reduce matches the oracle."""
    import torch
    from paper_2108_10480_b200 import sharding
    O = oracle
    m0 = O.random_scene(12, 400)
    qs = O.QueryStream(62).draw_points(m0, 700)
    m, q = prep(O, m0, qs, prec)
    wt = O.Weights.build(m).table
    world = 4
    shards = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, wt.poly_index, world - 1)
    shards.append(None)  # rank 3 holds no primitives
    P = sd.SmoothParams(alpha=100.0, beta=beta)
    mode = sd.SD_BVH if beta > 0 else sd.SD_EXACT
    dev = torch.device("cuda", 0)
    n = len(q)
    per, counts = sharding.owner_blocks(n, world)
    fused = [torch.full((world * 4 * per,), np.nan, dtype=torch.float64, device=dev) for _ in range(world)]
    plain = [torch.full((world * 4 * per,), np.nan, dtype=torch.float64, device=dev) for _ in range(world)]
    tf = torch.tensor([b.data_ptr() for b in fused], dtype=torch.int64, device=dev)
    tp = torch.tensor([b.data_ptr() for b in plain], dtype=torch.int64, device=dev)
    qd = torch.tensor(q, dtype=torch.float64 if prec else torch.float32, device=dev)
    for r, s in enumerate(shards):
        e = sd.Engine(0, prec)
        if s is None:
            e.set_geometry(np.zeros((0, 3)), np.zeros((0, 3), np.int32), np.zeros(0, np.uint8))
            e.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, np.zeros(0, np.int32))
        else:
            e.set_geometry(s.vertices, s.simplices, s.kinds)
            e.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, s.poly_index)
            if beta > 0:
                e.build_bvh(sd.SD_BVH_MEDIAN)
        lf = torch.empty(n, dtype=torch.int64, device=dev)
        ff = torch.empty(n, dtype=torch.int64, device=dev)
        e.query_points_scatter(qd.data_ptr(), n, P, mode, tf.data_ptr(), world, r, per, lf.data_ptr(), ff.data_ptr())
        c = torch.empty(n, dtype=torch.float64, device=dev)
        g = torch.empty(n, 3, dtype=torch.float64, device=dev)
        d = torch.empty(n, dtype=torch.float64, device=dev)
        lp = torch.empty(n, dtype=torch.int64, device=dev)
        fp = torch.empty(n, dtype=torch.int64, device=dev)
        e.query_points_device(qd.data_ptr(), n, P, mode, d.data_ptr(), c_ptr=c.data_ptr(), grad_c_ptr=g.data_ptr(),
                              leaves_ptr=lp.data_ptr(), far_ptr=fp.data_ptr())
        e.scatter_partials(c.data_ptr(), g.data_ptr(), n, tp.data_ptr(), world, r, per)
        torch.cuda.synchronize()
        assert torch.equal(lf, lp) and torch.equal(ff, fp)
    for o in range(world):
        a = fused[o].view(world, 4, per)[:, :, :counts[o]]
        b = plain[o].view(world, 4, per)[:, :, :counts[o]]
        assert torch.equal(a, b), f"owner {o}"
    # owners finalise; the whole matches the oracle on the full mesh
    ref = O.query(m, O.Weights.from_table(wt), q, O.Params(alpha=100.0, beta=0.0))
    d_all = np.zeros(n)
    for o in range(world):
        dd = torch.empty(max(1, counts[o]), dtype=torch.float64, device=dev)
        e.reduce_owned(fused[o].data_ptr(), per, counts[o], world, P, dd.data_ptr(), None)
        torch.cuda.synchronize()
        d_all[o * per:o * per + counts[o]] = dd.cpu().numpy()[:counts[o]]
    if beta == 0.0:
        td = TOL[prec][0]
        fin = np.isfinite(ref.d_hat)
        assert (np.isfinite(d_all) == fin).all()
        assert (np.abs(d_all[fin] - ref.d_hat[fin]) <= td * np.maximum(1.0, np.abs(ref.d_hat[fin]))).all()
    else:  # Barnes-Hut per shard: conservative w.r.t. the exact whole-mesh field
        fin = np.isfinite(ref.d_hat)
        assert (d_all[fin] <= ref.d_hat[fin] + 1e-5 * np.maximum(1.0, np.abs(ref.d_hat[fin]))).all()


@pytest.mark.parametrize("prec", [0, 1])
def test_huge_query_coordinates_underflow_like_the_reference(sd, oracle, prec):
    """Queries so far away that |q - p|^2 overflows the compute type (fp32:
    beyond ~1.8e19) give c = 0, d_hat = +inf and a zero gradient, as the
    reference's -708 mask does for the huge distance; exact and BVH, with
    identical decisions; ordinary queries in the same batch are unaffected."""
    O = oracle
    m0 = O.random_scene(5, 200)
    qs = np.concatenate([O.QueryStream(55).draw_points(m0, 40),
                         [[1e20, 0.0, 0.0], [0.0, -1e30, 0.0], [3e19, 3e19, 3e19], [1e15, 2.0, -1e15]]])
    m, q = prep(O, m0, qs, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    for beta in (0.0, 0.5):
        p = O.Params(alpha=100.0, beta=beta)
        ref = O.query(m, w, q, p, tree=t if beta > 0 else None)
        got = e.smooth_min_dist(q, sd.SmoothParams(alpha=100.0, beta=beta)) if beta > 0 else \
            e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=100.0, beta=0.0))
        assert np.isinf(ref.d_hat[-4:]).all() and np.isinf(got.d_hat[-4:]).all()
        assert not got.grad[-4:].any() and not np.isnan(got.grad).any()
        assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
        assert_close(got, ref, prec, 100.0, f"huge coords beta {beta}")


@pytest.mark.parametrize("prec", [0, 1])
def test_nan_query_coordinates_propagate_like_the_reference(sd, oracle, prec):
    """A query with a NaN coordinate gives NaN d_hat and gradient, as the
    reference's exp(NaN) does (c = NaN skips the c <= 0 branch of
    result_from_accum, smooth.hpp:151-157); exact and BVH, device and host
    entry points; the other queries of the batch are unaffected."""
    O = oracle
    m0 = O.random_scene(6, 200)
    qs = np.concatenate([O.QueryStream(56).draw_points(m0, 40), [[np.nan, 0.0, 0.0], [0.1, 0.2, np.nan]]])
    m, q = prep(O, m0, qs, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    for beta in (0.0, 0.5):
        p = O.Params(alpha=100.0, beta=beta)
        ref = O.query(m, w, q[:-2], p, tree=t if beta > 0 else None)
        got = e.smooth_min_dist(q, sd.SmoothParams(alpha=100.0, beta=beta)) if beta > 0 else \
            e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=100.0, beta=0.0))
        assert np.isnan(got.d_hat[-2:]).all() and np.isnan(got.grad[-2:]).all()
        sub = type(got)(got.d_hat[:-2], got.grad[:-2])
        assert_close(sub, ref, prec, 100.0, f"nan batch beta {beta}")


@pytest.mark.parametrize("splits,cluster", [(1, "1"), (2, "1"), (3, "1"), (8, "1"), (12, "1"), (16, "1"), (17, "1"),
                                            (3, "0"), (8, "")])
@pytest.mark.parametrize("cfg,prec", [(2, 0), (2, 1), (3, 0)])
def test_exact_split_merge(sd, oracle, splits, cluster, cfg, prec, monkeypatch):
    """The exact kernel's primitive splits: 2..16 split CTAs of a query block
    form a thread-block cluster and merge their fp64 totals over distributed
    shared memory (only split 0 writes; the next segment launch continues
    from it -- cfg2 has three weight-polynomial segments); 17 splits and
    SDGPU_CLUSTER=0 (and "", the default) write every split's partial for
    the finalize kernel. Same results within the tolerance either way."""
    O = oracle
    monkeypatch.setenv("SDGPU_EXACT_SPLITS", str(splits))
    monkeypatch.setenv("SDGPU_CLUSTER", cluster)
    m, q = _cfg(O, cfg, 700 if cfg == 2 else 300, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    ref = O.query(m, w, q, O.Params(alpha=100.0, beta=0.0))
    got = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=100.0, beta=0.0))
    assert_close(got, ref, prec, 100.0, f"cfg{cfg} splits {splits} cluster {cluster}")


@pytest.mark.parametrize("prec", [0, 1])
def test_pipelined_host_batches_equal_blocking_calls(sd, oracle, prec):
    """sd_query_points_async: five batches of different sizes submitted back
    to back (two in flight, a third submission waits for the oldest), exact
    and tree mode alternating, results bit-equal to the blocking
    sd_query_points calls; wait(ticket) and wait() semantics."""
    O = oracle
    m0 = O.random_scene(9, 300)
    m, _ = prep(O, m0, np.zeros((1, 3)), prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    P = sd.SmoothParams(alpha=120.0, beta=0.4)
    batches = []
    for k, n in enumerate((700, 33, 2048, 1, 517)):
        q = O.QueryStream(900 + k).draw_points(m0, n)
        if prec == 0:
            q = q.astype(np.float32).astype(np.float64)
        batches.append((np.ascontiguousarray(q), sd.SD_BVH if k % 2 else sd.SD_EXACT))
    outs = [sd.SmoothResults(np.empty(len(q)), np.empty((len(q), 3))) for q, _ in batches]
    tickets = [e.query_points_async(q, P, mode, outs[k]) for k, (q, mode) in enumerate(batches)]
    assert tickets == sorted(tickets) and len(set(tickets)) == len(tickets)
    e.wait(tickets[-1])
    e.wait()
    for (q, mode), got in zip(batches, outs):
        ref = e.query_points(q, P, mode)
        assert np.array_equal(got.d_hat, ref.d_hat) and np.array_equal(got.grad, ref.grad)


@pytest.mark.parametrize("prec,chunk", [(0, "1"), (1, "1"), (0, "4"), (0, "")])
def test_query_sharded_tree_walk_equals_the_whole_batch(sd, oracle, prec, chunk, monkeypatch):
    """sd_query_points_device_shard: ranks 0..world-1 each walk the
    interleaved packets r, r + world, ... of the whole sorted batch and write
    only their queries' outputs; together they reproduce the single walk of
    the batch bit for bit (same packets, same per-lane work), entries of
    other ranks are left untouched, decision hashes equal the oracle's."""
    import torch
    O = oracle
    monkeypatch.setenv("SDGPU_FRONTIER", "0")
    monkeypatch.setenv("SDGPU_SPLIT", "0")
    monkeypatch.setenv("SDGPU_SHARD_CHUNK", chunk)  # packets per round-robin chunk ("" = the default 64)
    m0 = O.random_scene(12, 400)
    qs = O.QueryStream(1212).draw_points(m0, 3000)  # 94 packets, the last one ragged
    m, q = prep(O, m0, qs, prec)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = engine_for(sd, O, m, w, prec, tree=t)
    P = sd.SmoothParams(alpha=150.0, beta=0.5)
    whole = e.smooth_min_dist(q, P)
    dev = torch.device("cuda", 0)
    Q = len(q)
    qd = torch.tensor(q, dtype=torch.float64 if prec else torch.float32, device=dev)
    world = 3
    d = torch.full((Q,), float("nan"), dtype=torch.float64, device=dev)
    g = torch.full((Q, 3), float("nan"), dtype=torch.float64, device=dev)
    hs = torch.zeros(Q, dtype=torch.int64, device=dev)
    written = []
    for r in range(world):
        before = d.clone()
        e.query_points_device_shard(qd.data_ptr(), Q, P, world, r, d.data_ptr(), g.data_ptr(),
                                    hash_ptr=hs.data_ptr())
        torch.cuda.synchronize()
        now = ~torch.isnan(d) & torch.isnan(before)
        written.append(now.cpu().numpy())
    cover = np.sum(written, axis=0)
    assert (cover == 1).all()  # every query by exactly one rank
    if chunk == "1":
        assert 0.25 < written[0].mean() < 0.42
    assert np.array_equal(d.cpu().numpy(), whole.d_hat) and np.array_equal(g.cpu().numpy(), whole.grad)
    ref = O.query(m, w, q, O.Params(alpha=150.0, beta=0.5), tree=t)
    assert (hs.cpu().numpy().view(np.uint64) == ref.decision_hash).all()


# ------------------------------------------------- pruned exact evaluation
def _prune_bound(n_prims, bits):
    """Relative bound on c of sd_set_exact_pruning (include/sdgpu.h)."""
    return n_prims * 2.0 ** -bits


@pytest.mark.parametrize("prec,bits", [(0, 48.0), (0, 32.0), (1, 64.0)])
@pytest.mark.parametrize("seed", [1, 4, 7, 10])
def test_pruned_exact_on_random_scenes(sd, oracle, prec, bits, seed):
    """sd_set_exact_pruning on mixed point / edge / triangle scenes: oracle
    parity at the unpruned tolerances, and the documented bound against
    the engine's own all-pairs sum (c, grad_c compared directly)."""
    O = oracle
    m0 = O.random_scene(seed, 400)
    qs = O.QueryStream(2000 + seed).draw_points(m0, 700)
    m, q = prep(O, m0, qs, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    for alpha in (100.0, 900.0, 20.0):
        P = sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=0.0)
        e.set_exact_pruning(0.0)
        full = e.query_points(q, P, sd.SD_EXACT, want_c=True)
        e.set_exact_pruning(bits)
        got = e.query_points(q, P, sd.SD_EXACT, want_c=True)
        ref = O.query(m, w, q, O.Params(alpha=alpha, alpha_u=600.0, beta=0.0))
        assert_close(got, ref, prec, alpha, f"pruned seed {seed} alpha {alpha}")
        assert (np.isfinite(got.d_hat) == np.isfinite(full.d_hat)).all()
        pos = full.c > 0
        rel = np.abs(got.c[pos] - full.c[pos]) / full.c[pos]
        # the fp32 tile sums regroup when tiles drop out: allow their rounding
        slack = 5e-6 if prec == 0 else 1e-13
        assert rel.max() <= _prune_bound(m.num_simplices, bits) + slack, rel.max()
        assert (got.c[pos] <= full.c[pos] * (1 + slack)).all()  # pruning only removes positive terms
    e.set_exact_pruning(0.0)
    again = e.query_points(q, P, sd.SD_EXACT, want_c=True)
    assert np.array_equal(again.d_hat, full.d_hat) and np.array_equal(again.grad, full.grad)


def test_pruned_exact_config3_subset(sd, oracle):
    """cfg3 (262,144 triangles), 4,096 queries, alpha in {10, 100, 1000}:
    pruned at 48 bits against the oracle and against the all-pairs kernel."""
    O = oracle
    m, q = _cfg(O, 3, 4096, 0)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, 0)
    idx = np.arange(0, len(q), 16)
    for alpha in (10.0, 100.0, 1000.0):
        P = sd.SmoothParams(alpha=alpha, beta=0.0)
        e.set_exact_pruning(0.0)
        full = e.query_points(q, P, sd.SD_EXACT)
        e.set_exact_pruning(48.0)
        got = e.query_points(q, P, sd.SD_EXACT)
        fin = np.isfinite(full.d_hat)
        assert (np.isfinite(got.d_hat) == fin).all()
        assert np.abs(got.d_hat[fin] - full.d_hat[fin]).max() <= 2e-6 / alpha + 1e-7
        assert np.abs(got.grad[fin] - full.grad[fin]).max() <= 1e-5
        ref = O.query(m, w, q[idx], O.Params(alpha=alpha, beta=0.0))
        assert_close(type(got)(got.d_hat[idx], got.grad[idx]), ref, 0, alpha, f"pruned cfg3 alpha {alpha}")


def test_pruning_threshold_is_validated(sd, oracle):
    O = oracle
    m = O.random_scene(3, 50)
    e = engine_for(sd, O, m, O.Weights.build(m), 0)
    for bad in (-1.0, 8.0, float("nan"), float("inf")):
        with pytest.raises(sd.SdError):
            e.set_exact_pruning(bad)
    e.set_exact_pruning(24.0)
    e.set_exact_pruning(0.0)


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("side", [1.0, -1.0])
def test_far_tile_first_then_near_tiles(sd, oracle, prec, side, monkeypatch):
    """A far cluster (alpha d = 700, just inside the -708 mask) summed before
    a nearer one (alpha d = 530) by the same CTA: the totals stay anchored at
    the far tile's shift (below 2^-1074), and the de-shift in K4 must still
    return c ~ 600 e^-530 instead of 0 (found on cfg5: d_hat = +inf for
    queries ~5.3 from the nearest primitive)."""
    O = oracle
    rng = np.random.default_rng(5)
    far = np.array([3.0, 0.0, 0.0]) + 0.005 * rng.standard_normal((1024, 3))
    near = np.array([4.7, 0.0, 0.0]) + 0.005 * rng.standard_normal((600, 3))
    v = side * np.concatenate([far, near])
    n = len(v)
    simp = np.stack([np.arange(n), np.full(n, -1), np.full(n, -1)], axis=1).astype(np.int32)
    m0 = O.Mesh.from_arrays(v, simp, np.zeros(n, np.uint8))
    qs = side * (np.array([10.0, 0.0, 0.0]) + 0.01 * rng.standard_normal((70, 3)))
    m, q = prep(O, m0, qs, prec)
    w = O.Weights.build(m)
    e = engine_for(sd, O, m, w, prec)
    P = sd.SmoothParams(alpha=100.0, beta=0.0)
    ref = O.query(m, w, q, O.Params(alpha=100.0, beta=0.0))
    assert np.isfinite(ref.d_hat).all() and (ref.c < 1e-200).all()
    for splits in ("1", "2", ""):
        if splits:
            monkeypatch.setenv("SDGPU_EXACT_SPLITS", splits)
        else:
            monkeypatch.delenv("SDGPU_EXACT_SPLITS", raising=False)
        got = e.query_points(q, P, sd.SD_EXACT, want_c=True)
        assert_close(got, ref, prec, 100.0, f"far tile first, splits {splits!r}")
        assert np.abs(got.c / ref.c - 1).max() < (1e-3 if prec == 0 else 1e-9)
