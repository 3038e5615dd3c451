"""The oracle restatement pinned against the REFERENCE ITSELF: the unmodified
reference headers compiled into oracle/_ref/libsdref.so (oracle/Makefile
`ref`, Eigen-subset shim oracle/eigen_shim). Both sides run on the same
inputs and the same WeightSet table; the restatement must agree BIT FOR BIT
(d_hat, grad, c, grad_c, leaf / far-field counts, trees) on random mixed
scenes, query simplices, and subsets of every BASELINE config.

Skipped when the library is absent (it is built where /root/reference
exists: here, by __graft_entry__.build(); it travels to the GPU box)."""
import numpy as np
import pytest

import oracle as O
from oracle import reference as R

pytestmark = pytest.mark.skipif(not R.available() and R.build() is None,
                                reason="oracle/_ref not built (reference headers absent)")


def same(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b), equal_nan=True)


def check_point_queries(m, w, q, params, tree=None, scene=None):
    sc = scene or R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    if tree is not None and scene is None:
        sc.set_bvh(tree.nodes())
    a = O.query(m, w, q, params, tree=tree)
    b = sc.query(q, params, tree=tree is not None)
    for f in ("d_hat", "grad", "c", "grad_c", "leaves", "far_field"):
        assert same(getattr(a, f), getattr(b, f)), f
    return a


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 7, 8])
def test_random_scenes_bit_identical(seed):
    """Mixed point / edge / triangle scenes, exact and Barnes-Hut, several
    (alpha, alpha_u, beta): the restatement is the reference, bit for bit;
    the reference's own build_bvh gives the oracle's tree byte for byte."""
    m = O.random_scene(seed, 300)
    w = O.Weights.build(m)
    t = O.Tree.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    sc.set_bvh(None)  # the reference's build_bvh
    assert sc.bvh().tobytes() == t.nodes().tobytes()
    q = O.QueryStream(700 + seed).draw_points(m, 300)
    for alpha, alpha_u, beta in ((100.0, 600.0, 0.0), (100.0, 600.0, 0.5), (20.0, 600.0, 0.2), (900.0, 600.0, 0.9),
                                 (400.0, 1200.0, 0.5)):
        p = O.Params(alpha=alpha, alpha_u=alpha_u, beta=beta)
        check_point_queries(m, w, q, p, tree=t if beta > 0 else None, scene=sc)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_query_simplices_bit_identical(seed):
    """Edge / triangle / point QUERY simplices (smooth_min_dist with a
    SimplexGeom, the face-enumeration QP and the halfspace box test)."""
    m = O.random_scene(seed, 200)
    w = O.Weights.build(m)
    t = O.Tree.build(m)
    c, d = O.random_queries(seed + 50, m, 120)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    sc.set_bvh(t.nodes())
    for beta in (0.0, 0.5):
        p = O.Params(alpha=100.0, beta=beta)
        a = O.query_simplices(m, w, c, d, p, tree=t if beta > 0 else None)
        b = sc.query(np.asarray(c).reshape(-1, 9), p, tree=beta > 0, dims=d)
        for f in ("d_hat", "grad", "leaves", "far_field"):
            assert same(getattr(a, f), getattr(b, f)), (f, beta)


def test_underflow_and_known_answers_through_the_reference():
    """FarQueryUnderflowsToInfinity (test_smooth.cpp:201-219) and the
    single-point closed form, run through the compiled reference."""
    m = O.point_cluster(20, 2, 0.05)
    w = O.Weights.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    r = sc.query([[3.0, 0.0, 0.0]], O.Params(alpha=400.0, beta=0.0))
    assert r.c[0] == 0.0 and np.isinf(r.d_hat[0]) and not r.grad.any()
    m1 = O.Mesh.from_arrays([[0, 0, 0]], [[0, -1, -1]], [0])
    sc1 = R.Scene(m1.vertices, m1.simplices, m1.kinds, O.Weights.build(m1).table)
    q = np.array([[0.3, -0.2, 0.6]])
    r = sc1.query(q, O.Params(alpha=50.0, beta=0.0))
    assert abs(r.d_hat[0] - np.linalg.norm(q)) < 1e-12


@pytest.mark.parametrize("cfg", [1, 2])
def test_edge_and_point_weight_sets_match_the_reference_build(cfg):
    """For meshes without triangles the reference's whole build_weight_set
    runs (closed-form edge polynomials, weights.hpp:46-76, 589-621): the
    oracle's table is identical (A, sup, coefficients, assignment)."""
    m = O.config_mesh(cfg)
    w = O.Weights.build(m).table
    val, A, sup, ea, pi = R.build_weights_no_tris(m.vertices, m.simplices, m.kinds)
    assert A == w.A and sup == w.sup_wtilde
    assert same(ea, w.edge_a) and same(pi, w.poly_index)


@pytest.mark.parametrize("cfg,nq,alphas", [(1, 512, (50.0,)), (2, 128, (100.0,)), (3, 16, (10.0, 100.0, 1000.0))])
def test_exact_config_subsets_bit_identical(cfg, nq, alphas):
    """BASELINE configs[0..2] on query subsets, exact LSE
    (smooth_min_dist_flat, smooth.hpp:189-198)."""
    m = O.config_mesh(cfg)
    if cfg != 1:
        m = m.quantized()
    q = O.config_queries(cfg, m, nq)
    w = O.Weights.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    for alpha in alphas:
        check_point_queries(m, w, q, O.Params(alpha=alpha, beta=0.0), scene=sc)


def test_cfg3_reference_tree_equals_oracle_tree():
    """build_bvh (bvh.hpp:34-91) on the 262,144-triangle torus: the
    reference's tree and the restatement's are byte-identical."""
    m = O.config_mesh(3).quantized()
    w = O.Weights.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    sc.set_bvh(None)
    assert sc.bvh().tobytes() == O.Tree.build(m).nodes().tobytes()


def test_cfg4_bvh_subset_bit_identical():
    """BASELINE configs[3] (5,242,880 triangles, alpha 200, beta 0.5): 512
    queries from both halves of the distribution on the oracle's tree, plus
    4 exact queries; the tree is the reference's (checked on cfg3 above
    and on the random scenes)."""
    m = O.config_mesh(4).quantized()
    qa = O.config_queries(4, m, 1 << 14)
    q = np.concatenate([qa[:256], qa[8192:8192 + 256]])
    w = O.Weights.build(m)
    t = O.Tree.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    sc.set_bvh(t.nodes())
    check_point_queries(m, w, q, O.Params(alpha=200.0, beta=0.5), tree=t, scene=sc)
    check_point_queries(m, w, q[::128], O.Params(alpha=200.0, beta=0.0), scene=sc)


def test_cfg5_subset_bit_identical():
    """BASELINE configs[4] (16.8M triangles + 1M edges + 1M points, alpha
    100): 4 exact queries over all 18.8M primitives and 64 Barnes-Hut
    queries on the oracle's tree."""
    m = O.config_mesh(5).quantized()
    q = O.config_queries(5, m, 4096)
    w = O.Weights.build(m)
    sc = R.Scene(m.vertices, m.simplices, m.kinds, w.table)
    check_point_queries(m, w, q[::1024], O.Params(alpha=100.0, beta=0.0), scene=sc)
    t = O.Tree.build(m)
    sc.set_bvh(t.nodes())
    check_point_queries(m, w, q[::64], O.Params(alpha=100.0, beta=0.5), tree=t, scene=sc)
