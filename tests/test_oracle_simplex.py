"""CPU oracle for SIMPLEX queries (edge / triangle query primitives, SURVEY
8(f) rank 2), pinned against the reference's own tests for that path:
T/test_exact.cpp (simplex_distance, the face-enumeration QP),
T/test_bvh.cpp:96-166 (box_primitive_proximity) and T/test_smooth.cpp
(smooth_min_dist / smooth_mesh_dist with random_query draws of all kinds).
"""
import math

import numpy as np
import pytest


def _pairs(O, seed, n):
    """n (f, g) pairs of random_query simplices over [-1,1]^3 with size 0.6
    (test_exact.cpp:19-24); corners (3,3), dims."""
    box = O.Mesh.from_arrays([[-1, -1, -1], [1, 1, 1]], [[0, -1, -1], [1, -1, -1]], [0, 0])
    c, d = O.random_queries_scaled(seed, box, 2 * n, 0.6)
    return [((c[2 * i], d[2 * i]), (c[2 * i + 1], d[2 * i + 1])) for i in range(n)]


def _sd(O, f, g, qp=False):
    return O.simplex_distance(f[0][: f[1] + 1], f[1], g[0][: g[1] + 1], g[1], qp=qp)


def _shift(g, v):
    c = g[0].copy()
    c[: g[1] + 1] += v
    return (c, g[1])


# ---------------------------------------------------------- test_exact.cpp
def test_parallel_edges_resolve_deterministically(oracle):  # :220-230
    O = oracle
    r = O.simplex_distance([0, 0, 0, 1, 0, 0], 1, [0, 1, 0, 1, 1, 0], 1)
    assert r.distance == 1.0 and r.phi[0] == 0.0 and r.lam[0] == 0.0
    assert O.simplex_distance([0, 0, 0, 1, 0, 0], 1, [1, 1, 0, 0, 1, 0], 1).distance == 1.0


def test_contact_and_overlap(oracle):  # :232-250
    O = oracle
    tri = [0, 0, 0, 2, 0, 0, 0, 2, 0]
    on = O.simplex_distance(tri, 2, [0.5, 0.5, 0], 0)
    assert on.distance == 0.0 and not on.grad.any()
    assert abs(O.simplex_distance(tri, 2, [0.5, 0.5, -1, 0.5, 0.5, 1], 1).distance) <= 1e-12
    e = [0, 0, 0, 1, 2, 3]
    s = O.simplex_distance(e, 1, e, 1)
    assert s.distance == 0.0 and not s.grad.any()


def test_coplanar_parallel_triangle_pair(oracle):  # :252-260
    O = oracle
    r = O.simplex_distance([0, 0, 0, 1, 0, 0, 0, 1, 0], 2, [0, 0, 0.5, 1, 0, 0.5, 0, 1, 0.5], 2)
    assert abs(r.distance - 0.5) <= 1e-12 and abs(abs(r.grad[2]) - 1.0) <= 1e-12


def test_symmetry_under_argument_swap(oracle):  # :114-123
    O = oracle
    for f, g in _pairs(O, 101, 300):
        a, b = _sd(O, f, g).distance, _sd(O, g, f).distance
        assert abs(a - b) <= 1e-6 * (1 + a)


def test_qp_matches_closed_forms(oracle):  # :125-138
    O = oracle
    used = 0
    for f, g in _pairs(O, 202, 500):
        if f[1] == 2 and g[1] == 2:
            continue
        closed, qp = _sd(O, f, g).distance, _sd(O, f, g, qp=True).distance
        assert abs(qp - closed) <= 1e-6 * (1 + closed)
        used += 1
    assert used > 300


def test_gradient_matches_central_difference(oracle):  # :140-161
    O = oracle
    h, used = 1e-6, 0
    for f, g in _pairs(O, 303, 400):
        r = _sd(O, f, g)
        if r.distance < 1e-3:
            continue
        for a in range(3):
            e = np.zeros(3)
            e[a] = h
            fd = (_sd(O, f, _shift(g, e)).distance - _sd(O, f, _shift(g, -e)).distance) / (2 * h)
            assert abs(fd - r.grad[a]) <= 1e-4 * max(1.0, abs(r.grad[a]))
        used += 1
    assert used > 250


def _at(c, dim, b):
    c = np.asarray(c, np.float64).reshape(3, 3)
    if dim == 0:
        return c[0]
    if dim == 1:
        return c[0] + b[0] * (c[1] - c[0])
    return c[0] + b[0] * (c[1] - c[0]) + b[1] * (c[2] - c[0])


def test_closest_points_are_consistent(oracle):  # :163-179
    O = oracle
    for f, g in _pairs(O, 404, 300):
        r = _sd(O, f, g)
        assert abs(np.linalg.norm(r.point_g - r.point_f) - r.distance) <= 1e-12 * (1 + r.distance)
        assert np.linalg.norm(_at(f[0], f[1], r.phi) - r.point_f) <= 1e-12
        assert np.linalg.norm(_at(g[0], g[1], r.lam) - r.point_g) <= 1e-12
        if r.distance > 0:
            assert np.linalg.norm(r.grad * r.distance - (r.point_g - r.point_f)) <= 1e-9 * (1 + r.distance)
        else:
            assert not r.grad.any()


def _point_to(O, f, pts):
    return np.array([O.simplex_distance(f[0][: f[1] + 1], f[1], p, 0).distance for p in pts])


def test_edge_triangle_against_dense_sampling(oracle):  # :181-203
    O = oracle
    tri = (np.array([[0, 0, 0], [1, 0, 0], [0.2, 0.9, 0.1]], float), 2)
    a, b = np.array([-0.4, 0.5, 0.8]), np.array([1.3, -0.2, 0.4])
    exact = O.simplex_distance(tri[0], 2, np.concatenate([a, b]), 1).distance
    n = 20000  # grid overshoot <= |b - a| / (2 n) < 5e-5
    t = np.linspace(0, 1, n + 1)[:, None]
    sampled = _point_to(O, tri, a + t * (b - a)).min()
    assert exact <= sampled + 1e-12 and abs(exact - sampled) <= 1e-4


def test_triangle_triangle_against_convex_refinement(oracle):  # :205-218
    """Coarse barycentric grid on g, then compass refinement of the convex
    objective x -> d(x, f) (the reference's refined_triangle_distance)."""
    O = oracle
    used = 0
    for f, g in _pairs(O, 606, 200):
        if f[1] != 2 or g[1] != 2:
            continue
        N = 64
        grid = [(i / N, j / N) for i in range(N + 1) for j in range(N + 1 - i)]
        pts = np.array([_at(g[0], 2, uv) for uv in grid])
        d = _point_to(O, f, pts)
        k = int(np.argmin(d))
        best, (bu, bv) = d[k], grid[k]
        step = 1.0 / N
        while step > 1e-12:
            moved = False
            for cu, cv in ((bu + step, bv), (bu - step, bv), (bu, bv + step), (bu, bv - step)):
                if cu < 0 or cv < 0 or cu + cv > 1:
                    continue
                dd = _point_to(O, f, [_at(g[0], 2, (cu, cv))])[0]
                if dd < best:
                    best, bu, bv, moved = dd, cu, cv, True
            if not moved:
                step *= 0.5
        exact = _sd(O, f, g).distance
        assert exact <= best + 1e-9 and abs(exact - best) <= 1e-6 * (1 + exact)
        used += 1
        if used == 6:
            break
    assert used == 6


# ------------------------------------------------------------ test_bvh.cpp
def test_box_separating_halfspace_cases(oracle):  # :96-125
    O = oracle
    lo, hi = [0, 0, 0], [1, 1, 1]
    d, y, _, md = O.box_primitive_proximity(lo, hi, [2, 2, 2, 3, 2, 2], 1)
    assert not md and abs(d - math.sqrt(3)) <= 1e-12 and np.linalg.norm(y - 1) <= 1e-12
    d, _, _, md = O.box_primitive_proximity(lo, hi, [2, 2, 0.2, 2, 2, 0.8], 1)
    assert not md and abs(d - math.sqrt(2)) <= 1e-12
    d, _, _, md = O.box_primitive_proximity(lo, hi, [2, 0.2, 0.2, 2, 0.8, 0.8], 1)
    assert not md and abs(d - 1.0) <= 1e-12
    d, _, _, md = O.box_primitive_proximity(lo, hi, [-1, 0.5, 0.5, 2, 0.5, 0.5], 1)
    assert md and d == 0.0


def test_box_matches_point_overload(oracle):  # :127-142
    O = oracle
    lo, hi = np.array([-1.0, 0, 2]), np.array([1.0, 1, 3])
    rng = np.random.default_rng(7)
    q = rng.uniform(-3, 5, (100, 3))
    d0, y0 = O.box_point_proximity(lo, hi, q)
    for i in range(100):
        d, y, _, md = O.box_primitive_proximity(lo, hi, q[i], 0)
        assert d == d0[i] and (y == y0[i]).all() and not md


def _subtree_prims(nodes, i):
    out, st = [], [i]
    while st:
        k = st.pop()
        if nodes["left"][k] < 0:
            out.append(int(nodes["primitive"][k]))
        else:
            st += [int(nodes["left"][k]), int(nodes["right"][k])]
    return out


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_box_never_exceeds_contained_primitive_distance(oracle, seed):  # :144-166
    O = oracle
    m = O.random_scene(seed, 200)
    nodes = O.Tree.build(m).nodes()
    c, d = O.random_queries(23 + seed, m, 10)
    V, S, K = m.vertices, m.simplices, m.kinds
    for q in range(10):
        g = (c[q], int(d[q]))
        pd = np.array([O.simplex_distance(V[S[p, : K[p] + 1]], int(K[p]), g[0][: g[1] + 1], g[1]).distance
                       for p in range(len(K))])
        for i in range(len(nodes)):
            dist, _, _, _ = O.box_primitive_proximity(nodes["lo"][i], nodes["hi"][i], g[0][: g[1] + 1], g[1])
            assert dist <= pd[_subtree_prims(nodes, i)].min() + 1e-12


# --------------------------------------------------------- test_smooth.cpp
def _exact_min(O, m, c, d):
    V, S, K = m.vertices, m.simplices, m.kinds
    return np.array([min(O.simplex_distance(V[S[p, : K[p] + 1]], int(K[p]), c[i][: d[i] + 1], int(d[i])).distance
                         for p in range(len(K))) for i in range(len(d))])


@pytest.mark.parametrize("seed", [1, 4, 7, 10])
def test_conservative_and_beta_monotone_simplex_queries(oracle, seed):  # :92-120
    O = oracle
    m = O.random_scene(seed, 120)
    w, t = O.Weights.build(m), O.Tree.build(m)
    c, d = O.random_queries(99 + seed, m, 20)
    base = O.Params(alpha=100.0, alpha_u=600.0, beta=0.0)
    slack = math.log(w.max_attenuated_weight(base) * m.num_simplices) / base.alpha
    dmin = _exact_min(O, m, c, d)
    r0 = O.query_simplices(m, w, c, d, base, tree=t)
    assert (r0.leaves == m.num_simplices).all()
    assert (r0.d_hat <= dmin + 1e-9).all() and (r0.d_hat >= dmin - slack - 1e-9).all()
    for beta in (0.3, 0.8):
        rb = O.query_simplices(m, w, c, d, O.Params(alpha=100.0, alpha_u=600.0, beta=beta), tree=t)
        assert (rb.d_hat <= r0.d_hat + 1e-9).all()


@pytest.mark.parametrize("seed", [6, 7])
def test_flat_matches_tree_simplex_queries(oracle, seed):  # :221-241
    O = oracle
    m = O.random_scene(seed, 100)
    w, t = O.Weights.build(m), O.Tree.build(m)
    c, d = O.random_queries(31, m, 30)
    p = O.Params(beta=0.0)
    a, b = O.query_simplices(m, w, c, d, p, tree=t), O.query_simplices(m, w, c, d, p)
    assert (a.leaves == b.leaves).all()
    fin = np.isfinite(b.d_hat)
    assert (np.isfinite(a.d_hat) == fin).all()
    assert (np.abs(a.d_hat[fin] - b.d_hat[fin]) <= 1e-10 * np.maximum(1, np.abs(b.d_hat[fin]))).all()
    assert (np.linalg.norm(a.grad - b.grad, axis=1) <= 1e-10 * np.maximum(1, np.linalg.norm(b.grad, axis=1))).all()


def test_simplex_gradient_matches_central_difference(oracle):  # :143-175
    """Translation gradient of d_hat for edge / triangle queries (unit
    weights; see test_oracle_golden.test_gradient_matches_central_difference
    for why built weights use the reference's alpha-scaled weight term)."""
    O = oracle
    p = O.Params(alpha=100.0, alpha_u=600.0, beta=0.0)
    h, used = 1e-5, 0
    for seed in (2, 3, 4):
        m = O.random_scene(seed, 80)
        w = O.Weights.unit(m)
        c, d = O.random_queries(12 + seed, m, 40)
        keep = d > 0
        c, d = c[keep], d[keep]
        r = O.query_simplices(m, w, c, d, p)
        ok = np.isfinite(r.d_hat) & (r.d_hat > 1e-2) & (r.d_hat < 3.0)
        for i in np.nonzero(ok)[0]:
            fd = np.zeros(3)
            for a in range(3):
                e = np.zeros(3)
                e[a] = h
                cp, cm = c[i].copy(), c[i].copy()
                cp[: d[i] + 1] += e
                cm[: d[i] + 1] -= e
                dp = O.query_simplices(m, w, cp[None], d[i:i + 1], p).d_hat[0]
                dm = O.query_simplices(m, w, cm[None], d[i:i + 1], p).d_hat[0]
                fd[a] = (dp - dm) / (2 * h)
            assert np.linalg.norm(fd - r.grad[i]) <= 1e-4 * max(1.0, np.linalg.norm(r.grad[i])), (seed, i)
            used += 1
    assert used >= 20


def test_simplex_translation_invariance(oracle):  # :177-199
    O = oracle
    m = O.random_scene(13, 60)
    shift = np.array([0.37, -1.2, 0.55])
    m2 = O.Mesh.from_arrays(m.vertices + shift, m.simplices, m.kinds)
    w, w2 = O.Weights.build(m), O.Weights.build(m2)
    c, d = O.random_queries(21, m, 30)
    c2 = c.copy()
    for i in range(len(d)):
        c2[i, : d[i] + 1] += shift
    p = O.Params(beta=0.0)
    a, b = O.query_simplices(m, w, c, d, p), O.query_simplices(m2, w2, c2, d, p)
    # a query simplex INTERSECTING a primitive (d_min ~ 1e-16) has a whole
    # segment of closest pairs; the QP's first-strictly-best tie-break then
    # depends on rounding, and so does the weight at phi -- the reference's
    # own algorithm, not restatement noise. Those queries are excluded.
    fin = np.isfinite(a.d_hat) & (_exact_min(O, m, c, d) > 1e-9)
    assert np.isfinite(b.d_hat[fin]).all() and fin.sum() >= 20
    assert (np.abs(a.d_hat[fin] - b.d_hat[fin]) <= 1e-9 * np.maximum(1, np.abs(a.d_hat[fin]))).all()


def test_points_through_simplex_path_are_bit_identical(oracle):
    """A point query through the simplex path is the point path exactly
    (exact.hpp:344, bvh.hpp:122)."""
    O = oracle
    m = O.random_scene(5, 150)
    w, t = O.Weights.build(m), O.Tree.build(m)
    q = O.random_point_queries(8, m, 200)
    c = np.zeros((len(q), 3, 3))
    c[:, 0] = q
    for beta in (0.0, 0.5):
        p = O.Params(beta=beta)
        a = O.query(m, w, q, p, tree=t)
        b = O.query_simplices(m, w, c, np.zeros(len(q), np.int32), p, tree=t)
        assert (a.d_hat == b.d_hat).all() and (a.grad == b.grad).all()
        assert (a.decision_hash == b.decision_hash).all()


def test_mesh_dist_rigid_translation_consistency(oracle):  # test_smooth.cpp:332-356
    O = oracle
    f = O.icosphere(0)
    # unit weights: the reference's alpha-scaled weight-gradient term
    # (weights.hpp:668-697) is not the derivative of d_hat by design
    w, t = O.Weights.unit(f), O.Tree.build(f)
    q0 = O.random_scene(11, 30)
    assert (q0.kinds > 0).any()
    qv = q0.vertices + np.array([2.5, 0, 0])
    p = O.Params(beta=0.0)
    md = O.mesh_dist(f, w, O.Mesh.from_arrays(qv, q0.simplices, q0.kinds), p, tree=t)
    assert math.isfinite(md.d_hat)
    total = md.vertex_grads.sum(axis=0)
    h = 1e-5
    for a in range(3):
        e = np.zeros(3)
        e[a] = h
        dp = O.mesh_dist(f, w, O.Mesh.from_arrays(qv + e, q0.simplices, q0.kinds), p, tree=t).d_hat
        dm = O.mesh_dist(f, w, O.Mesh.from_arrays(qv - e, q0.simplices, q0.kinds), p, tree=t).d_hat
        assert abs(total[a] - (dp - dm) / (2 * h)) <= 1e-4 * max(1.0, abs(total[a]))


def test_mesh_dist_softmin_identity_and_bounds(oracle):  # test_smooth.cpp:282-300
    O = oracle
    f = O.icosphere(1)
    w, t = O.Weights.build(f), O.Tree.build(f)
    q0 = O.random_scene(42, 40)
    q = O.Mesh.from_arrays(q0.vertices + np.array([2.5, 0, 0]), q0.simplices, q0.kinds)
    p = O.Params(beta=0.0, alpha_q=120.0)
    md = O.mesh_dist(f, w, q, p, tree=t)
    assert math.isfinite(md.d_hat)
    mass = np.exp(-p.alpha_q * (md.per_primitive - md.d_hat)).sum()
    dmin = md.per_primitive.min()
    assert abs(mass - 1.0) <= 1e-9
    assert dmin - math.log(q.num_simplices) / p.alpha_q - 1e-9 <= md.d_hat <= dmin + 1e-12


# ------------------------------------------------- reference caches (CPU)
def test_oracle_cache_round_trips(oracle, tmp_path):
    """SDBV0001 / SDWT0001 (bvh.hpp:190-236, weights.hpp:700-781): save ->
    load -> save is byte-identical, and the loaded tree / table equal the
    originals."""
    O = oracle
    m = O.random_scene(4, 150)
    t, w = O.Tree.build(m), O.Weights.build(m)
    pb, pw = str(tmp_path / "t.sdbv"), str(tmp_path / "w.sdwt")
    O.save_bvh_cache(t, pb)
    t2 = O.load_bvh_cache(pb)
    assert t2.nodes().tobytes() == t.nodes().tobytes()
    O.save_bvh_cache(t2, pb + "2")
    assert open(pb, "rb").read() == open(pb + "2", "rb").read()
    raw = open(pb, "rb").read()
    assert raw[:8] == b"SDBV0001" and len(raw) == 16 + 72 * len(t.nodes())
    O.save_weight_cache(w, pw)
    w2 = O.load_weight_cache(pw)
    O.save_weight_cache(w2, pw + "2")
    assert open(pw, "rb").read() == open(pw + "2", "rb").read()
    a, b = w.table, w2.table
    assert a.A == b.A and a.sup_wtilde == b.sup_wtilde
    assert (a.edge_a == b.edge_a).all() and (a.tri_stored == b.tri_stored).all()
    assert (a.poly_index == b.poly_index).all()
    with pytest.raises(RuntimeError):
        O.load_bvh_cache(pw)  # wrong magic
