"""GPU parity for SIMPLEX queries (edge / triangle query primitives, SURVEY
8(f) rank 2) through sd_query_simplices / sd_mesh_dist, against the CPU
oracle (oracle/sdoracle_simplex.hpp) on the same seeded inputs.

The simplex path computes in fp64 with no FMA contraction in both context
precisions, so the Barnes-Hut decisions (per-query leaves / far-field
counts and the decision hash) must be identical and the values agree to
fp64 tolerance: |d - d_ref| <= 1e-10 max(1, |d_ref|), |g - g_ref| <= 1e-9
max(1, |g_ref|). fp32 contexts see float-rounded geometry (both sides).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TD, TG = 1e-10, 1e-9


def _engine(sd, mesh, weights, prec, tree=None):
    e = sd.Engine(0, prec)
    e.set_geometry(mesh.vertices, mesh.simplices, mesh.kinds)
    e.set_weight_table(weights.table)
    if tree is not None:
        e.set_bvh(tree.nodes())
    return e


def _close(got, ref, what=""):
    fin = np.isfinite(ref.d_hat)
    assert (np.isfinite(got.d_hat) == fin).all(), f"{what}: +inf mismatch"
    err = np.abs(got.d_hat[fin] - ref.d_hat[fin]) / np.maximum(1.0, np.abs(ref.d_hat[fin]))
    assert err.size == 0 or err.max() <= TD, f"{what}: d_hat err {err.max():.3g}"
    gn = np.linalg.norm(ref.grad[fin], axis=1)
    gerr = np.linalg.norm(got.grad[fin] - ref.grad[fin], axis=1) / np.maximum(1.0, gn)
    assert gerr.size == 0 or gerr.max() <= TG, f"{what}: grad err {gerr.max():.3g}"
    assert not got.grad[~fin].any()


def _scene(O, seed, nprim, nq, prec, qseed):
    m = O.random_scene(seed, nprim)
    c, d = O.random_queries(qseed, m, nq)
    if prec == 0:
        m = m.quantized()
        c = c.astype(np.float32).astype(np.float64)
    return m, c, d


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("seed", [1, 2, 3, 5, 8, 13])
def test_simplex_tree_decisions_and_values(sd, oracle, prec, seed):
    O = oracle
    m, c, d = _scene(O, seed, 200, 300, prec, 500 + seed)
    assert (d == 1).any() and (d == 2).any()
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, prec, tree=t)
    for beta in (0.3, 0.6, 0.9):
        ref = O.query_simplices(m, w, c, d, O.Params(alpha=100.0, beta=beta), tree=t)
        got = e.query_simplices(c, d, sd.SmoothParams(alpha=100.0, beta=beta))
        assert (got.leaves == ref.leaves).all() and (got.far_field == ref.far_field).all()
        assert (got.decision_hash == ref.decision_hash).all()
        _close(got, ref, f"seed {seed} beta {beta}")


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("seed", [4, 6, 7])
def test_simplex_flat(sd, oracle, prec, seed):
    O = oracle
    m, c, d = _scene(O, seed, 150, 200, prec, 700 + seed)
    w = O.Weights.build(m)
    e = _engine(sd, m, w, prec)
    for alpha, alpha_u in ((100.0, 600.0), (20.0, 600.0), (900.0, 600.0)):
        p = O.Params(alpha=alpha, alpha_u=alpha_u, beta=0.0)
        ref = O.query_simplices(m, w, c, d, p)
        got = e.query_simplices(c, d, sd.SmoothParams(alpha=alpha, alpha_u=alpha_u, beta=0.0), mode=sd.SD_EXACT)
        assert (got.leaves == m.num_simplices).all() and not got.far_field.any()
        _close(got, ref, f"flat seed {seed} alpha {alpha}")


def test_simplex_tree_beta0_equals_flat(sd, oracle):
    O = oracle
    m, c, d = _scene(O, 9, 120, 150, 1, 901)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, 1, tree=t)
    p = sd.SmoothParams(alpha=100.0, beta=0.0)
    a = e.query_simplices(c, d, p, mode=sd.SD_BVH)
    b = e.query_simplices(c, d, p, mode=sd.SD_EXACT)
    assert (a.leaves == b.leaves).all() and not a.far_field.any()
    _close(a, O.query_simplices(m, w, c, d, O.Params(beta=0.0), tree=t), "beta0 tree")
    fin = np.isfinite(b.d_hat)
    assert (np.abs(a.d_hat[fin] - b.d_hat[fin]) <= 1e-10 * np.maximum(1, np.abs(b.d_hat[fin]))).all()


def test_simplex_lbvh_decisions(sd, oracle):
    """GPU LBVH exported to the oracle: identical decisions for simplex queries."""
    O = oracle
    m, c, d = _scene(O, 11, 200, 250, 0, 1100)
    w = O.Weights.build(m)
    e = _engine(sd, m, w, 0)
    e.build_bvh(sd.SD_BVH_LBVH)
    t = O.Tree.from_nodes(e.export_bvh())
    ref = O.query_simplices(m, w, c, d, O.Params(alpha=150.0, beta=0.5), tree=t)
    got = e.query_simplices(c, d, sd.SmoothParams(alpha=150.0, beta=0.5))
    assert (got.decision_hash == ref.decision_hash).all()
    _close(got, ref, "lbvh")


@pytest.mark.parametrize("split", ["0", "3", "", "frontier", "frontier32", "warp8", "warp16", "warp32"])
def test_simplex_split_traversal(sd, oracle, split, monkeypatch):
    """Every simplex traversal kernel -- K3W (group-cooperative QP, 8/16/32
    lanes per node), K3F (node-parallel), K3 (packets, slot split at depth
    0/3/auto) -- makes the oracle's decisions."""
    if split.startswith("warp"):
        monkeypatch.setenv("SDGPU_SIMPLEX_KERNEL", "warp")
        monkeypatch.setenv("SDGPU_SIMPLEX_GW", split[4:])
    elif split.startswith("frontier"):
        monkeypatch.setenv("SDGPU_SIMPLEX_KERNEL", "frontier")
        monkeypatch.setenv("SDGPU_FRONTIER_G", split[8:] or "4")
    else:
        monkeypatch.setenv("SDGPU_SIMPLEX_KERNEL", "pair")
        monkeypatch.setenv("SDGPU_SPLIT", split)
    O = oracle
    m, c, d = _scene(O, 3, 300, 100, 1, 333)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, 1, tree=t)
    ref = O.query_simplices(m, w, c, d, O.Params(alpha=120.0, beta=0.4), tree=t)
    got = e.query_simplices(c, d, sd.SmoothParams(alpha=120.0, beta=0.4))
    assert (got.decision_hash == ref.decision_hash).all() and (got.leaves == ref.leaves).all()
    _close(got, ref, f"split {split!r}")


def test_simplex_points_match_point_path_decisions(sd, oracle):
    """Point queries through the simplex path decide exactly like the
    oracle's point path (exact.hpp:344, bvh.hpp:122)."""
    O = oracle
    m = O.random_scene(5, 150)
    w, t = O.Weights.build(m), O.Tree.build(m)
    q = O.random_point_queries(8, m, 300)
    c = np.zeros((len(q), 3, 3))
    c[:, 0] = q
    e = _engine(sd, m, w, 1, tree=t)
    ref = O.query(m, w, q, O.Params(beta=0.5), tree=t)
    got = e.query_simplices(c, np.zeros(len(q), np.int32), sd.SmoothParams(beta=0.5))
    assert (got.decision_hash == ref.decision_hash).all()
    _close(got, ref, "points via simplex path")


def test_simplex_contact_queries(sd, oracle):
    """Query simplices touching / crossing primitives (d = 0 leaves: zero
    pair gradient, exact.hpp:62) -- same tie-breaks as the oracle."""
    O = oracle
    m = O.random_scene(21, 100)
    V, S, K = m.vertices, m.simplices, m.kinds
    rng = np.random.default_rng(3)
    c = np.zeros((60, 3, 3))
    d = np.zeros(60, np.int32)
    for i in range(60):
        p = int(rng.integers(len(K)))
        a = V[S[p, 0]]
        b = V[S[p, K[p]]] if K[p] > 0 else a + 0.1
        mid = 0.5 * (a + b)
        n = rng.normal(size=3) * 0.2
        c[i, 0], c[i, 1], c[i, 2] = mid - n, mid + n, mid + rng.normal(size=3) * 0.2
        d[i] = 1 + i % 2
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, 1, tree=t)
    for beta in (0.0, 0.5):
        ref = O.query_simplices(m, w, c, d, O.Params(alpha=200.0, beta=beta), tree=t)
        got = e.query_simplices(c, d, sd.SmoothParams(alpha=200.0, beta=beta), mode=sd.SD_BVH)
        assert (got.decision_hash == ref.decision_hash).all()
        _close(got, ref, f"contact beta {beta}")


def test_simplex_edge_cases(sd, oracle):
    O = oracle
    m = O.random_scene(2, 50)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, 1, tree=t)
    p = sd.SmoothParams(beta=0.5)
    r = e.query_simplices(np.zeros((0, 3, 3)), np.zeros(0, np.int32), p)
    assert r.d_hat.shape == (0,)
    with pytest.raises(sd.SdError):
        e.query_simplices(np.zeros((1, 3, 3)), np.array([3], np.int32), p)
    # degenerate query simplices (coincident corners) are valid queries
    c = np.zeros((2, 3, 3))
    c[:, :, 0] = 5.0
    ref = O.query_simplices(m, w, c, np.array([1, 2], np.int32), O.Params(beta=0.5), tree=t)
    got = e.query_simplices(c, np.array([1, 2], np.int32), p)
    assert (got.decision_hash == ref.decision_hash).all()
    _close(got, ref, "degenerate queries")
    # far queries underflow to +inf with a zero gradient (smooth.hpp:151-155)
    c = np.full((1, 3, 3), 50.0)
    got = e.query_simplices(c, np.array([2], np.int32), sd.SmoothParams(alpha=400.0, beta=0.5))
    assert math.isinf(got.d_hat[0]) and not got.grad.any()


@pytest.mark.parametrize("beta", [0.0, 0.5])
def test_mesh_dist_general_query_mesh(sd, oracle, beta):
    """smooth_mesh_dist with an edge + triangle query mesh (the paper's
    timing-table rows): d_hat, per-primitive inner distances and vertex
    gradients against the oracle."""
    O = oracle
    f = O.icosphere(2)
    w, t = O.Weights.build(f), O.Tree.build(f)
    q0 = O.random_scene(11, 60)
    assert (q0.kinds > 0).any()
    qv = q0.vertices * 0.3 + np.array([1.3, 0.1, -0.2])
    e = _engine(sd, f, w, 1, tree=t)
    p = O.Params(alpha=100.0, beta=beta, alpha_q=50.0)
    ref = O.mesh_dist(f, w, O.Mesh.from_arrays(qv, q0.simplices, q0.kinds), p, tree=t)
    got = e.smooth_mesh_dist_general(qv, q0.simplices, q0.kinds,
                                     sd.SmoothParams(alpha=100.0, beta=beta, alpha_q=50.0),
                                     mode=sd.SD_BVH)
    assert abs(got.d_hat - ref.d_hat) <= TD * max(1.0, abs(ref.d_hat))
    assert np.allclose(got.per_primitive, ref.per_primitive, rtol=0, atol=TD)
    err = np.linalg.norm(got.vertex_grads - ref.vertex_grads, axis=1)
    assert err.max() <= TG * max(1.0, np.abs(ref.vertex_grads).max())
