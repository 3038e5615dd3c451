"""The reference's acceptance gate (T/acceptance.cpp) run on
the GPU path, scaled to seconds: [1] underestimate and beta-dominance,
[2] the log(W N)/alpha lower bound, [3] finite-difference gradients,
[7] time grows with the leaves visited, [9] alpha-monotonicity with unit
weights. (The checks on the weight build [4], quadrature [5] and the demo
[8] are outside the query path; [6] is covered by test_callers.py.)
Distances d_min come from the oracle's exact point-simplex minimum."""
import math
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _engine(sd, O, m, w, prec, tree=None):
    e = sd.Engine(0, prec)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.set_weight_table(w.table)
    if tree is not None:
        e.set_bvh(tree.nodes())
    return e


@pytest.mark.parametrize("prec", [0, 1])
def test_acceptance_1_2_bounds_and_beta_dominance(sd, oracle, prec):
    """[1] d_hat <= d_min and d_hat(beta) <= d_hat(0) for beta in
    {0.2, 0.5, 0.9}; [2] d_hat >= d_min - log(W N) / alpha
    (acceptance.cpp:76-150): 25 scenes x 40 queries."""
    O = oracle
    tol = 1e-5 if prec == 0 else 1e-9
    for seed in range(1, 26):
        m = O.random_scene(seed, 150)
        if prec == 0:
            m = m.quantized()
        w, t = O.Weights.build(m), O.Tree.build(m)
        q = O.random_point_queries(500 + seed, m, 40)
        if prec == 0:
            q = q.astype(np.float32).astype(np.float64)
        e = _engine(sd, O, m, w, prec, tree=t)
        alpha = 100.0
        W = w.max_attenuated_weight(O.Params(alpha=alpha, alpha_u=600.0))
        slack = math.log(W * m.num_simplices) / alpha
        dmin, _ = O.exact_min(m, q)
        r0 = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=0.0))
        fin = np.isfinite(r0.d_hat)
        scale = np.maximum(1.0, np.abs(dmin))
        assert (r0.d_hat[fin] <= dmin[fin] + tol * scale[fin]).all(), f"[1] seed {seed}"
        assert (r0.d_hat[fin] >= dmin[fin] - slack - tol * scale[fin]).all(), f"[2] seed {seed}"
        for beta in (0.2, 0.5, 0.9):
            rb = e.smooth_min_dist(q, sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=beta))
            assert (rb.d_hat <= r0.d_hat + tol * np.maximum(1.0, np.abs(r0.d_hat))).all(), f"[1] beta {beta}"


def test_acceptance_3_finite_difference_gradients(sd, oracle):
    """[3] the returned gradient against central differences of d_hat with
    the reference's criterion (acceptance.cpp:157-249): alpha 100, h = 1e-5,
    probes with d_hat > 1e-2, |fd - grad| / max(|grad|, |fd|, 1e-2) < 1e-4;
    fp64, exact (beta 0, as the reference) and Barnes-Hut (probes whose
    decisions change across the stencil skipped). Unit weights: with built
    weights the reference's gradient is not the derivative of its d_hat --
    weight_gradient_world (weights.hpp:675-697) already divides the shape
    gradient by alpha and push_leaf_term (smooth.hpp:51-61) divides grad w by
    alpha again -- and the oracle restatement misses this very check by up
    to 2e-2 on these scenes; the GPU reproduces the reference's value there
    (parity tests), so the derivative check runs where the two agree."""
    O = oracle
    h = 1e-5
    checked = 0
    for seed in range(3001, 3011):
        m = O.random_scene(seed, 200)
        w, t = O.Weights.unit(m), O.Tree.build(m)
        q = O.random_point_queries(seed, m, 120)
        e = _engine(sd, O, m, w, 1, tree=t)
        for beta in (0.0, 0.5):
            p = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=beta)
            f = (lambda x: e.smooth_min_dist(x, p)) if beta > 0 else (lambda x: e.smooth_min_dist_flat(x, p))
            r = f(q)
            fd = np.zeros_like(q)
            same = np.isfinite(r.d_hat) & (r.d_hat > 1e-2)
            for a in range(3):
                dq = np.zeros(3)
                dq[a] = h
                rp, rm = f(q + dq), f(q - dq)
                same &= (rp.far_field == rm.far_field) & (rp.leaves == rm.leaves)
                same &= np.isfinite(rp.d_hat) & np.isfinite(rm.d_hat)
                fd[:, a] = (rp.d_hat - rm.d_hat) / (2 * h)
            den = np.maximum(np.maximum(np.linalg.norm(r.grad, axis=1), np.linalg.norm(fd, axis=1)), 1e-2)
            err = (np.linalg.norm(fd - r.grad, axis=1) / den)[same]
            assert (err < 1e-4).all(), (seed, beta, err.max())
            checked += int(same.sum())
    assert checked > 500


def test_acceptance_7_time_grows_with_leaves(sd, oracle):
    """[7] evaluation time against leaves visited (acceptance.cpp:395-422,
    Pearson r > 0.9): on the GPU the unit of timing is a batch, so the batch
    time over beta in {0, 0.05, ..., 0.9} on a 20k-triangle torus is
    correlated with the batch's total exact leaves + far-field terms."""
    import torch
    O = oracle
    m = O.uv_torus(0.35, 0.15, 100, 100)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, O, m, w, 0, tree=t)
    q = O.random_point_queries(77, m, 16384).astype(np.float32)
    dev = torch.device("cuda", 0)
    qd = torch.tensor(q, device=dev)
    n = len(q)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    lv = torch.empty(n, dtype=torch.int64, device=dev)
    fr = torch.empty(n, dtype=torch.int64, device=dev)
    work, times = [], []
    for beta in (0.0, 0.05, 0.1, 0.2, 0.3, 0.5, 0.7, 0.9):
        p = sd.SmoothParams(alpha=200.0, alpha_u=600.0, beta=beta)
        run = lambda: e.query_points_device(qd.data_ptr(), n, p, sd.SD_BVH, d.data_ptr(), leaves_ptr=lv.data_ptr(),
                                            far_ptr=fr.data_ptr())
        run()
        torch.cuda.synchronize()
        work.append(float(lv.double().sum() * 20.0 + fr.double().sum()))  # a leaf term ~ 20 far terms
        t0 = time.perf_counter()
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) / 5)
    r = np.corrcoef(work, times)[0, 1]
    assert r > 0.9, (r, work, times)


@pytest.mark.parametrize("prec", [0, 1])
def test_acceptance_9_alpha_monotone_unit_weights(sd, oracle, prec):
    """[9] with unit weights d_hat is nondecreasing in alpha
    (acceptance.cpp:466-495): alpha in {10, 20, 50, 100, 200, 400}."""
    O = oracle
    tol = 1e-5 if prec == 0 else 1e-12
    for seed in (3, 8, 13):
        m = O.random_scene(seed, 150)
        if prec == 0:
            m = m.quantized()
        w = O.Weights.unit(m)
        q = O.random_point_queries(70 + seed, m, 60)
        if prec == 0:
            q = q.astype(np.float32).astype(np.float64)
        e = _engine(sd, O, m, w, prec)
        prev = None
        for alpha in (10.0, 20.0, 50.0, 100.0, 200.0, 400.0):
            r = e.smooth_min_dist_flat(q, sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=0.0))
            if prev is not None:
                fin = np.isfinite(r.d_hat) & np.isfinite(prev)
                assert (r.d_hat[fin] >= prev[fin] - tol * np.maximum(1.0, np.abs(prev[fin]))).all(), (seed, alpha)
            prev = r.d_hat
