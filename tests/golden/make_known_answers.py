"""Writes tests/golden/reference_known_answers.json.

The reference (/root/reference/proj) cannot be built in this image (Eigen3,
GTest and CLI11 are absent), so its outputs cannot be captured directly.
What pins the hot path instead are the known-answer tests the reference
itself holds; this script restates each one as data: the input, the
closed-form expected output derived in that test, its tolerance, and the
test's file:line. tests/test_oracle_golden.py checks the CPU oracle against
every case; tests/test_gpu_parity.py checks the CUDA path against the
smooth-distance cases.

Run:  python tests/golden/make_known_answers.py
"""
import json
import math
import os

T = "proj/tests/"
cases = []


def case(name, cite, kind, **kw):
    cases.append({"name": name, "cite": cite, "kind": kind, **kw})


# --- smooth distance closed forms (test_smooth.cpp) ------------------------
q = [0.3, -0.2, 0.6]
nq = math.sqrt(sum(x * x for x in q))
case("SinglePointClosedForm", T + "test_smooth.cpp:40-55", "smooth",
     mesh={"vertices": [[0, 0, 0]], "simplices": [[0, -1, -1]], "kinds": [0]},
     params={"alpha": 50.0, "alpha_u": 600.0, "beta": 0.0},
     queries=[q], expect_d_hat=[nq], expect_grad=[[x / nq for x in q]],
     expect_leaves=[1], expect_far=[0], tol_d=1e-12, tol_g=1e-12)

p = [0.1, 0.2, 0.3]
q = [1.0, 0.0, 0.0]
d = math.sqrt(sum((a - b) ** 2 for a, b in zip(q, p)))
case("CoincidentPointsShiftByLogCount", T + "test_smooth.cpp:57-72", "smooth",
     mesh={"vertices": [p, p], "simplices": [[0, -1, -1], [1, -1, -1]], "kinds": [0, 0]},
     params={"alpha": 80.0, "alpha_u": 600.0, "beta": 0.0},
     queries=[q], expect_d_hat=[d - math.log(2.0) / 80.0], tol_d=1e-12)

# FarClusterCollapsesToFarField: point_cluster(4, mt19937_64(3), 1e-3),
# alpha 100, beta 0.9, q = (2, .4, -.3): exactly one far-field term, zero
# leaves, d_hat = d_B - ln 4 / alpha, grad = (q - y_B)/|q - y_B|.
case("FarClusterCollapsesToFarField", T + "test_smooth.cpp:74-90", "far_cluster",
     cluster={"n": 4, "seed": 3, "spread": 1e-3},
     params={"alpha": 100.0, "alpha_u": 600.0, "beta": 0.9},
     queries=[[2.0, 0.4, -0.3]], expect_far=[1], expect_leaves=[0], tol_d=1e-12, tol_g=1e-9)

# FarQueryUnderflowsToInfinity: point_cluster(20, mt19937_64(2), 0.05),
# beta 0, q = (3, 0, 0): alpha 400 -> c == 0, +inf, zero gradient;
# alpha 200 -> finite, |d_hat - d_min| < 0.05, |grad| = 1 +- 1e-3.
case("FarQueryUnderflowsToInfinity", T + "test_smooth.cpp:201-219", "underflow",
     cluster={"n": 20, "seed": 2, "spread": 0.05}, queries=[[3.0, 0.0, 0.0]],
     alpha_inf=400.0, alpha_finite=200.0, tol_finite=0.05, tol_gnorm=1e-3)

# Quadrature negative control needs the edge integral (out of scope); the
# unit-edge exactness case is a quadrature rule test, not this path.

# --- exact distances (test_exact.cpp) --------------------------------------
case("PointPointExample", T + "test_exact.cpp:68-78", "pair",
     corners=[[3, 4, 0]], dim=0, q=[0, 0, 0], expect_distance=5.0, expect_grad=[-0.6, -0.8, 0.0], tol=1e-15)
case("EdgeEndpointClamp", T + "test_exact.cpp:79-85", "pair",
     corners=[[0, 0, 0], [1, 0, 0]], dim=1, q=[2, 1, 0], expect_distance=math.sqrt(2.0), expect_phi=[1.0, 0.0],
     expect_point_f=[1, 0, 0], tol=0.0)
case("EdgeInteriorProjection", T + "test_exact.cpp:87-93", "pair",
     corners=[[0, 0, 0], [1, 0, 0]], dim=1, q=[0.25, 2, 0], expect_distance=2.0, expect_phi=[0.25, 0.0],
     expect_grad=[0, 1, 0], tol=1e-15)
tri = [[0, 0, 0], [1, 0, 0], [0, 1, 0]]
case("TriangleInterior", T + "test_exact.cpp:95-103", "pair",
     corners=tri, dim=2, q=[0.25, 0.25, 3], expect_distance=3.0, expect_phi=[0.25, 0.25], tol=0.0)
case("TriangleVertexRegion", T + "test_exact.cpp:104-106", "pair",
     corners=tri, dim=2, q=[-1, -1, 0], expect_distance=math.sqrt(2.0), expect_point_f=[0, 0, 0], tol=0.0)
case("TriangleHypotenuseMidpoint", T + "test_exact.cpp:108-111", "pair",
     corners=tri, dim=2, q=[1, 1, 0], expect_distance=math.sqrt(0.5), expect_point_f=[0.5, 0.5, 0], tol=1e-15)
case("ContactOnTriangle", T + "test_exact.cpp:232-239", "pair",
     corners=[[0, 0, 0], [2, 0, 0], [0, 2, 0]], dim=2, q=[0.5, 0.5, 0], expect_distance=0.0,
     expect_grad=[0, 0, 0], tol=0.0)
case("BruteForceMinimumOverMesh", T + "test_exact.cpp:262-280", "exact_min",
     mesh={"vertices": [[0, 0, 0], [10, 0, 0], [10, 1, 0]], "simplices": [[0, -1, -1], [1, 2, -1]], "kinds": [0, 1]},
     queries=[[1, 0, 0], [9, 0.5, 0]], expect_distance=[1.0, 1.0], expect_argmin=[0, 1])

# --- bvh (test_bvh.cpp) ----------------------------------------------------
case("BoxProximityPointQueries", T + "test_bvh.cpp:82-94", "box",
     lo=[0, 0, 0], hi=[1, 1, 1], queries=[[2, 0.5, 0.5], [0.5, 0.5, 0.5]], expect_distance=[1.0, 0.0],
     expect_yb=[[1, 0.5, 0.5], [0.5, 0.5, 0.5]])
case("BhConditionTruthTable", T + "test_bvh.cpp:168-185", "bh",
     rows=[[1.0, 3.0, 0, 0.5, True], [1.0, 3.0, 0, 0.0, False], [1.0, 3.0, 0, 0.3, False],
           [1.0, 0.0, 0, 0.5, False], [1.0, 3.0, 1, 0.5, False]])

# --- weights (test_weights.cpp) --------------------------------------------
case("FrozenQuarticForValence22", T + "test_weights.cpp:23-33", "edge_poly",
     valences=[2, 2], expect_a=[0.5, 0.0, 8.0, -16.0, 8.0], expect_sup=1.0, expect_inf=0.5)
case("IsolatedEdgeIsConstantOne", T + "test_weights.cpp:35-41", "edge_poly",
     valences=[1, 1], expect_a=[1, 0, 0, 0, 0], expect_sup=1.0, expect_inf=1.0)
case("TriWeightInterpolationTargets", T + "test_weights.cpp:56-67", "tri_targets",
     valences=[6, 2], points=[[0, 0], [1, 0], [0, 1], [1 / 3, 0], [2 / 3, 0], [1 / 3, 2 / 3], [1 / 3, 1 / 3]],
     expect=[1 / 6, 1 / 6, 1 / 6, 0.5, 0.5, 0.5, 5 / 6], tol=1e-7)
case("MaxAttenuatedWeightBound", T + "test_weights.cpp:137-151", "max_weight",
     A=3.0, sup=1.2, params={"alpha": 300.0, "alpha_u": 600.0}, expect=math.sqrt(3.6))
case("PointPrimitivesGetScaledUnitWeight", T + "test_weights.cpp:153-169", "point_weight",
     fan={"k": 5, "seed": 42}, extra_point=[9, 9, 9], params={"alpha": 100.0, "alpha_u": 100.0},
     expect_A=5.0, expect_w=5.0)
case("FloorKeepsOutOfModelWeightsFinite", T + "test_weights.cpp:171-192", "floor_weight",
     params={"alpha": 100.0, "alpha_u": 600.0}, stored0=-2.0, phi=[0.2, 0.3],
     expect_w=1e-300 ** (100.0 / 600.0))
case("AttenuationExponentExamples", T + "test_weights.cpp:111-120", "attenuation",
     rows=[[600.0, 600.0, 1.0], [50.0, 600.0, 50.0 / 600.0], [1200.0, 600.0, 1.0]])

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_known_answers.json")
with open(out, "w") as f:
    json.dump({"source": "/root/reference/proj/tests (known-answer tests restated as data)",
               "generator": "tests/golden/make_known_answers.py", "cases": cases}, f, indent=1)
print(f"wrote {len(cases)} cases to {out}")
