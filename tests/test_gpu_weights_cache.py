"""the GPU WeightSet precompute (adjacency, valences and
first-occurrence polynomial assignment on the device, adjacency.cu) and the
reference's binary caches (SDBV0001 bvh.hpp:190-236, SDWT0001
weights.hpp:700-781) through the C ABI, checked against the oracle's
restatements byte for byte."""
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mesh_cases(O):
    yield "scene1", O.random_scene(1, 200)
    yield "scene6", O.random_scene(6, 400)
    yield "icosphere4", O.icosphere(4)
    yield "fan", O.triangle_fan(9, 3)
    yield "polyline", O.polyline(300, 5)
    yield "cfg2", O.config_mesh(2)


@pytest.mark.parametrize("case", ["scene1", "scene6", "icosphere4", "fan", "polyline", "cfg2"])
def test_gpu_assignment_matches_reference_build(sd, oracle, case, tmp_path):
    """Valences, first-occurrence polynomial ids, edge polynomials, A and
    the triangle (v, e) keys equal the restated build_weight_set
    (weights.hpp:589-621); triangle coefficients may differ in LP ties
    (DESIGN.md 2), so they are not compared."""
    O = oracle
    m = dict(_mesh_cases(O))[case]
    ref = O.Weights.build(m).table
    e = sd.Engine(0, sd.SD_FP64)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    got = e.build_weights()
    assert got.A == ref.A
    assert (got.poly_index == ref.poly_index).all()
    assert got.edge_a.shape == ref.edge_a.shape and (got.edge_a == ref.edge_a).all()
    assert got.tri_stored.shape == ref.tri_stored.shape
    path = str(tmp_path / "w.sdwt")
    e.save_weight_cache(path)
    back = O.load_weight_cache(path).table
    assert (back.edge_val == ref.edge_val).all() and (back.tri_val == ref.tri_val).all()
    assert np.allclose(back.edge_supinf, ref.edge_supinf, rtol=0, atol=1e-15)
    if len(ref.tri_stored) == 0:
        assert got.sup_wtilde == ref.sup_wtilde


def test_gpu_assignment_equals_host_pass_at_cfg4_scale(sd, monkeypatch):
    """5.24M triangles (BASELINE configs[3]): device assignment == the host
    hash-map pass, bit for bit."""
    from paper_2108_10480_b200 import configs
    w, _ = configs.cfg4(nq=1)
    e = sd.Engine(0, sd.SD_FP32)
    e.set_geometry(configs.quantize(w.vertices), w.simplices, w.kinds)
    t0 = time.perf_counter()
    gpu = e.build_weights()
    t_gpu = time.perf_counter() - t0
    monkeypatch.setenv("SDGPU_WEIGHTS_HOST", "1")
    t0 = time.perf_counter()
    host = e.build_weights()
    t_host = time.perf_counter() - t0
    print(f"build_weights cfg4: device assignment {t_gpu:.3f} s, host pass {t_host:.3f} s")
    assert gpu.A == host.A and gpu.sup_wtilde == host.sup_wtilde
    assert (gpu.poly_index == host.poly_index).all()
    assert (gpu.edge_a == host.edge_a).all() and (gpu.tri_stored == host.tri_stored).all()


def test_bvh_cache_interchange(sd, oracle, tmp_path):
    O = oracle
    m = O.random_scene(3, 300)
    t = O.Tree.build(m)
    po, pg = str(tmp_path / "o.sdbv"), str(tmp_path / "g.sdbv")
    O.save_bvh_cache(t, po)
    e = sd.Engine(0, sd.SD_FP32)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.load_bvh_cache(po)
    assert e.export_bvh().tobytes() == t.nodes().tobytes()
    e.save_bvh_cache(pg)
    assert open(pg, "rb").read() == open(po, "rb").read()
    # a GPU-built LBVH read back by the oracle
    e.build_bvh(sd.SD_BVH_LBVH)
    e.save_bvh_cache(pg)
    assert O.load_bvh_cache(pg).nodes().tobytes() == e.export_bvh().tobytes()
    # wrong mesh size / wrong magic are errors, as in load_bvh_cache
    e2 = sd.Engine(0, sd.SD_FP32)
    m2 = O.random_scene(4, 50)
    e2.set_geometry(m2.vertices, m2.simplices, m2.kinds)
    with pytest.raises(sd.SdError):
        e2.load_bvh_cache(po)
    O.save_weight_cache(O.Weights.build(m2), str(tmp_path / "w"))
    with pytest.raises(sd.SdError):
        e2.load_bvh_cache(str(tmp_path / "w"))


def test_weight_cache_interchange(sd, oracle, tmp_path):
    O = oracle
    m = O.random_scene(8, 300)
    w, t = O.Weights.build(m), O.Tree.build(m)
    po, pg = str(tmp_path / "o.sdwt"), str(tmp_path / "g.sdwt")
    O.save_weight_cache(w, po)
    e = sd.Engine(0, sd.SD_FP64)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.load_weight_cache(po)
    got = e.weight_table()
    assert got.A == w.table.A and got.sup_wtilde == w.table.sup_wtilde
    assert (got.edge_a == w.table.edge_a).all() and (got.tri_stored == w.table.tri_stored).all()
    assert (got.poly_index == w.table.poly_index).all()
    e.save_weight_cache(pg)
    assert open(pg, "rb").read() == open(po, "rb").read()
    # evaluating with the loaded table reproduces the oracle
    e.set_bvh(t.nodes())
    q = O.random_point_queries(17, m, 200)
    ref = O.query(m, w, q, O.Params(beta=0.5), tree=t)
    r = e.smooth_min_dist(q, sd.SmoothParams(beta=0.5))
    assert (r.decision_hash == ref.decision_hash).all()
    assert np.abs(r.d_hat - ref.d_hat).max() <= 1e-10 * max(1.0, np.abs(ref.d_hat).max())
