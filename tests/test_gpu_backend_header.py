"""The reference-typed drop-in include/smoothdist_gpu_backend.hpp, compiled
against the reference's OWN headers (oracle/_ref/backend_check, built where
/root/reference exists by `make -C oracle ref`) and run on the GPU: the
scene reaches it through the reference's load_mesh / load_weight_cache /
build_bvh, and every batched Backend call (tree, flat, query simplices,
mesh-to-mesh) is compared in-process with the reference's own per-query
evaluator (tests/cpp/backend_check.cpp)."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "backend_check")


def write_obj(m, path):
    with open(path, "w") as f:
        for v in m.vertices:
            f.write("v %.17g %.17g %.17g\n" % tuple(v))
        for s, k in zip(m.simplices, m.kinds):
            f.write({0: "p %d\n", 1: "l %d %d\n", 2: "f %d %d %d\n"}[int(k)] % tuple(int(x) + 1 for x in s[:k + 1]))


def test_backend_check_is_built_where_the_reference_is():
    if not os.path.isdir("/root/reference/proj/include/smoothdist"):
        pytest.skip("reference headers absent (GPU box): the prebuilt binary is used there")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    assert os.access(EXE, os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("prec,alpha,beta", [(0, 100.0, 0.5), (1, 100.0, 0.5), (1, 300.0, 0.3)])
def test_backend_header_matches_the_reference_on_gpu(oracle, prec, alpha, beta, tmp_path):
    if not os.access(EXE, os.X_OK):
        pytest.skip("oracle/_ref/backend_check not built")
    O = oracle
    m = O.random_scene(21, 300)
    q = O.QueryStream(2121).draw_points(m, 400)
    if prec == 0:
        m = m.quantized()
        q = q.astype(np.float32).astype(np.float64)
    w = O.Weights.build(m)
    write_obj(m, tmp_path / "mesh.obj")
    O.save_weight_cache(w, str(tmp_path / "w.sdwt"))
    np.ascontiguousarray(q, np.float64).tofile(tmp_path / "q.bin")
    r = subprocess.run([EXE, str(tmp_path / "mesh.obj"), str(tmp_path / "w.sdwt"), str(tmp_path / "q.bin"), str(prec),
                        str(alpha), str(beta)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "BACKEND CHECK OK" in r.stdout, r.stdout + r.stderr
