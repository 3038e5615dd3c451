"""the batched callers -- render (render.hpp:77-134) as a
device wavefront, grid_benchmark (bench.hpp:29-70) as one batch -- and their
writers (write_ppm / write_png / write_grid_csv), against the oracle's
restatements (oracle/sdoracle_callers.hpp)."""
import math
import os

import numpy as np
import pytest


def _benchmark_frame(O, m):
    """normalize_to_benchmark_frame (mesh.hpp:126-135): scale 0.5 / diagonal,
    centre to (0.5, 0.5, 0.5)."""
    v = m.vertices
    lo, hi = v.min(0), v.max(0)
    e = hi - lo
    diag = math.sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2])
    scale = 0.5 / diag if diag > 0 else 1.0
    off = 0.5 - scale * (0.5 * (lo + hi))
    return O.Mesh.from_arrays(scale * v + off, m.simplices, m.kinds)


# ------------------------------------------------------- writers (CPU)
def test_ppm_bytes_are_exact(sd, oracle, tmp_path):  # test_render.cpp:120-137
    rgb = (np.arange(5 * 3 * 3) * 7 % 256).astype(np.uint8).reshape(3, 5, 3)
    a, b = str(tmp_path / "a.ppm"), str(tmp_path / "b.ppm")
    sd.write_ppm(rgb, a)
    oracle.write_ppm(rgb, b)
    data = open(a, "rb").read()
    assert data == open(b, "rb").read()
    assert data == b"P6\n5 3\n255\n" + rgb.tobytes()


def test_png_header_and_dimensions(sd, tmp_path):  # test_render.cpp:139-160
    import zlib
    rgb = (np.arange(48 * 32 * 3) % 251).astype(np.uint8).reshape(32, 48, 3)
    p = str(tmp_path / "a.png")
    sd.write_png(rgb, p)
    b = open(p, "rb").read()
    assert b[:8] == bytes([137, 80, 78, 71, 13, 10, 26, 10])
    assert int.from_bytes(b[8:12], "big") == 13 and b[12:16] == b"IHDR"
    assert int.from_bytes(b[16:20], "big") == 48 and int.from_bytes(b[20:24], "big") == 32
    assert b[24] == 8 and b[25] == 2
    # the IDAT payload decompresses to filter-0 scanlines of the image
    n = int.from_bytes(b[33:37], "big")
    assert b[37:41] == b"IDAT"
    raw = zlib.decompress(b[41:41 + n])
    assert raw == b"".join(b"\0" + rgb[y].tobytes() for y in range(32))


def test_grid_csv_matches_reference_writer(sd, oracle, tmp_path):
    n = 3
    rng = np.random.default_rng(1)
    d = rng.normal(size=n ** 3)
    d[4] = np.inf
    lv = rng.integers(0, 1000, n ** 3)
    fr = rng.integers(0, 1000, n ** 3)
    ss = rng.uniform(0, 1, n)
    a, b = str(tmp_path / "a.csv"), str(tmp_path / "b.csv")
    sd.write_grid_csv(d, lv, fr, n, ss, a)
    oracle.write_grid_csv(d, lv, fr, n, ss, b)
    assert open(a).read() == open(b).read()
    assert open(a).readline() == "voxel_index,d_hat,leaves_visited,far_field,slab_time_s\n"


# ---------------------------------------------------------------- GPU
def _engine(sd, m, w, t, prec):
    e = sd.Engine(0, prec)
    e.set_geometry(m.vertices, m.simplices, m.kinds)
    e.set_weight_table(w.table)
    e.set_bvh(t.nodes())
    return e


@pytest.mark.gpu
def test_render_mesh_behind_camera_misses(sd, oracle):  # test_render.cpp:44-56
    O = oracle
    m = O.icosphere(0)
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, t, 1)
    r = e.render(sd.SmoothParams(), origin=(0, 0, 3), target=(0, 0, 6), width=16, height=16)
    assert r.hits == 0 and r.rays == 256 and (r.hit_t == -1.0).all() and not r.rgb.any()


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [1, 0])
def test_render_single_point_matches_oracle(sd, oracle, prec):  # test_render.cpp:58-86
    """Hit in the centre, miss in the corner; every pixel as the oracle.
    (The reference test also expects a near-white centre pixel, but its own
    march steps from t = 0 straight to t = d_hat = 3, the point itself, where
    the slightly off-axis ray sees a gradient almost orthogonal to it: both
    the oracle and the GPU shade it 17.)"""
    O = oracle
    m = O.Mesh.from_arrays([[0, 0, 0]], [[0, -1, -1]], [0])
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, t, prec)
    cfg = dict(origin=(0, 0, 3), target=(0, 0, 0), width=64, height=64, threshold=0.5)
    r = e.render(sd.SmoothParams(beta=0.0), **cfg)
    ref = O.render(m, w, t, O.Params(beta=0.0), O.render_config(**cfg))
    assert r.hits > 0 and 2.4 <= r.hit_t[32, 32] <= 3.01 and r.hit_t[0, 0] == -1.0 and r.rgb[0, 0, 0] == 0
    assert (r.hit_t >= 0).sum() == r.hits == ref.hits
    assert np.array_equal(r.hit_t >= 0, ref.hit_t >= 0)
    assert np.abs(r.hit_t - ref.hit_t).max() <= (1e-9 if prec == 1 else 1e-5)  # fp32 d_hat: 1e-5 relative
    assert np.abs(r.rgb.astype(int) - ref.rgb.astype(int)).max() <= (0 if prec == 1 else 1)


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [1, 0])
def test_render_icosphere_benchmark_frame(sd, oracle, prec):  # test_render.cpp:88-118
    """Default camera on icosphere(1) in the benchmark frame: deterministic,
    self-consistent (hits = lit pixels, gray >= 16), and pixel for pixel the
    oracle's image (fp64: identical hit sets and shades; fp32 d_hat moves
    a hit by at most one marching step on a few grazing rays)."""
    O = oracle
    m = _benchmark_frame(O, O.icosphere(1))
    if prec == 0:
        m = m.quantized()
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, t, prec)
    a = e.render(sd.SmoothParams(), width=48, height=48)
    b = e.render(sd.SmoothParams(), width=48, height=48)
    assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.hit_t, b.hit_t) and a.leaves == b.leaves
    assert a.hits > 0 and a.rays == 48 * 48
    hit = a.hit_t >= 0
    assert hit.sum() == a.hits and (a.rgb[..., 0] > 0).sum() == a.hits
    assert (a.rgb[hit][:, 0] >= 16).all()
    assert (a.rgb[..., 0] == a.rgb[..., 1]).all() and (a.rgb[..., 0] == a.rgb[..., 2]).all()
    ref = O.render(m, w, t, O.Params(), O.render_config(width=48, height=48))
    same = (a.hit_t >= 0) == (ref.hit_t >= 0)
    if prec == 1:
        assert same.all() and a.leaves == ref.leaves and a.far_field == ref.far_field
        assert np.abs(a.hit_t - ref.hit_t).max() <= 1e-9
        assert np.abs(a.rgb.astype(int) - ref.rgb.astype(int)).max() <= 1
    else:
        assert same.mean() >= 0.99
        both = (a.hit_t >= 0) & (ref.hit_t >= 0)
        assert np.abs(a.hit_t[both] - ref.hit_t[both]).max() <= 2e-3


@pytest.mark.gpu
@pytest.mark.parametrize("prec", [1, 0])
def test_grid_benchmark_matches_oracle(sd, oracle, prec):
    O = oracle
    m = _benchmark_frame(O, O.random_scene(3, 150))
    if prec == 0:
        m = m.quantized()
    w, t = O.Weights.build(m), O.Tree.build(m)
    e = _engine(sd, m, w, t, prec)
    n = 12
    d, lv, fr, secs = e.grid_benchmark(sd.SmoothParams(alpha=100.0, beta=0.5), n)
    rd, rl, rf = O.grid_benchmark(m, w, t, O.Params(alpha=100.0, beta=0.5), n)
    assert (lv == rl).all() and (fr == rf).all() and secs > 0
    tol = 1e-10 if prec == 1 else 1e-5
    fin = np.isfinite(rd)
    assert (np.isfinite(d) == fin).all()
    assert (np.abs(d[fin] - rd[fin]) <= tol * np.maximum(1, np.abs(rd[fin]))).all()
