"""bench.py's multi-process plumbing on CPU (gloo): --gpus N without torchrun
spawns N ranks, the fixed batch is split into blocks that tile it exactly
once, the all-gathered results equal a single-rank evaluation, and a
world-size / --gpus mismatch is refused. Also the parity-statistics and
roofline-peak helpers the bench reports with."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _env():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["OMP_NUM_THREADS"] = "1"
    return env


def _last_json(out: str):
    lines = [x for x in out.splitlines() if x.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_spawn_two_ranks_split_fixed_batch():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=240, env=_env(), cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = _last_json(p.stdout)
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["backend"] == "gloo"
    blocks = line["blocks"]
    assert blocks[0][0] == 0 and blocks[-1][1] == 4096
    assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
    assert abs(line["checksum"] - line["checksum_single"]) <= 1e-9 * abs(line["checksum_single"])
    assert line["ms_per_step"] > 0 and line["value"] > 0


def test_single_rank_stub():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--stub", "--steps", "1", "--warmup", "1"],
                       capture_output=True, text=True, timeout=120, env=_env(), cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = _last_json(p.stdout)
    assert line["n_gpus"] == 1 and line["blocks"] == [[0, 4096]]


def test_world_size_must_match_gpus():
    env = _env()
    env.update({"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--stub"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert p.returncode != 0 and "WORLD_SIZE=1 but --gpus 2" in p.stderr


def test_parity_stats_forms():
    ref = np.array([0.004, 1.0, 10.0, np.inf])
    got = ref + np.array([1e-7, 2e-6, 5e-5, 0.0])
    g = np.tile([1.0, 0.0, 0.0], (4, 1))
    s = bench.parity_stats(got, g, ref, g, alpha=200.0, dtype="f32")
    assert s["inf_mismatch"] == 0 and s["finite"] == 3
    # survey form: 1e-7/1, 2e-6/1, 5e-5/10
    assert abs(s["d_hat_max_err_survey"] - 5e-6) < 1e-12
    # strict form: 1e-7/max(0.004, 1/200) = 2e-5 dominates
    assert abs(s["d_hat_max_err_strict"] - 2e-5) < 1e-12
    assert s["pass_survey"] and not s["pass_strict"] and s["d_hat_over_tol_strict"] == 1
    s = bench.parity_stats(np.array([1.0, np.inf]), None, np.array([1.0, 2.0]), None, 100.0, "f32")
    assert s["inf_mismatch"] == 1 and not s["pass_survey"]


def test_roofline_peak_is_the_largest_candidate():
    pk, src, c = bench.compute_peak({"ffma_tflops": 69.8, "ffma2_tflops": 72.9, "dfma_tflops": 36.5}, 1965.0, False)
    assert src == "nominal_at_sampled_clock" and abs(pk - 148 * 128 * 2 * 1.965e9 / 1e12) < 1e-9
    pk, src, _ = bench.compute_peak({"ffma_tflops": 80.0, "dfma_tflops": 36.5}, 1965.0, False)
    assert src == "ffma_probe" and pk == 80.0
    pk, src, _ = bench.compute_peak(None, 1000.0, True)
    assert abs(pk - 148 * 64 * 2 * 1e9 / 1e12) < 1e-9


def test_strong_blocks_tile_the_batch():
    for n, w in ((1048576, 8), (262144, 3), (5, 4)):
        b = bench.strong_blocks(n, w)
        assert b[0][0] == 0 and b[-1][1] == n and all(x[1] == y[0] for x, y in zip(b, b[1:]))
        sizes = [hi - lo for lo, hi in b]
        assert max(sizes) - min(sizes) <= 1
