"""The C++ front end (include/smoothdist_gpu.hpp, the reference's names over
the C ABI) builds with g++ and runs on the GPU: examples/query_example.cpp
(point queries exact + tree, query edges / triangles, mesh-to-mesh)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_example_runs(tmp_path):
    lib = os.path.join(ROOT, "paper_2108_10480_b200")
    exe = str(tmp_path / "query_example")
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "query_example.cpp"), "-L", lib, "-lsdgpu",
                    f"-Wl,-rpath,{lib}", "-o", exe], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mesh-to-mesh d_hat" in r.stdout and "g1 (dim 2)" in r.stdout
