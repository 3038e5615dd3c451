"""The REFERENCE itself, compiled -- TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/_ref/libsdref.so``: the unmodified reference
headers (/root/reference/proj/include/smoothdist, read-only, never copied)
compiled by ``make -C oracle ref`` with the Eigen-subset shim of
``oracle/eigen_shim`` (Eigen is not in the image; see that header for what
it pins and what it cannot: Eigen's SIMD rounding, and the triangle
weight-polynomial SVD, for which the WeightSet table is fed in).

Used to pin the fp64 restatement in ``oracle/`` against the reference's own
code (tests/test_oracle_reference.py) and, where present, by the GPU parity
tests and bench.py's reference arm. The library is built here (where
/root/reference exists) and travels to the GPU box with the repo snapshot;
callers check ``available()`` first.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libsdref.so")
REF_INCLUDE = "/root/reference/proj/include"
_lib = None

NODE_DTYPE = np.dtype(
    [("lo", "<f8", 3), ("hi", "<f8", 3), ("left", "<i4"), ("right", "<i4"),
     ("primitive", "<i4"), ("count", "<i4"), ("diameter", "<f8")], align=False)


def build() -> str | None:
    """Compile oracle/_ref when the reference headers are present."""
    if os.path.isdir(os.path.join(REF_INCLUDE, "smoothdist")):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
    return LIB_PATH if os.path.exists(LIB_PATH) else None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise ImportError(f"{LIB_PATH} is missing: run `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        P = C.POINTER
        sig = {
            "sdr_last_error": (C.c_char_p, []),
            "sdr_scene_create": (vp, [vp, i64, vp, vp, i64, f64, f64, i32, vp, i32, vp, vp]),
            "sdr_scene_free": (None, [vp]),
            "sdr_scene_set_bvh": (C.c_int, [vp, vp, i64]),
            "sdr_scene_bvh_size": (i64, [vp]),
            "sdr_scene_export_bvh": (C.c_int, [vp, vp]),
            "sdr_query": (C.c_int, [vp, vp, vp, i64, vp, C.c_int, C.c_int, vp, vp, vp, vp, vp, vp, P(f64)]),
            "sdr_build_weights_no_tris": (C.c_int, [vp, i64, vp, vp, i64, vp, P(f64), P(f64), P(i32), vp, i32,
                                                    vp]),
        }
        for name, (res, argt) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = argt
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().sdr_last_error().decode())


@dataclass
class Results:
    d_hat: np.ndarray
    grad: np.ndarray
    c: np.ndarray
    grad_c: np.ndarray
    leaves: np.ndarray
    far_field: np.ndarray
    seconds: float


class Scene:
    """smoothdist::SimplexMesh + WeightSet (+ Bvh) of the compiled reference."""

    def __init__(self, vertices, simplices, kinds, table):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(simplices, np.int32).reshape(-1, 3)
        k = np.ascontiguousarray(kinds, np.uint8).reshape(-1)
        ea = np.ascontiguousarray(table.edge_a, np.float64).reshape(-1, 5)
        ts = np.ascontiguousarray(table.tri_stored, np.float64).reshape(-1, 13)
        pi = np.ascontiguousarray(table.poly_index, np.int32).reshape(-1)
        self.n = len(k)
        self.h = lib().sdr_scene_create(_ptr(v), len(v), _ptr(s), _ptr(k), len(k), float(table.A),
                                        float(table.sup_wtilde), len(ea), _ptr(ea), len(ts), _ptr(ts), _ptr(pi))
        if not self.h:
            raise RuntimeError(lib().sdr_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdr_scene_free(self.h)
            self.h = None

    def set_bvh(self, nodes=None):
        """Install a reference-layout tree, or build one with the reference's build_bvh."""
        if nodes is None:
            _check(lib().sdr_scene_set_bvh(self.h, None, 0))
        else:
            nodes = np.ascontiguousarray(nodes, NODE_DTYPE)
            _check(lib().sdr_scene_set_bvh(self.h, _ptr(nodes), len(nodes)))

    def bvh(self) -> np.ndarray:
        out = np.zeros(lib().sdr_scene_bvh_size(self.h), NODE_DTYPE)
        _check(lib().sdr_scene_export_bvh(self.h, _ptr(out)))
        return out

    def query(self, q, params, tree: bool = False, threads: int = 0, dims=None) -> Results:
        """smooth_min_dist (tree) / smooth_min_dist_flat for point queries
        (q: Q x 3) or query simplices (q: Q x 9 corners, dims: Q)."""
        if dims is None:
            q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
        else:
            q = np.ascontiguousarray(q, np.float64).reshape(-1, 9)
            dims = np.ascontiguousarray(dims, np.int32)
        n = len(q)
        r = Results(np.zeros(n), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)), np.zeros(n, np.int64),
                    np.zeros(n, np.int64), 0.0)
        p = np.array([params.alpha, params.alpha_u, params.beta, params.epsilon,
                      getattr(params, "alpha_q", 100.0)], np.float64)
        secs = C.c_double()
        _check(lib().sdr_query(self.h, _ptr(q), _ptr(dims), n, _ptr(p), 1 if tree else 0,
                               threads or os.cpu_count() or 1, _ptr(r.d_hat), _ptr(r.grad), _ptr(r.c), _ptr(r.grad_c),
                               _ptr(r.leaves), _ptr(r.far_field), C.byref(secs)))
        r.seconds = secs.value
        return r


def build_weights_no_tris(vertices, simplices, kinds):
    """The reference's build_adjacency + build_weight_set for a mesh
    without triangles: (vertex valences, A, sup_wtilde, edge_a, poly_index)."""
    v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
    s = np.ascontiguousarray(simplices, np.int32).reshape(-1, 3)
    k = np.ascontiguousarray(kinds, np.uint8).reshape(-1)
    val = np.zeros(len(v), np.int32)
    A, sup, ne = C.c_double(), C.c_double(), C.c_int32()
    cap = 4096
    ea = np.zeros((cap, 5))
    pi = np.zeros(len(k), np.int32)
    _check(lib().sdr_build_weights_no_tris(_ptr(v), len(v), _ptr(s), _ptr(k), len(k), _ptr(val), C.byref(A),
                                           C.byref(sup), C.byref(ne), _ptr(ea), cap, _ptr(pi)))
    return val, A.value, sup.value, ea[:ne.value].copy(), pi
