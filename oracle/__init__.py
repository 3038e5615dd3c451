"""CPU oracle for the smooth-distance hot path -- TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/_build/liboracle.so`` (built from
``oracle/*.cpp`` by ``oracle/Makefile``), a plain fp64 C++ restatement of
the reference evaluator in /root/reference/proj/include/smoothdist
(see the file:line citations in ``oracle/sdoracle.hpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import this package. It is the checker, never the thing
measured or shipped: ``paper_2108_10480_b200`` does not import it.

Parity pin: the reference cannot be built here (Eigen3, GTest and CLI11
are absent), so the restatement is pinned against every
known-answer test the reference holds for this path
(tests/golden/reference_known_answers.json, tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

NODE_DTYPE = np.dtype(
    [("lo", "<f8", 3), ("hi", "<f8", 3), ("left", "<i4"), ("right", "<i4"),
     ("primitive", "<i4"), ("count", "<i4"), ("diameter", "<f8")], align=False)
assert NODE_DTYPE.itemsize == 72  # reference BvhNode (bvh.hpp:14-22)


def build() -> str:
    """Compile the oracle library (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    vp, i64, i32, f64, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
    P = C.POINTER
    sig = {
        "sdo_last_error": (C.c_char_p, []),
        "sdo_mesh_create": (vp, [vp, i64, vp, vp, i64]),
        "sdo_mesh_free": (None, [vp]),
        "sdo_mesh_nv": (i64, [vp]),
        "sdo_mesh_ns": (i64, [vp]),
        "sdo_mesh_export": (None, [vp, vp, vp, vp]),
        "sdo_mesh_validate": (C.c_int, [vp]),
        "sdo_mesh_mean_edge": (f64, [vp]),
        "sdo_gen_config_mesh": (vp, [C.c_int]),
        "sdo_gen_config_queries": (C.c_int, [C.c_int, vp, i64, vp]),
        "sdo_gen_random_scene": (vp, [u64, C.c_int]),
        "sdo_gen_point_cluster": (vp, [C.c_int, u64, f64]),
        "sdo_gen_icosphere": (vp, [C.c_int]),
        "sdo_gen_uv_torus": (vp, [f64, f64, C.c_int, C.c_int]),
        "sdo_gen_triangle_fan": (vp, [C.c_int, u64]),
        "sdo_gen_polyline": (vp, [C.c_int, u64]),
        "sdo_gen_random_queries": (None, [u64, vp, C.c_int, vp, vp]),
        "sdo_gen_random_queries_scaled": (None, [u64, vp, C.c_int, f64, vp, vp]),
        "sdo_rng_new": (vp, [u64]),
        "sdo_rng_free": (None, [vp]),
        "sdo_rng_random_queries": (None, [vp, vp, C.c_int, vp, vp]),
        "sdo_weights_build": (vp, [vp]),
        "sdo_weights_unit": (vp, [vp]),
        "sdo_weights_free": (None, [vp]),
        "sdo_weights_info": (None, [vp, P(f64), P(f64), P(i32), P(i32), P(i64)]),
        "sdo_weights_export": (None, [vp] * 8),
        "sdo_weights_from_arrays": (vp, [f64, f64, i32, vp, i32, vp, i64, vp]),
        "sdo_weights_max_attenuated": (f64, [vp, vp]),
        "sdo_weights_eval": (None, [vp, vp, i64, vp, C.c_int, vp, vp, vp, vp]),
        "sdo_edge_weight": (None, [i32, i32, vp, vp]),
        "sdo_tri_weight": (None, [i32, i32, vp, vp]),
        "sdo_tri_poly_eval": (None, [vp, C.c_int, vp, vp, vp, vp]),
        "sdo_tri_poly_grid": (None, [vp, vp]),
        "sdo_bvh_build": (vp, [vp]),
        "sdo_bvh_from_nodes": (vp, [vp, i64]),
        "sdo_bvh_free": (None, [vp]),
        "sdo_bvh_size": (i64, [vp]),
        "sdo_bvh_export": (None, [vp, vp]),
        "sdo_box_point_proximity": (None, [vp, vp, C.c_int, vp, vp, vp]),
        "sdo_bh_condition": (C.c_int, [f64, f64, C.c_int, f64]),
        "sdo_point_simplex": (None, [vp, C.c_int, vp, vp]),
        "sdo_exact_min": (None, [vp, i64, vp, vp, vp, C.c_int]),
        "sdo_query": (C.c_int, [vp, vp, vp, vp, i64, vp, C.c_int] + [vp] * 8),
        "sdo_decision_mix": (u64, [u64, u64]),
        "sdo_mesh_dist": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp]),
        "sdo_hardware_threads": (C.c_int, []),
        "sdo_render": (C.c_int, [vp, vp, vp, vp, vp, C.c_int, vp, vp, vp, vp]),
        "sdo_write_ppm": (C.c_int, [vp, C.c_int, C.c_int, C.c_char_p]),
        "sdo_grid_benchmark": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, vp, vp, vp]),
        "sdo_write_grid_csv": (C.c_int, [vp, vp, vp, C.c_int, vp, C.c_char_p]),
        "sdo_save_bvh_cache": (C.c_int, [vp, C.c_char_p]),
        "sdo_load_bvh_cache": (vp, [C.c_char_p]),
        "sdo_save_weight_cache": (C.c_int, [vp, C.c_char_p]),
        "sdo_load_weight_cache": (vp, [C.c_char_p]),
        "sdo_query_simplices": (C.c_int, [vp, vp, vp, vp, vp, i64, vp, C.c_int] + [vp] * 8),
        "sdo_simplex_distance": (C.c_int, [vp, C.c_int, vp, C.c_int, C.c_int, vp]),
        "sdo_box_primitive_proximity": (C.c_int, [vp, vp, vp, C.c_int, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().sdo_last_error().decode())


def hardware_threads() -> int:
    return int(lib().sdo_hardware_threads())


def decision_mix(node: int, kind: int) -> int:
    return int(lib().sdo_decision_mix(node, kind))


# --------------------------------------------------------------------- mesh
class Mesh:
    """Oracle-side SimplexMesh (mesh.hpp:31-50); arrays are numpy copies."""

    def __init__(self, handle=None, vertices=None, simplices=None, kinds=None):
        if handle is None:
            vertices = np.ascontiguousarray(vertices, dtype=np.float64).reshape(-1, 3)
            simplices = np.ascontiguousarray(simplices, dtype=np.int32).reshape(-1, 3)
            kinds = np.ascontiguousarray(kinds, dtype=np.uint8).reshape(-1)
            handle = lib().sdo_mesh_create(_ptr(vertices), len(vertices), _ptr(simplices), _ptr(kinds), len(kinds))
        self.h = handle
        nv, ns = lib().sdo_mesh_nv(handle), lib().sdo_mesh_ns(handle)
        self.vertices = np.empty((nv, 3), np.float64)
        self.simplices = np.empty((ns, 3), np.int32)
        self.kinds = np.empty(ns, np.uint8)
        lib().sdo_mesh_export(handle, _ptr(self.vertices), _ptr(self.simplices), _ptr(self.kinds))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdo_mesh_free(self.h)
            self.h = None

    @property
    def num_simplices(self):
        return len(self.kinds)

    def validate(self):
        _check(lib().sdo_mesh_validate(self.h))

    def mean_edge_length(self):
        return float(lib().sdo_mesh_mean_edge(self.h))

    def quantized(self) -> "Mesh":
        """Copy with vertices rounded to float32 (fp32 configs)."""
        v = self.vertices.astype(np.float32).astype(np.float64)
        return Mesh(vertices=v, simplices=self.simplices, kinds=self.kinds)

    @staticmethod
    def from_arrays(vertices, simplices, kinds):
        return Mesh(vertices=vertices, simplices=simplices, kinds=kinds)


def config_mesh(cfg: int) -> Mesh:
    h = lib().sdo_gen_config_mesh(cfg)
    if not h:
        raise RuntimeError(lib().sdo_last_error().decode())
    return Mesh(h)


def config_queries(cfg: int, mesh: Mesh, nq: int) -> np.ndarray:
    out = np.empty((nq, 3), np.float64)
    _check(lib().sdo_gen_config_queries(cfg, mesh.h, nq, _ptr(out)))
    return out


def random_scene(seed: int, max_prims: int = 200) -> Mesh:
    return Mesh(lib().sdo_gen_random_scene(seed, max_prims))


def point_cluster(n: int, seed: int, spread: float = 0.4) -> Mesh:
    return Mesh(lib().sdo_gen_point_cluster(n, seed, spread))


def icosphere(sub: int) -> Mesh:
    return Mesh(lib().sdo_gen_icosphere(sub))


def uv_torus(major=0.35, minor=0.15, nu=60, nv=60) -> Mesh:
    return Mesh(lib().sdo_gen_uv_torus(major, minor, nu, nv))


def triangle_fan(k: int, seed: int) -> Mesh:
    return Mesh(lib().sdo_gen_triangle_fan(k, seed))


def polyline(n: int, seed: int) -> Mesh:
    return Mesh(lib().sdo_gen_polyline(n, seed))


def random_queries(seed: int, mesh: Mesh, n: int):
    """n query simplices from one mt19937_64(seed) stream (shapes.hpp:243-265):
    returns (corners (n,3,3), dims (n,))."""
    corners = np.empty((n, 3, 3), np.float64)
    dims = np.empty(n, np.int32)
    lib().sdo_gen_random_queries(seed, mesh.h, n, _ptr(corners), _ptr(dims))
    return corners, dims


def random_queries_scaled(seed: int, mesh: Mesh, n: int, size_scale: float):
    """random_query(rng, bounding_box(mesh), size_scale) x n (shapes.hpp:243-265)."""
    corners = np.empty((n, 3, 3), np.float64)
    dims = np.empty(n, np.int32)
    lib().sdo_gen_random_queries_scaled(seed, mesh.h, n, size_scale, _ptr(corners), _ptr(dims))
    return corners, dims


class QueryStream:
    """One mt19937_64 stream of random_query draws shared across scenes."""

    def __init__(self, seed: int):
        self.h = lib().sdo_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdo_rng_free(self.h)
            self.h = None

    def draw(self, mesh: Mesh, n: int):
        corners = np.empty((n, 3, 3), np.float64)
        dims = np.empty(n, np.int32)
        lib().sdo_rng_random_queries(self.h, mesh.h, n, _ptr(corners), _ptr(dims))
        return corners, dims

    def draw_points(self, mesh: Mesh, n: int) -> np.ndarray:
        corners, dims = self.draw(mesh, n)
        return np.ascontiguousarray(corners[dims == 0, 0, :])


def random_point_queries(seed: int, mesh: Mesh, n: int) -> np.ndarray:
    """The point queries among the first n draws of random_query."""
    corners, dims = random_queries(seed, mesh, n)
    return np.ascontiguousarray(corners[dims == 0, 0, :])


# ------------------------------------------------------------------ weights
@dataclass
class WeightTable:
    """A WeightSet (weights.hpp:565-579) as flat arrays -- the one table that
    both the oracle and the GPU consume (parity is defined given it)."""
    A: float
    sup_wtilde: float
    edge_a: np.ndarray      # (ne, 5)
    tri_stored: np.ndarray  # (nt, 13)
    poly_index: np.ndarray  # (N,) int32, -1 = unit weight
    edge_val: np.ndarray = None
    edge_supinf: np.ndarray = None
    tri_val: np.ndarray = None
    tri_sir: np.ndarray = None


class Weights:
    def __init__(self, handle):
        self.h = handle
        L = lib()
        A, sup = C.c_double(), C.c_double()
        ne, nt, npi = C.c_int32(), C.c_int32(), C.c_int64()
        L.sdo_weights_info(handle, C.byref(A), C.byref(sup), C.byref(ne), C.byref(nt), C.byref(npi))
        t = WeightTable(A.value, sup.value, np.zeros((ne.value, 5)), np.zeros((nt.value, 13)),
                        np.zeros(npi.value, np.int32), np.zeros((ne.value, 2), np.int32),
                        np.zeros((ne.value, 2)), np.zeros((nt.value, 2), np.int32), np.zeros((nt.value, 3)))
        L.sdo_weights_export(handle, _ptr(t.edge_a), _ptr(t.edge_val), _ptr(t.edge_supinf), _ptr(t.tri_stored),
                             _ptr(t.tri_val), _ptr(t.tri_sir), _ptr(t.poly_index))
        self.table = t

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdo_weights_free(self.h)
            self.h = None

    @staticmethod
    def build(mesh: Mesh) -> "Weights":
        h = lib().sdo_weights_build(mesh.h)
        if not h:
            raise RuntimeError(lib().sdo_last_error().decode())
        return Weights(h)

    @staticmethod
    def unit(mesh: Mesh) -> "Weights":
        return Weights(lib().sdo_weights_unit(mesh.h))

    @staticmethod
    def from_table(t: WeightTable) -> "Weights":
        ea = np.ascontiguousarray(t.edge_a, np.float64)
        ts = np.ascontiguousarray(t.tri_stored, np.float64)
        pi = np.ascontiguousarray(t.poly_index, np.int32)
        return Weights(lib().sdo_weights_from_arrays(t.A, t.sup_wtilde, len(ea), _ptr(ea), len(ts), _ptr(ts),
                                                     len(pi), _ptr(pi)))

    def max_attenuated_weight(self, params) -> float:
        return float(lib().sdo_weights_max_attenuated(self.h, _ptr(_params_array(params))))

    def evaluate(self, mesh: Mesh, i: int, phi, dim: int, params):
        p = np.ascontiguousarray(phi, np.float64)
        w, dw, gw = np.zeros(1), np.zeros(2), np.zeros(3)
        lib().sdo_weights_eval(mesh.h, self.h, i, _ptr(p), dim, _ptr(_params_array(params)), _ptr(w), _ptr(dw),
                               _ptr(gw))
        return w[0], dw, gw


def edge_weight(v0: int, v1: int):
    a, si = np.zeros(5), np.zeros(2)
    lib().sdo_edge_weight(v0, v1, _ptr(a), _ptr(si))
    return a, si[0], si[1]


def tri_weight(v: int, e: int):
    """(stored[13], sup, inf, residual) of build_tri_weight(v, e)."""
    s, sir = np.zeros(13), np.zeros(3)
    lib().sdo_tri_weight(v, e, _ptr(s), _ptr(sir))
    return s, sir[0], sir[1], sir[2]


def tri_poly_eval(stored, xy):
    st = np.ascontiguousarray(stored, np.float64)
    xy = np.ascontiguousarray(xy, np.float64).reshape(-1, 2)
    n = len(xy)
    v, dx, dy = np.zeros(n), np.zeros(n), np.zeros(n)
    lib().sdo_tri_poly_eval(_ptr(st), n, _ptr(xy), _ptr(v), _ptr(dx), _ptr(dy))
    return v, dx, dy


def tri_poly_grid(stored) -> np.ndarray:
    st = np.ascontiguousarray(stored, np.float64)
    g = np.zeros(64)
    lib().sdo_tri_poly_grid(_ptr(st), _ptr(g))
    return g.reshape(8, 8)


# ---------------------------------------------------------------------- bvh
class Tree:
    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sdo_bvh_free(self.h)
            self.h = None

    @staticmethod
    def build(mesh: Mesh) -> "Tree":
        return Tree(lib().sdo_bvh_build(mesh.h))

    @staticmethod
    def from_nodes(nodes: np.ndarray) -> "Tree":
        nodes = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
        return Tree(lib().sdo_bvh_from_nodes(_ptr(nodes), len(nodes)))

    def nodes(self) -> np.ndarray:
        n = lib().sdo_bvh_size(self.h)
        out = np.zeros(n, NODE_DTYPE)
        lib().sdo_bvh_export(self.h, _ptr(out))
        return out


def box_point_proximity(lo, hi, q):
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
    d, yb = np.zeros(len(q)), np.zeros((len(q), 3))
    lib().sdo_box_point_proximity(_ptr(lo), _ptr(hi), len(q), _ptr(q), _ptr(d), _ptr(yb))
    return d, yb


def bh_condition(diameter, distance, must_descend, beta) -> bool:
    return bool(lib().sdo_bh_condition(diameter, distance, int(must_descend), beta))


def point_simplex(corners, dim, q):
    c = np.zeros(9)
    cc = np.asarray(corners, np.float64).reshape(-1)
    c[:len(cc)] = cc
    qq = np.ascontiguousarray(q, np.float64)
    out = np.zeros(9)
    lib().sdo_point_simplex(_ptr(c), dim, _ptr(qq), _ptr(out))
    return {"distance": out[0], "phi": out[1:3], "point_f": out[3:6], "grad": out[6:9]}


def exact_min(mesh: Mesh, q, threads: int = 0):
    q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
    d, a = np.zeros(len(q)), np.zeros(len(q), np.int64)
    lib().sdo_exact_min(mesh.h, len(q), _ptr(q), _ptr(d), _ptr(a), threads or hardware_threads())
    return d, a


# ------------------------------------------------------------------- smooth
@dataclass
class Params:
    """SmoothParams (params.hpp:13-22)."""
    alpha: float = 100.0
    alpha_u: float = 600.0
    beta: float = 0.5
    alpha_q: float = 100.0
    epsilon: float = 1e-300

    def attenuation(self) -> float:
        return self.alpha / max(self.alpha, self.alpha_u)


def _params_array(p) -> np.ndarray:
    return np.array([p.alpha, p.alpha_u, p.beta, p.epsilon], np.float64)


@dataclass
class Results:
    d_hat: np.ndarray
    grad: np.ndarray
    c: np.ndarray
    grad_c: np.ndarray
    leaves: np.ndarray
    far_field: np.ndarray
    decision_hash: np.ndarray
    seconds: float


def query(mesh: Mesh, weights: Weights, q, params: Params, tree: Tree | None = None, threads: int = 0) -> Results:
    """Batched point queries: smooth_min_dist_flat when tree is None, else
    smooth_min_dist on that tree (smooth.hpp:166-198)."""
    q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
    n = len(q)
    r = Results(np.zeros(n), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)), np.zeros(n, np.int64),
                np.zeros(n, np.int64), np.zeros(n, np.uint64), 0.0)
    secs = np.zeros(1)
    _check(lib().sdo_query(mesh.h, weights.h, tree.h if tree is not None else None, _ptr(q), n,
                           _ptr(_params_array(params)), threads or hardware_threads(), _ptr(r.d_hat), _ptr(r.grad),
                           _ptr(r.c), _ptr(r.grad_c), _ptr(r.leaves), _ptr(r.far_field), _ptr(r.decision_hash),
                           _ptr(secs)))
    r.seconds = float(secs[0])
    return r


@dataclass
class MeshDistResults:
    d_hat: float
    vertex_grads: np.ndarray
    per_primitive: np.ndarray
    leaves: int
    far_field: int


def mesh_dist(mesh: Mesh, weights: Weights, query: Mesh, params: Params, tree: Tree | None = None,
              threads: int = 0) -> MeshDistResults:
    """smooth_mesh_dist (smooth.hpp:212-255) for any query mesh."""
    p = np.array([params.alpha, params.alpha_u, params.beta, params.epsilon, params.alpha_q], np.float64)
    d = np.zeros(1)
    vg = np.zeros((len(query.vertices), 3))
    pp = np.zeros(query.num_simplices)
    cnt = np.zeros(2, np.int64)
    _check(lib().sdo_mesh_dist(mesh.h, weights.h, tree.h if tree is not None else None, query.h, _ptr(p),
                               threads or hardware_threads(), _ptr(d), _ptr(vg), _ptr(pp), _ptr(cnt)))
    return MeshDistResults(float(d[0]), vg, pp, int(cnt[0]), int(cnt[1]))


# ------------------------------------------------------- simplex queries
def _corners(c, dims):
    c = np.ascontiguousarray(c, np.float64).reshape(-1, 9)
    d = np.ascontiguousarray(dims, np.int32).reshape(-1)
    assert len(c) == len(d)
    return c, d


def query_simplices(mesh: Mesh, weights: Weights, corners, dims, params: Params, tree: Tree | None = None,
                    threads: int = 0) -> Results:
    """Batched query SIMPLICES (points, edges, triangles; corners (n,3,3),
    unused corners ignored): smooth_min_dist(_flat) with a SimplexGeom g."""
    c, d = _corners(corners, dims)
    n = len(d)
    r = Results(np.zeros(n), np.zeros((n, 3)), np.zeros(n), np.zeros((n, 3)), np.zeros(n, np.int64),
                np.zeros(n, np.int64), np.zeros(n, np.uint64), 0.0)
    secs = np.zeros(1)
    _check(lib().sdo_query_simplices(mesh.h, weights.h, tree.h if tree is not None else None, _ptr(c), _ptr(d), n,
                                     _ptr(_params_array(params)), threads or hardware_threads(), _ptr(r.d_hat),
                                     _ptr(r.grad), _ptr(r.c), _ptr(r.grad_c), _ptr(r.leaves), _ptr(r.far_field),
                                     _ptr(r.decision_hash), _ptr(secs)))
    r.seconds = float(secs[0])
    return r


@dataclass
class PairResult:
    distance: float
    phi: np.ndarray
    lam: np.ndarray
    point_f: np.ndarray
    point_g: np.ndarray
    grad: np.ndarray


def simplex_distance(f, fdim: int, g, gdim: int, qp: bool = False) -> PairResult:
    """exact.hpp:342-367 (qp=True: simplex_distance_qp, :158-313)."""
    fc = np.zeros(9)
    gc = np.zeros(9)
    fa, ga = np.asarray(f, np.float64).reshape(-1), np.asarray(g, np.float64).reshape(-1)
    fc[:len(fa)] = fa
    gc[:len(ga)] = ga
    out = np.zeros(14)
    _check(lib().sdo_simplex_distance(_ptr(fc), fdim, _ptr(gc), gdim, int(qp), _ptr(out)))
    return PairResult(float(out[0]), out[1:3].copy(), out[3:5].copy(), out[5:8].copy(), out[8:11].copy(),
                      out[11:14].copy())


def box_primitive_proximity(lo, hi, g, gdim: int):
    """bvh.hpp:113-180 -> (distance, y_b, lambda, must_descend)."""
    gc = np.zeros(9)
    ga = np.asarray(g, np.float64).reshape(-1)
    gc[:len(ga)] = ga
    out = np.zeros(7)
    _check(lib().sdo_box_primitive_proximity(_ptr(np.asarray(lo, np.float64)), _ptr(np.asarray(hi, np.float64)),
                                             _ptr(gc), gdim, _ptr(out)))
    return float(out[0]), out[1:4].copy(), out[4:6].copy(), bool(out[6])


# ------------------------------------------------------- reference caches
def save_bvh_cache(tree: Tree, path: str):
    """save_bvh_cache (bvh.hpp:196-212, SDBV0001)."""
    _check(lib().sdo_save_bvh_cache(tree.h, path.encode()))


def load_bvh_cache(path: str) -> Tree:
    h = lib().sdo_load_bvh_cache(path.encode())
    if not h:
        raise RuntimeError(lib().sdo_last_error().decode())
    return Tree(h)


def save_weight_cache(weights: Weights, path: str):
    """save_weight_cache (weights.hpp:715-742, SDWT0001)."""
    _check(lib().sdo_save_weight_cache(weights.h, path.encode()))


def load_weight_cache(path: str) -> Weights:
    h = lib().sdo_load_weight_cache(path.encode())
    if not h:
        raise RuntimeError(lib().sdo_last_error().decode())
    return Weights(h)


# ------------------------------------------------------------- callers
@dataclass
class RenderResult:
    rgb: np.ndarray    # (H, W, 3) uint8
    hit_t: np.ndarray  # (H, W), -1 on miss
    leaves: int
    far_field: int
    rays: int
    hits: int
    seconds: float


def render_config(origin=(1.5, 1.5, 1.5), target=(0.5, 0.5, 0.5), up=(0, 1, 0), fov_deg=45.0, width=256,
                  height=256, threshold=0.0, max_steps=128) -> np.ndarray:
    """RenderConfig (render.hpp:17-25) as the 14 doubles the C entry takes."""
    return np.array([*origin, *target, *up, fov_deg, width, height, threshold, max_steps], np.float64)


def render(mesh: Mesh, weights: Weights, tree: Tree, params: Params, cfg=None, threads: int = 0) -> RenderResult:
    """render (render.hpp:77-134): per-pixel sphere tracing of d_hat = 0."""
    cfg = render_config() if cfg is None else np.asarray(cfg, np.float64)
    w, h = int(cfg[10]), int(cfg[11])
    rgb = np.zeros((h, w, 3), np.uint8)
    hit = np.zeros((h, w))
    st = np.zeros(4, np.int64)
    secs = np.zeros(1)
    _check(lib().sdo_render(mesh.h, weights.h, tree.h, _ptr(_params_array(params)), _ptr(cfg),
                            threads or hardware_threads(), _ptr(rgb), _ptr(hit), _ptr(st), _ptr(secs)))
    return RenderResult(rgb, hit, int(st[0]), int(st[1]), int(st[2]), int(st[3]), float(secs[0]))


def write_ppm(rgb: np.ndarray, path: str):
    rgb = np.ascontiguousarray(rgb, np.uint8)
    _check(lib().sdo_write_ppm(_ptr(rgb), rgb.shape[1], rgb.shape[0], path.encode()))


def grid_benchmark(mesh: Mesh, weights: Weights, tree: Tree, params: Params, n: int, threads: int = 0):
    """grid_benchmark (bench.hpp:29-70): (d_hat, leaves, far_field), x fastest."""
    n3 = n ** 3
    d, lv, fr = np.zeros(n3), np.zeros(n3, np.int64), np.zeros(n3, np.int64)
    _check(lib().sdo_grid_benchmark(mesh.h, weights.h, tree.h, _ptr(_params_array(params)), n,
                                    threads or hardware_threads(), _ptr(d), _ptr(lv), _ptr(fr)))
    return d, lv, fr


def write_grid_csv(d, leaves, far, n: int, slab_seconds, path: str):
    d = np.ascontiguousarray(d, np.float64)
    lv = np.ascontiguousarray(leaves, np.int64)
    fr = np.ascontiguousarray(far, np.int64)
    ss = np.ascontiguousarray(slab_seconds, np.float64)
    _check(lib().sdo_write_grid_csv(_ptr(d), _ptr(lv), _ptr(fr), n, _ptr(ss), path.encode()))
