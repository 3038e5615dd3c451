"""B200-native smooth-distance query engine (arXiv 2108.10480).

Python host mirror of the reference C++ evaluator API
(/root/reference/proj/include/smoothdist/smooth.hpp:166-198), bound through
ctypes to the C ABI of ``include/sdgpu.h`` implemented by ``libsdgpu.so``
(hand-written sm_100a CUDA, built in-tree by ``make -C paper_2108_10480_b200``).

Names follow the reference: :class:`SmoothParams` (params.hpp:13-22),
:class:`SmoothResult` fields (smooth.hpp:20-27), ``smooth_min_dist`` /
``smooth_min_dist_flat`` as batched calls. There is no CPU fallback: when the
library or a CUDA device is missing every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SDGPU_LIB: another build of the same library (A/B timing, tools/lib_ab.py)
LIB_PATH = os.environ.get("SDGPU_LIB") or os.path.join(_HERE, "libsdgpu.so")

SD_FP32, SD_FP64 = 0, 1
SD_EXACT, SD_BVH = 0, 1
SD_BVH_MEDIAN, SD_BVH_LBVH, SD_BVH_AUTO = 0, 1, 2
SD_POINT, SD_EDGE, SD_TRIANGLE = 0, 1, 2

NODE_DTYPE = np.dtype(
    [("lo", "<f8", 3), ("hi", "<f8", 3), ("left", "<i4"), ("right", "<i4"),
     ("primitive", "<i4"), ("count", "<i4"), ("diameter", "<f8")], align=False)
assert NODE_DTYPE.itemsize == 72

# Every symbol include/sdgpu.h declares (tests check the library exports them).
EXPORTED_SYMBOLS = (
    "sd_last_error", "sd_abi_version", "sd_create", "sd_destroy", "sd_set_geometry", "sd_set_weights",
    "sd_set_bvh", "sd_build_bvh", "sd_bvh_size", "sd_export_bvh", "sd_query_points", "sd_query_points_device",
    "sd_finalize_device", "sd_query_points_async", "sd_query_wait", "sd_query_points_device_shard", "sd_last_launch_count", "sd_set_kernel_timing", "sd_set_exact_pruning", "sd_kernel_times", "sd_build_weights", "sd_weights_info", "sd_export_weights",
    "sd_mesh_dist_points",
    "sd_query_simplices",
    "sd_mesh_dist",
    "sd_scatter_partials",
    "sd_query_points_scatter",
    "sd_reduce_owned",
    "sd_render",
    "sd_grid_benchmark",
    "sd_write_ppm",
    "sd_write_png",
    "sd_write_grid_csv",
    "sd_save_bvh_cache",
    "sd_load_bvh_cache",
    "sd_save_weight_cache",
    "sd_load_weight_cache",
)


class SdError(RuntimeError):
    """A failed C-ABI call (the reference raises std::runtime_error via fail())."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"sdgpu error {code}: {msg}")
        self.code = code


class _Params(C.Structure):
    _fields_ = [("alpha", C.c_double), ("alpha_u", C.c_double), ("beta", C.c_double), ("epsilon", C.c_double)]


class _RenderConfig(C.Structure):
    _fields_ = [("origin", C.c_double * 3), ("target", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_deg", C.c_double), ("width", C.c_int32), ("height", C.c_int32), ("threshold", C.c_double),
                ("max_steps", C.c_int32)]


class _Outputs(C.Structure):
    _fields_ = [("d_hat", C.c_void_p), ("grad", C.c_void_p), ("c", C.c_void_p), ("grad_c", C.c_void_p),
                ("leaves", C.c_void_p), ("far_field", C.c_void_p), ("decision_hash", C.c_void_p)]


_lib = None


def build(force: bool = False) -> str:
    """Compile libsdgpu.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    args = ["make", "-s", "-C", _HERE, "-j4"]
    if force:
        subprocess.run(["make", "-s", "-C", _HERE, "clean"], check=True)
    subprocess.run(args, check=True)
    return LIB_PATH


def lib():
    """Load libsdgpu.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2108_10480_b200.build() (make -C paper_2108_10480_b200)")
        L = C.CDLL(LIB_PATH)
        vp, i64, i32, f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        P = C.POINTER
        sig = {
            "sd_last_error": (C.c_char_p, []),
            "sd_abi_version": (C.c_int, []),
            "sd_create": (C.c_int, [P(vp), C.c_int, C.c_int]),
            "sd_destroy": (C.c_int, [vp]),
            "sd_set_geometry": (C.c_int, [vp, vp, i64, vp, vp, i64]),
            "sd_set_weights": (C.c_int, [vp, f64, f64, i32, vp, i32, vp, vp]),
            "sd_set_bvh": (C.c_int, [vp, vp, i64]),
            "sd_build_bvh": (C.c_int, [vp, C.c_int]),
            "sd_bvh_size": (C.c_int, [vp, P(i64)]),
            "sd_export_bvh": (C.c_int, [vp, vp, i64]),
            "sd_query_points": (C.c_int, [vp, vp, i64, P(_Params), C.c_int, P(_Outputs)]),
            "sd_query_points_device": (C.c_int, [vp, vp, i64, P(_Params), C.c_int, P(_Outputs), vp]),
            "sd_query_points_async": (C.c_int, [vp, vp, i64, P(_Params), C.c_int, P(_Outputs), P(i64)]),
            "sd_query_points_device_shard": (C.c_int, [vp, vp, i64, P(_Params), P(_Outputs), i32, i32, vp]),
            "sd_query_wait": (C.c_int, [vp, i64]),
            "sd_finalize_device": (C.c_int, [vp, vp, vp, i64, P(_Params), vp, vp, vp]),
            "sd_last_launch_count": (C.c_int, [vp, P(i64)]),
            "sd_set_kernel_timing": (C.c_int, [vp, C.c_int]),
            "sd_set_exact_pruning": (C.c_int, [vp, C.c_double]),
            "sd_kernel_times": (C.c_int, [vp, vp, i64, P(i64)]),
            "sd_build_weights": (C.c_int, [vp]),
            "sd_weights_info": (C.c_int, [vp, P(f64), P(f64), P(i32), P(i32)]),
            "sd_export_weights": (C.c_int, [vp, vp, vp, vp]),
            "sd_mesh_dist_points": (C.c_int, [vp, vp, i64, vp, i64, P(_Params), f64, C.c_int, vp, vp, vp]),
            "sd_query_simplices": (C.c_int, [vp, vp, vp, i64, P(_Params), C.c_int, P(_Outputs)]),
            "sd_mesh_dist": (C.c_int, [vp, vp, i64, vp, vp, i64, P(_Params), f64, C.c_int, vp, vp, vp]),
            "sd_render": (C.c_int, [vp, P(_Params), C.c_int, P(_RenderConfig), vp, vp, vp, vp]),
            "sd_scatter_partials": (C.c_int, [vp, vp, vp, i64, vp, i32, i32, i64, vp]),
            "sd_query_points_scatter": (C.c_int, [vp, vp, i64, P(_Params), C.c_int, vp, i32, i32, i64, vp, vp, vp]),
            "sd_reduce_owned": (C.c_int, [vp, vp, i64, i64, i32, P(_Params), vp, vp, vp]),
            "sd_grid_benchmark": (C.c_int, [vp, P(_Params), C.c_int, i32, vp, vp, vp, vp]),
            "sd_write_ppm": (C.c_int, [vp, i32, i32, C.c_char_p]),
            "sd_write_png": (C.c_int, [vp, i32, i32, C.c_char_p]),
            "sd_write_grid_csv": (C.c_int, [vp, vp, vp, i32, vp, C.c_char_p]),
            "sd_save_bvh_cache": (C.c_int, [vp, C.c_char_p]),
            "sd_load_bvh_cache": (C.c_int, [vp, C.c_char_p]),
            "sd_save_weight_cache": (C.c_int, [vp, C.c_char_p]),
            "sd_load_weight_cache": (C.c_int, [vp, C.c_char_p]),
        }
        for name, (res, argt) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = argt
        _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise SdError(rc, lib().sd_last_error().decode())


def _ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


@dataclass
class SmoothParams:
    """SmoothParams (params.hpp:13-22); defaults are the reference's."""
    alpha: float = 100.0
    alpha_u: float = 600.0
    beta: float = 0.5
    alpha_q: float = 100.0
    epsilon: float = 1e-300

    def attenuation(self) -> float:
        return self.alpha / max(self.alpha, self.alpha_u)

    def _c(self) -> _Params:
        return _Params(self.alpha, self.alpha_u, self.beta, self.epsilon)


@dataclass
class WeightTable:
    """WeightSet as flat arrays (weights.hpp:565-579)."""
    A: float
    sup_wtilde: float
    edge_a: np.ndarray      # (ne, 5)
    tri_stored: np.ndarray  # (nt, 13)
    poly_index: np.ndarray  # (N,) int32, -1 = unit weight


@dataclass
class MeshDistResult:
    """MeshDistResult (smooth.hpp:281-286)."""
    d_hat: float
    vertex_grads: np.ndarray
    per_primitive: np.ndarray


@dataclass
class SmoothResults:
    """Batched SmoothResult (smooth.hpp:20-27): one row per query."""
    d_hat: np.ndarray
    grad: np.ndarray | None = None
    c: np.ndarray | None = None
    grad_c: np.ndarray | None = None
    leaves: np.ndarray | None = None
    far_field: np.ndarray | None = None
    decision_hash: np.ndarray | None = None


class Engine:
    """One sd_ctx bound to one CUDA device (one process per GPU)."""

    def __init__(self, device: int = 0, precision: int = SD_FP32):
        h = C.c_void_p()
        _check(lib().sd_create(C.byref(h), device, precision))
        self.h = h
        self.device = device
        self.precision = precision
        self.num_simplices = 0

    def close(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.sd_destroy(self.h)
            self.h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- geometry / weights / tree (mesh.hpp, weights.hpp, bvh.hpp) --
    def set_geometry(self, vertices, simplices, kinds):
        v = np.ascontiguousarray(vertices, np.float64).reshape(-1, 3)
        s = np.ascontiguousarray(simplices, np.int32).reshape(-1, 3)
        k = np.ascontiguousarray(kinds, np.uint8).reshape(-1)
        _check(lib().sd_set_geometry(self.h, _ptr(v), len(v), _ptr(s), _ptr(k), len(k)))
        self.num_simplices = len(k)

    def set_weights(self, A, sup_wtilde, edge_a, tri_stored, poly_index):
        ea = np.ascontiguousarray(edge_a, np.float64).reshape(-1, 5)
        ts = np.ascontiguousarray(tri_stored, np.float64).reshape(-1, 13)
        pi = np.ascontiguousarray(poly_index, np.int32).reshape(-1)
        _check(lib().sd_set_weights(self.h, float(A), float(sup_wtilde), len(ea), _ptr(ea), len(ts), _ptr(ts),
                                    _ptr(pi)))

    def set_weight_table(self, t):
        """Accepts any object with A, sup_wtilde, edge_a, tri_stored, poly_index."""
        self.set_weights(t.A, t.sup_wtilde, t.edge_a, t.tri_stored, t.poly_index)

    def build_weights(self) -> "WeightTable":
        """build_weight_set (weights.hpp:589-621): adjacency, valences and the
        polynomial assignment on the device, polynomials on the host;
        installs and returns the table."""
        _check(lib().sd_build_weights(self.h))
        return self.weight_table()

    def weight_table(self) -> "WeightTable":
        A, sup = C.c_double(), C.c_double()
        ne, nt = C.c_int32(), C.c_int32()
        _check(lib().sd_weights_info(self.h, C.byref(A), C.byref(sup), C.byref(ne), C.byref(nt)))
        t = WeightTable(A.value, sup.value, np.zeros((ne.value, 5)), np.zeros((nt.value, 13)),
                        np.zeros(self.num_simplices, np.int32))
        _check(lib().sd_export_weights(self.h, _ptr(t.edge_a), _ptr(t.tri_stored), _ptr(t.poly_index)))
        return t

    def set_bvh(self, nodes: np.ndarray):
        nodes = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
        _check(lib().sd_set_bvh(self.h, _ptr(nodes), len(nodes)))

    def build_bvh(self, method: int = SD_BVH_LBVH):
        _check(lib().sd_build_bvh(self.h, method))

    def export_bvh(self) -> np.ndarray:
        n = C.c_int64()
        _check(lib().sd_bvh_size(self.h, C.byref(n)))
        out = np.zeros(n.value, NODE_DTYPE)
        _check(lib().sd_export_bvh(self.h, _ptr(out), n.value))
        return out

    # -- queries (smooth.hpp:166-198) --
    def query_points(self, q, params: SmoothParams, mode: int = SD_EXACT, *, want_grad=True, want_c=False,
                     want_counters=False, out: SmoothResults | None = None) -> SmoothResults:
        """Host-buffer batched query: H2D, evaluate, D2H (blocking). `out`
        may supply preallocated (e.g. pinned) result arrays."""
        q = np.ascontiguousarray(q, np.float64).reshape(-1, 3)
        n = len(q)
        if out is not None:
            r = out
            o = _Outputs(*(None if a is None else a.ctypes.data for a in
                           (r.d_hat, r.grad, r.c, r.grad_c, r.leaves, r.far_field, r.decision_hash)))
            _check(lib().sd_query_points(self.h, _ptr(q), n, C.byref(params._c()), mode, C.byref(o)))
            return r
        r = SmoothResults(np.empty(n))
        if want_grad:
            r.grad = np.empty((n, 3))
        if want_c:
            r.c, r.grad_c = np.empty(n), np.empty((n, 3))
        if want_counters:
            r.leaves, r.far_field = np.empty(n, np.int64), np.empty(n, np.int64)
            r.decision_hash = np.empty(n, np.uint64)
        o = _Outputs(*(None if a is None else a.ctypes.data for a in
                       (r.d_hat, r.grad, r.c, r.grad_c, r.leaves, r.far_field, r.decision_hash)))
        _check(lib().sd_query_points(self.h, _ptr(q), n, C.byref(params._c()), mode, C.byref(o)))
        return r

    def query_points_async(self, q, params: SmoothParams, mode: int, out: SmoothResults) -> int:
        """Pipelined host-buffer batch (sd_query_points_async): returns a
        ticket at once; q and out must stay alive and untouched until
        wait(ticket). Use pinned arrays for copy / compute overlap."""
        assert q.dtype == np.float64 and q.flags.c_contiguous
        r = out
        o = _Outputs(*(None if a is None else a.ctypes.data for a in
                       (r.d_hat, r.grad, r.c, r.grad_c, r.leaves, r.far_field, r.decision_hash)))
        t = C.c_int64()
        _check(lib().sd_query_points_async(self.h, _ptr(q), len(q), C.byref(params._c()), mode, C.byref(o),
                                           C.byref(t)))
        return t.value

    def wait(self, ticket: int = -1):
        """Wait for one pipelined batch (or every batch in flight)."""
        _check(lib().sd_query_wait(self.h, ticket))

    def query_points_device(self, q_ptr: int, n: int, params: SmoothParams, mode: int, d_hat_ptr: int,
                            grad_ptr: int | None = None, c_ptr: int | None = None, grad_c_ptr: int | None = None,
                            leaves_ptr: int | None = None, far_ptr: int | None = None, hash_ptr: int | None = None,
                            stream: int | None = None):
        """Device-buffer batched query on `stream` (raw CUDA pointers, e.g.
        torch ``tensor.data_ptr()``); q is float32 (SD_FP32) or float64."""
        o = _Outputs(d_hat_ptr, grad_ptr, c_ptr, grad_c_ptr, leaves_ptr, far_ptr, hash_ptr)
        _check(lib().sd_query_points_device(self.h, C.c_void_p(q_ptr), n, C.byref(params._c()), mode, C.byref(o),
                                            C.c_void_p(stream) if stream else None))

    def query_points_device_shard(self, q_ptr: int, n: int, params: SmoothParams, world: int, rank: int,
                                  d_hat_ptr: int, grad_ptr: int | None = None, leaves_ptr: int | None = None,
                                  far_ptr: int | None = None, hash_ptr: int | None = None,
                                  stream: int | None = None):
        """This rank's interleaved share (packets rank, rank + world, ...)
        of the tree evaluation of the whole device batch q_ptr
        (sd_query_points_device_shard); other output entries untouched."""
        o = _Outputs(d_hat_ptr, grad_ptr, None, None, leaves_ptr, far_ptr, hash_ptr)
        _check(lib().sd_query_points_device_shard(self.h, C.c_void_p(q_ptr), n, C.byref(params._c()), C.byref(o),
                                                  world, rank, C.c_void_p(stream) if stream else None))

    def finalize_device(self, c_ptr: int, grad_c_ptr: int, n: int, params: SmoothParams, d_hat_ptr: int,
                        grad_ptr: int | None, stream: int | None = None):
        _check(lib().sd_finalize_device(self.h, C.c_void_p(c_ptr), C.c_void_p(grad_c_ptr), n, C.byref(params._c()),
                                        C.c_void_p(d_hat_ptr), C.c_void_p(grad_ptr) if grad_ptr else None,
                                        C.c_void_p(stream) if stream else None))

    def scatter_partials(self, c_ptr: int, grad_c_ptr: int, n: int, peer_table_ptr: int, world: int, rank: int,
                         q_per_owner: int, stream: int | None = None):
        """Store this rank's partial sums into the owners' symmetric buffers
        (peer_table_ptr: device array of the world buffer pointers)."""
        _check(lib().sd_scatter_partials(self.h, C.c_void_p(c_ptr), C.c_void_p(grad_c_ptr), n,
                                         C.c_void_p(peer_table_ptr), world, rank, q_per_owner,
                                         C.c_void_p(stream) if stream else None))

    def query_points_scatter(self, q_ptr: int, n: int, params: SmoothParams, mode: int, peer_table_ptr: int,
                             world: int, rank: int, q_per_owner: int, leaves_ptr: int | None = None,
                             far_ptr: int | None = None, stream: int | None = None):
        """Evaluate this rank's shard for device queries q_ptr and store the
        partial sums straight into the owners' symmetric buffers from the
        finalize epilogue (the fused form of query_points_device +
        scatter_partials)."""
        _check(lib().sd_query_points_scatter(self.h, C.c_void_p(q_ptr), n, C.byref(params._c()), mode,
                                             C.c_void_p(peer_table_ptr), world, rank, q_per_owner,
                                             C.c_void_p(leaves_ptr) if leaves_ptr else None,
                                             C.c_void_p(far_ptr) if far_ptr else None,
                                             C.c_void_p(stream) if stream else None))

    def reduce_owned(self, sbuf_ptr: int, q_per_owner: int, n_owned: int, world: int, params: SmoothParams,
                     d_hat_ptr: int, grad_ptr: int | None, stream: int | None = None):
        """Sum the world contributions of this rank's owned queries and finalise."""
        _check(lib().sd_reduce_owned(self.h, C.c_void_p(sbuf_ptr), q_per_owner, n_owned, world, C.byref(params._c()),
                                     C.c_void_p(d_hat_ptr), C.c_void_p(grad_ptr) if grad_ptr else None,
                                     C.c_void_p(stream) if stream else None))

    def set_exact_pruning(self, bits: float = 48.0):
        """Pruned exact evaluation (sd_set_exact_pruning): tiles whose terms are
        below 2^-bits of a lower bound of the query's sum are skipped; 0
        restores the sum over all pairs (smooth.hpp:189-198)."""
        _check(lib().sd_set_exact_pruning(self.h, float(bits)))

    def set_kernel_timing(self, on: bool = True):
        """Record a CUDA event pair around the dominant compute launches of
        every following query call (see sd_set_kernel_timing)."""
        _check(lib().sd_set_kernel_timing(self.h, 1 if on else 0))

    def kernel_times(self) -> np.ndarray:
        """Milliseconds of the timed launch groups since the last read (synchronises)."""
        n = C.c_int64()
        _check(lib().sd_kernel_times(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.float64)
        _check(lib().sd_kernel_times(self.h, _ptr(out), n.value, C.byref(n)))
        return out

    def last_launch_count(self) -> int:
        n = C.c_int64()
        _check(lib().sd_last_launch_count(self.h, C.byref(n)))
        return n.value

    def smooth_min_dist(self, q, params: SmoothParams) -> SmoothResults:
        """Batched smooth_min_dist (smooth.hpp:166-184): tree path when beta > 0."""
        mode = SD_BVH if params.beta > 0 else SD_EXACT
        return self.query_points(q, params, mode, want_c=True, want_counters=True)

    def smooth_mesh_dist(self, query_vertices, params: SmoothParams, query_points=None,
                         mode: int | None = None) -> "MeshDistResult":
        """smooth_mesh_dist (smooth.hpp:212-255) for a point-cloud query mesh:
        outer LogSumExp with params.alpha_q over the inner smooth distances;
        tree path when beta > 0."""
        v = np.ascontiguousarray(query_vertices, np.float64).reshape(-1, 3)
        pts = None if query_points is None else np.ascontiguousarray(query_points, np.int32).reshape(-1)
        n = len(v) if pts is None else len(pts)
        d = np.zeros(1)
        vg = np.zeros((len(v), 3))
        pp = np.zeros(n)
        if mode is None:
            mode = SD_BVH if params.beta > 0 else SD_EXACT
        _check(lib().sd_mesh_dist_points(self.h, _ptr(v), len(v), _ptr(pts), n, C.byref(params._c()),
                                         float(params.alpha_q), mode, _ptr(d), _ptr(vg), _ptr(pp)))
        return MeshDistResult(float(d[0]), vg, pp)

    def query_simplices(self, corners, dims, params: SmoothParams, mode: int | None = None) -> SmoothResults:
        """Batched query SIMPLICES (smooth_min_dist / _flat with a SimplexGeom
        g, smooth.hpp:166-198): corners (n, 3, 3) (unused corners ignored),
        dims (n,) in {0, 1, 2}; tree path when beta > 0 unless `mode` says."""
        c = np.ascontiguousarray(corners, np.float64).reshape(-1, 9)
        d = np.ascontiguousarray(dims, np.int32).reshape(-1)
        if len(c) != len(d):
            raise ValueError("corners and dims differ in length")
        n = len(d)
        if mode is None:
            mode = SD_BVH if params.beta > 0 else SD_EXACT
        r = SmoothResults(np.empty(n), np.empty((n, 3)), np.empty(n), np.empty((n, 3)), np.empty(n, np.int64),
                          np.empty(n, np.int64), np.empty(n, np.uint64))
        o = _Outputs(*(a.ctypes.data for a in (r.d_hat, r.grad, r.c, r.grad_c, r.leaves, r.far_field,
                                               r.decision_hash)))
        _check(lib().sd_query_simplices(self.h, _ptr(c), _ptr(d), n, C.byref(params._c()), mode, C.byref(o)))
        return r

    def smooth_mesh_dist_general(self, query_vertices, query_simplices, query_kinds, params: SmoothParams,
                                 mode: int | None = None) -> "MeshDistResult":
        """smooth_mesh_dist (smooth.hpp:212-255) for any query mesh: simplices
        (n, 3) vertex indices (-1 past the corners), kinds (n,)."""
        v = np.ascontiguousarray(query_vertices, np.float64).reshape(-1, 3)
        sv = np.ascontiguousarray(query_simplices, np.int32).reshape(-1, 3)
        k = np.ascontiguousarray(query_kinds, np.uint8).reshape(-1)
        n = len(k)
        d = np.zeros(1)
        vg = np.zeros((len(v), 3))
        pp = np.zeros(n)
        if mode is None:
            mode = SD_BVH if params.beta > 0 else SD_EXACT
        _check(lib().sd_mesh_dist(self.h, _ptr(v), len(v), _ptr(sv), _ptr(k), n, C.byref(params._c()),
                                  float(params.alpha_q), mode, _ptr(d), _ptr(vg), _ptr(pp)))
        return MeshDistResult(float(d[0]), vg, pp)

    # -- batched callers (render.hpp:77-134, bench.hpp:29-70) --
    def render(self, params: SmoothParams, origin=(1.5, 1.5, 1.5), target=(0.5, 0.5, 0.5), up=(0.0, 1.0, 0.0),
               fov_deg=45.0, width=256, height=256, threshold=0.0, max_steps=128,
               mode: int = SD_BVH) -> "RenderResult":
        """Sphere-traced image of d_hat = 0 (render.hpp:77-134)."""
        cfg = _RenderConfig((C.c_double * 3)(*origin), (C.c_double * 3)(*target), (C.c_double * 3)(*up),
                            float(fov_deg), int(width), int(height), float(threshold), int(max_steps))
        rgb = np.zeros((height, width, 3), np.uint8)
        hit = np.zeros((height, width))
        st = np.zeros(4, np.int64)
        secs = np.zeros(1)
        _check(lib().sd_render(self.h, C.byref(params._c()), mode, C.byref(cfg), _ptr(rgb), _ptr(hit), _ptr(st),
                               _ptr(secs)))
        return RenderResult(rgb, hit, int(st[0]), int(st[1]), int(st[2]), int(st[3]), float(secs[0]))

    def grid_benchmark(self, params: SmoothParams, n: int, mode: int = SD_BVH):
        """d_hat, leaves, far-field counts at the n^3 voxel centres of [0,1]^3
        (x fastest) and the device seconds (bench.hpp:29-70)."""
        n3 = n ** 3
        d, lv, fr, secs = np.zeros(n3), np.zeros(n3, np.int64), np.zeros(n3, np.int64), np.zeros(1)
        _check(lib().sd_grid_benchmark(self.h, C.byref(params._c()), mode, n, _ptr(d), _ptr(lv), _ptr(fr),
                                       _ptr(secs)))
        return d, lv, fr, float(secs[0])

    # -- reference caches (SDBV0001 bvh.hpp:190-236, SDWT0001 weights.hpp:700-781) --
    def save_bvh_cache(self, path: str):
        _check(lib().sd_save_bvh_cache(self.h, os.fsencode(path)))

    def load_bvh_cache(self, path: str):
        _check(lib().sd_load_bvh_cache(self.h, os.fsencode(path)))

    def save_weight_cache(self, path: str):
        _check(lib().sd_save_weight_cache(self.h, os.fsencode(path)))

    def load_weight_cache(self, path: str):
        _check(lib().sd_load_weight_cache(self.h, os.fsencode(path)))

    def smooth_min_dist_flat(self, q, params: SmoothParams) -> SmoothResults:
        """Batched smooth_min_dist_flat (smooth.hpp:189-198)."""
        return self.query_points(q, params, SD_EXACT, want_c=True, want_counters=True)


@dataclass
class RenderResult:
    """RenderResult (render.hpp:37-45)."""
    rgb: np.ndarray    # (H, W, 3) uint8, rows top to bottom
    hit_t: np.ndarray  # (H, W), -1 on miss
    leaves: int
    far_field: int
    rays: int
    hits: int
    seconds: float

    @property
    def mean_leaves_per_ray(self) -> float:
        return self.leaves / self.rays if self.rays else 0.0


def write_ppm(rgb: np.ndarray, path: str):
    """write_ppm (render.hpp:139-146)."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    _check(lib().sd_write_ppm(_ptr(rgb), rgb.shape[1], rgb.shape[0], os.fsencode(path)))


def write_png(rgb: np.ndarray, path: str):
    """write_png (render.hpp:172-203)."""
    rgb = np.ascontiguousarray(rgb, np.uint8)
    _check(lib().sd_write_png(_ptr(rgb), rgb.shape[1], rgb.shape[0], os.fsencode(path)))


def write_grid_csv(d_hat, leaves, far_field, n: int, slab_seconds, path: str):
    """write_grid_csv (bench.hpp:75-88)."""
    d = np.ascontiguousarray(d_hat, np.float64)
    lv = np.ascontiguousarray(leaves, np.int64)
    fr = np.ascontiguousarray(far_field, np.int64)
    ss = np.ascontiguousarray(slab_seconds, np.float64)
    _check(lib().sd_write_grid_csv(_ptr(d), _ptr(lv), _ptr(fr), n, _ptr(ss), os.fsencode(path)))
