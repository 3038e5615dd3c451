"""Seeded synthetic workloads of BASELINE.json (numpy; no dataset needed).

Shapes, sizes and value distributions follow BASELINE.json ``configs`` with
the interpretations frozen in SURVEY.md 8(d); the paper's Thingi10K corpus
is not available and these inputs stand in for it. The tests build the same
configs with the CPU oracle's mt19937_64 generators; the bench uses these
numpy generators so that its GPU leg never executes oracle code.

Also: the host-side WeightSet pieces this path needs for meshes whose
polynomials have closed forms -- valences (mesh.hpp:163-183), edge
polynomials (weights.hpp:46-76), unit weights for points -- so that a
WeightSet can be assembled without the reference toolchain.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class Workload:
    name: str
    vertices: np.ndarray   # (V, 3) float64
    simplices: np.ndarray  # (N, 3) int32, -1 padded
    kinds: np.ndarray      # (N,) uint8
    alpha: float
    alpha_u: float = 600.0
    beta: float = 0.0
    precision: int = 0     # 0 fp32, 1 fp64


@dataclass
class WeightTable:
    A: float
    sup_wtilde: float
    edge_a: np.ndarray
    tri_stored: np.ndarray
    poly_index: np.ndarray


def edge_poly(v0: int, v1: int):
    """build_edge_weight (weights.hpp:46-76): coefficients and extrema."""
    P, Q = 1.0 / v1 - 1.0 / v0, 1.0 - 1.0 / v0
    a = [1.0 / v0, 0.0, -5 * P + 16 * Q, 14 * P - 32 * Q, 16 * Q - 8 * P]
    val = lambda t: a[0] + t * (a[1] + t * (a[2] + t * (a[3] + t * a[4])))
    sup, inf = max(val(0.0), val(1.0)), min(val(0.0), val(1.0))
    qa, qb, qc = 4 * a[4], 3 * a[3], 2 * a[2]
    cands = []
    if abs(qa) > 1e-300:
        disc = qb * qb - 4 * qa * qc
        if disc >= 0:
            rt = math.sqrt(disc)
            cands = [(-qb + rt) / (2 * qa), (-qb - rt) / (2 * qa)]
    elif abs(qb) > 1e-300:
        cands = [-qc / qb]
    for t in cands:
        if 0.0 < t < 1.0:
            sup, inf = max(sup, val(t)), min(inf, val(t))
    return np.array(a), sup, inf


def weights_without_triangles(simplices: np.ndarray, kinds: np.ndarray, nverts: int) -> WeightTable:
    """build_weight_set (weights.hpp:589-621) for point/edge meshes: vertex
    valence = incident non-point simplices; edge polynomial per (v0, v1)
    valence pair in first-occurrence order; A = max valence."""
    if (kinds == 2).any():
        raise ValueError("triangle weight polynomials need the SVD/LP construction (weights.hpp:352-560)")
    val = np.zeros(nverts, np.int64)
    e = kinds == 1
    np.add.at(val, simplices[e, 0], 1)
    np.add.at(val, simplices[e, 1], 1)
    poly_index = np.full(len(kinds), -1, np.int32)
    A, sup = 1.0, 1.0
    polys, cache = [], {}
    idx = np.nonzero(e)[0]
    pairs = np.stack([val[simplices[idx, 0]], val[simplices[idx, 1]]], 1)
    uniq, first, inv = np.unique(pairs, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first)  # first-occurrence order, as the reference's cache
    rank = np.empty(len(order), np.int64)
    rank[order] = np.arange(len(order))
    for u in order:
        a, s, _ = edge_poly(int(uniq[u, 0]), int(uniq[u, 1]))
        polys.append(a)
        sup = max(sup, s)
        A = max(A, float(uniq[u].max()))
    poly_index[idx] = rank[inv.reshape(-1)]
    return WeightTable(A, sup, np.array(polys).reshape(-1, 5), np.zeros((0, 13)), poly_index)


# ------------------------------------------------------------ workloads
def cfg1(nq: int = 65536, seed: int = 1001):
    rng = np.random.default_rng(seed)
    p = rng.standard_normal((4096, 3))
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    q = np.random.default_rng(seed + 1).uniform(-2, 2, (nq, 3))
    w = Workload("cfg1 point cloud 4096 pts, exact LSE, fp64", p, np.stack(
        [np.arange(4096), -np.ones(4096), -np.ones(4096)], 1).astype(np.int32), np.zeros(4096, np.uint8),
        alpha=50.0, precision=1)
    return w, q


def cfg2(nq: int = 262144, seed: int = 2001, block: int = 0):
    """Helix x = cos t, y = sin t, z = 0.05 t, t in [0, 40 pi], 20,001
    vertices with N(0, 1e-3^2) jitter; queries uniform in the AABB scaled
    x1.2 about its centre. `block` selects a disjoint query block of the
    same distribution (per-rank blocks for weak scaling)."""
    K = 20000
    t = 40.0 * math.pi * np.arange(K + 1) / K
    v = np.stack([np.cos(t), np.sin(t), 0.05 * t], 1)
    v += np.random.default_rng(seed).normal(0.0, 1e-3, v.shape)
    s = np.stack([np.arange(K), np.arange(1, K + 1), -np.ones(K, np.int64)], 1).astype(np.int32)
    lo, hi = v.min(0), v.max(0)
    c, h = 0.5 * (lo + hi), 0.6 * (hi - lo)
    q = np.random.default_rng([seed + 1, block]).uniform(c - h, c + h, (nq, 3))
    w = Workload("cfg2 helix polyline 20,000 edges, exact LSE", v, s, np.ones(K, np.uint8), alpha=100.0)
    return w, q


def torus(major=1.0, minor=0.3, nu=512, nv=256, seed=3001, jitter=True):
    """uv_torus (shapes.hpp:67-89) + N(0, (0.1 mean edge)^2) jitter."""
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    u, vv = 2 * np.pi * i / nu, 2 * np.pi * j / nv
    ring = major + minor * np.cos(vv)
    V = np.stack([ring * np.cos(u), minor * np.sin(vv), ring * np.sin(u)], -1).reshape(-1, 3)
    vid = lambda a, b: ((a % nu) * nv + (b % nv))
    t1 = np.stack([vid(i, j), vid(i + 1, j), vid(i, j + 1)], -1).reshape(-1, 3)
    t2 = np.stack([vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)], -1).reshape(-1, 3)
    T = np.stack([t1, t2], 1).reshape(-1, 3).astype(np.int32)
    e = np.concatenate([T[:, [0, 1]], T[:, [1, 2]], T[:, [2, 0]]])
    e = np.unique(np.sort(e, 1), axis=0)
    mel = np.linalg.norm(V[e[:, 0]] - V[e[:, 1]], axis=1).mean()
    if jitter:
        V = V + np.random.default_rng(seed).normal(0.0, 0.1 * mel, V.shape)
    return V, T


def benchmark_frame(V: np.ndarray) -> np.ndarray:
    """normalize_to_benchmark_frame (mesh.hpp:126-135): scale 0.5 / bbox
    diagonal, bbox centre to (0.5, 0.5, 0.5)."""
    lo, hi = V.min(0), V.max(0)
    e = hi - lo
    diag = math.sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2])
    scale = 0.5 / diag if diag > 0 else 1.0
    return scale * V + (0.5 - scale * (0.5 * (lo + hi)))


def quantize(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.float32).astype(np.float64)


def icosphere(sub: int):
    """shapes.hpp:25-63 (midpoint subdivision, projected to the unit sphere);
    vertex numbering by sorted unique edges rather than first use."""
    t = (1.0 + math.sqrt(5.0)) / 2.0
    V = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0], [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], float)
    F = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11], [1, 5, 9], [5, 11, 4], [11, 10, 2],
                  [10, 7, 6], [7, 1, 8], [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9], [4, 9, 5],
                  [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], np.int64)
    for _ in range(sub):
        e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
        e.sort(axis=1)
        key = e[:, 0] * (len(V) + 1) + e[:, 1]
        uk, inv = np.unique(key, return_inverse=True)
        a, b = uk // (len(V) + 1), uk % (len(V) + 1)
        mid = len(V) + inv.reshape(3, -1)
        V = np.concatenate([V, 0.5 * (V[a] + V[b])])
        ab, bc, ca = mid[0], mid[1], mid[2]
        F = np.concatenate([np.stack([F[:, 0], ab, ca], 1), np.stack([F[:, 1], bc, ab], 1),
                            np.stack([F[:, 2], ca, bc], 1), np.stack([ab, bc, ca], 1)])
    V /= np.linalg.norm(V, axis=1, keepdims=True)
    return V, F.astype(np.int32)


def cfg4(nq: int = 4194304, seed: int = 4001, block: int = 0):
    """icosphere(9) (5,242,880 triangles) with radial displacement
    r <- r (1 + 0.05 sin 8 theta cos 8 phi); queries half uniform in
    [-1.5, 1.5]^3, half on the surface + normal offset N(0, 0.01^2)
    clamped to +-0.02. alpha = 200, beta = 0.5 (params.hpp:16)."""
    V, F = icosphere(9)
    r = np.linalg.norm(V, axis=1)
    th, ph = np.arccos(V[:, 2] / r), np.arctan2(V[:, 1], V[:, 0])
    V = V * (1.0 + 0.05 * np.sin(8 * th) * np.cos(8 * ph))[:, None]
    rng = np.random.default_rng([seed, block])
    h1 = nq // 2
    q1 = rng.uniform(-1.5, 1.5, (h1, 3))
    tri = rng.integers(0, len(F), nq - h1)
    r1, r2 = rng.random(nq - h1), rng.random(nq - h1)
    s = np.sqrt(r1)
    b0, b1, b2 = 1 - s, s * (1 - r2), s * r2
    a, b, c = V[F[tri, 0]], V[F[tri, 1]], V[F[tri, 2]]
    p = b0[:, None] * a + b1[:, None] * b + b2[:, None] * c
    n = np.cross(b - a, c - a)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    d = np.clip(rng.normal(0.0, 0.01, nq - h1), -0.02, 0.02)
    q = np.concatenate([q1, p + d[:, None] * n])
    w = Workload("cfg4 icosphere(9) 5,242,880 triangles, BVH far field, alpha=200, beta=0.5", V, F,
                 np.full(len(F), 2, np.uint8), alpha=200.0, beta=0.5)
    return w, q


def _rotation(rng):
    """random axis-angle rotation (shapes.hpp:121-125)"""
    ax = rng.standard_normal(3)
    ax /= np.linalg.norm(ax)
    a = rng.uniform(0.0, 2 * np.pi)
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    return np.eye(3) + np.sin(a) * K + (1 - np.cos(a)) * (K @ K)


def cfg5(nq: int = 16777216, seed: int = 5001, n_extra: int = 1000000):
    """64 randomly rotated / translated copies (centres U[-10,10]^3) of the
    cfg3 jittered torus (16,777,216 triangles), plus 1M standalone edges
    (a surface sample and that sample + mean edge length x a random tangent)
    and 1M isolated points on the surfaces; queries uniform in the scene
    AABB. alpha = 100; exact or BVH (beta = 0.5)."""
    V0, T0 = torus()
    e = np.concatenate([T0[:, [0, 1]], T0[:, [1, 2]], T0[:, [2, 0]]])
    e = np.unique(np.sort(e, 1), axis=0)
    mel = np.linalg.norm(V0[e[:, 0]] - V0[e[:, 1]], axis=1).mean()
    rng = np.random.default_rng(seed)
    Vs, Ts = [], []
    for i in range(64):
        R = _rotation(rng)
        c = rng.uniform(-10, 10, 3)
        Vs.append(V0 @ R.T + c)
        Ts.append(T0 + i * len(V0))
    V = np.concatenate(Vs)
    T = np.concatenate(Ts).astype(np.int64)
    r3 = np.random.default_rng(seed + 2)

    def sample(n):
        tri = r3.integers(0, len(T), n)
        r1, r2 = r3.random(n), r3.random(n)
        s = np.sqrt(r1)
        a, b, c = V[T[tri, 0]], V[T[tri, 1]], V[T[tri, 2]]
        p = (1 - s)[:, None] * a + (s * (1 - r2))[:, None] * b + (s * r2)[:, None] * c
        nrm = np.cross(b - a, c - a)
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        return p, nrm

    p, nrm = sample(n_extra)
    t = r3.standard_normal((n_extra, 3))
    t -= (t * nrm).sum(1, keepdims=True) * nrm
    t /= np.linalg.norm(t, axis=1, keepdims=True)
    pe = p + mel * t
    pts, _ = sample(n_extra)
    nv = len(V)
    V = np.concatenate([V, p, pe, pts])
    E = np.stack([nv + np.arange(n_extra), nv + n_extra + np.arange(n_extra), -np.ones(n_extra, np.int64)], 1)
    P = np.stack([nv + 2 * n_extra + np.arange(n_extra), -np.ones(n_extra, np.int64), -np.ones(n_extra, np.int64)], 1)
    S = np.concatenate([T, E, P]).astype(np.int32)
    K = np.concatenate([np.full(len(T), 2), np.full(n_extra, 1), np.zeros(n_extra)]).astype(np.uint8)
    lo, hi = V.min(0), V.max(0)
    q = np.random.default_rng(seed + 1).uniform(lo, hi, (nq, 3))
    w = Workload("cfg5 64 tori (16.8M triangles) + 1M edges + 1M points", V, S, K, alpha=100.0, beta=0.5)
    return w, q


def terrain_bunny(seed: int = 6001):
    """Stand-ins for the paper's simulation row "Terrain (lidar points,
    6,591,087, alpha 100) vs Bunny (points, 3,485, alpha_q 20)"
    (PAPER.md:1378-1397): a lidar-like height-field point cloud over a
    10 x 10 patch (smooth hill + ripples + N(0, 0.01^2) noise) and a
    3,485-point bumpy closed blob resting just above the hill top."""
    rng = np.random.default_rng(seed)
    n = 6591087
    xy = rng.uniform(0.0, 10.0, (n, 2))

    def height(x, y):
        return 1.5 * np.exp(-((x - 5) ** 2 + (y - 5) ** 2) / 8.0) + 0.05 * np.sin(3 * x) * np.cos(2 * y)

    terrain = np.column_stack([xy, height(xy[:, 0], xy[:, 1]) + rng.normal(0, 0.01, n)])
    m = 3485
    d = rng.standard_normal((m, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = 0.5 * (1 + 0.1 * np.sin(5 * d[:, 0]) * np.cos(4 * d[:, 1]))
    bunny = d * r[:, None] * np.array([1.0, 0.8, 0.9])
    bunny += np.array([5.0, 5.0, height(5.0, 5.0) + 0.5 * 0.9 * 1.1 + 0.02]) - np.array([0, 0, 0])
    return terrain, bunny
