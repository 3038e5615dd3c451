"""Seeded stand-ins for the paper's mesh-to-mesh timing table
("Avg. Dist Time (ms)", 28 CPU threads): one data mesh
M and one query mesh Mq per row, with the row's primitive TYPES and COUNTS
|F|, |F_q| and its alpha / alpha_q. The real meshes (bowl, bunny, octopus,
lidar terrain, city street, ...) are not available; these shapes keep the
sizes and put the query mesh in near-contact with the data mesh, as in the
simulations the rows were timed on. beta is the reference default 0.5
(params.hpp:16).

Each generator returns a Row; meshes are (vertices (V,3) float64,
simplices (N,3) int32 with -1 padding, kinds (N,) uint8).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .configs import icosphere

POINT, EDGE, TRI = 0, 1, 2


@dataclass
class MeshArrays:
    vertices: np.ndarray
    simplices: np.ndarray
    kinds: np.ndarray

    @property
    def n(self) -> int:
        return len(self.kinds)


@dataclass
class Row:
    name: str
    data: MeshArrays
    query: MeshArrays
    alpha: float
    alpha_q: float
    paper_ms: float
    types: str  # "M type / Mq type"


def _mesh(V, simplices_by_kind):
    S, K = [], []
    for kind, arr in simplices_by_kind:
        arr = np.asarray(arr, np.int32).reshape(-1, kind + 1)
        pad = np.full((len(arr), 3), -1, np.int32)
        pad[:, : kind + 1] = arr
        S.append(pad)
        K.append(np.full(len(arr), kind, np.uint8))
    return MeshArrays(np.ascontiguousarray(V, np.float64), np.concatenate(S), np.concatenate(K))


def _points(P):
    return _mesh(P, [(POINT, np.arange(len(P)))])


def _unique_edges(F):
    e = np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]])
    e.sort(axis=1)
    return np.unique(e, axis=0)


def _closed_blob(nv, rng, scale=(1.0, 1.0, 1.0), bumps=0.1):
    """Closed genus-0 triangle mesh with exactly nv vertices and 2 nv - 4
    triangles (convex hull of points on the sphere), radially bumped."""
    from scipy.spatial import ConvexHull
    d = rng.standard_normal((nv, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    F = ConvexHull(d).simplices.astype(np.int32)
    assert len(F) == 2 * nv - 4
    r = 1.0 + bumps * np.sin(5 * d[:, 0]) * np.cos(4 * d[:, 1]) * np.sin(3 * d[:, 2] + 1)
    return d * r[:, None] * np.asarray(scale), F


def _bowl_edges():
    """Hemispherical bowl wireframe: 12 latitude rings x 32 + 11 x 32 meridian
    segments = 736 edges (radius 1, open at z = 0)."""
    nl, nr = 32, 12
    th = np.linspace(0.15 * math.pi, 0.5 * math.pi, nr)  # polar angle from -z
    ph = np.arange(nl) * 2 * math.pi / nl
    V = np.array([[math.sin(t) * math.cos(p), math.sin(t) * math.sin(p), -math.cos(t)] for t in th for p in ph])
    idx = lambda i, j: i * nl + (j % nl)
    E = [(idx(i, j), idx(i, j + 1)) for i in range(nr) for j in range(nl)]
    E += [(idx(i, j), idx(i + 1, j)) for i in range(nr - 1) for j in range(nl)]
    return V, np.array(E)


def row_bowl_icosphere(seed=7001):
    V, E = _bowl_edges()
    Vi, Fi = icosphere(1)
    Ei = _unique_edges(Fi)  # 120 edges
    Vi = Vi * 0.25 + np.array([0.0, 0.0, -1.0 + 0.25 + 0.03])
    return Row("Bowl vs Icosphere", _mesh(V, [(EDGE, E)]), _mesh(Vi, [(EDGE, Ei)]), 50.0, 50.0, 2.72934,
               "Edges 736 / Edges 120")


def row_bowl_spiky(seed=7002):
    V, E = _bowl_edges()
    Vi, Fi = icosphere(2)  # 162 vertices, 320 triangles, 480 edges
    Ei = _unique_edges(Fi)
    Vi = Vi * 0.2
    tips = Vi * 1.6
    tips2 = Vi[:4] * 2.0
    Vq = np.concatenate([Vi, tips, tips2]) + np.array([0.0, 0.0, -1.0 + 0.32 + 0.03])
    n = len(Vi)
    spikes = np.stack([np.arange(n), n + np.arange(n)], 1)
    spikes2 = np.stack([n + np.arange(4), 2 * n + np.arange(4)], 1)
    q = _mesh(Vq, [(TRI, Fi), (EDGE, np.concatenate([Ei, spikes, spikes2]))])
    assert q.n == 966
    return Row("Bowl vs Spiky Sphere", _mesh(V, [(EDGE, E)]), q, 50.0, 20.0, 34.7789, "Edges 736 / Tris+Edges 966")


def _terrain(rng, n=6591087):
    xy = rng.uniform(0.0, 10.0, (n, 2))
    h = lambda x, y: 1.5 * np.exp(-((x - 5) ** 2 + (y - 5) ** 2) / 8.0) + 0.05 * np.sin(3 * x) * np.cos(2 * y)
    return np.column_stack([xy, h(xy[:, 0], xy[:, 1]) + rng.normal(0, 0.01, n)]), h


def row_terrain_bunny(seed=6001):
    """The point-cloud row (same construction as configs.terrain_bunny)."""
    from .configs import terrain_bunny
    T, B = terrain_bunny(seed)
    return Row("Terrain vs Bunny", _points(T), _points(B), 100.0, 20.0, 250.0031, "Points 6591087 / Points 3485")


def _octopus(rng):
    """Body: 32 x 34 latitude-longitude sphere (2112 triangles) + 8 tentacle
    tubes of 5 x 29 quads (8 x 290 triangles) = 4432 triangles."""
    F, V = [], []
    nu, nv = 32, 34  # body: nv latitude bands incl. the two pole fans
    top = [0.0, 0.0, 1.0]
    V.append(top)
    for i in range(1, nv):
        t = math.pi * i / nv
        for j in range(nu):
            p = 2 * math.pi * j / nu
            V.append([math.sin(t) * math.cos(p), math.sin(t) * math.sin(p), math.cos(t)])
    V.append([0.0, 0.0, -1.0])
    ring = lambda i, j: 1 + (i - 1) * nu + (j % nu)
    bot = len(V) - 1
    for j in range(nu):
        F.append([0, ring(1, j), ring(1, j + 1)])
        F.append([bot, ring(nv - 1, j + 1), ring(nv - 1, j)])
    for i in range(1, nv - 1):
        for j in range(nu):
            a, b, c, d = ring(i, j), ring(i, j + 1), ring(i + 1, j), ring(i + 1, j + 1)
            F += [[a, c, b], [b, c, d]]
    assert len(F) == 2112
    for k in range(8):  # tentacles: open tubes hanging below the body
        ang = 2 * math.pi * k / 8
        base = len(V)
        for s in range(30):
            z = -0.6 - 0.05 * s
            cx, cy = (0.5 + 0.04 * s) * math.cos(ang), (0.5 + 0.04 * s) * math.sin(ang)
            r = 0.12 * (1 - s / 40)
            for j in range(5):
                p = 2 * math.pi * j / 5
                V.append([cx + r * math.cos(p), cy + r * math.sin(p), z])
        for s in range(29):
            for j in range(5):
                a, b = base + s * 5 + j, base + s * 5 + (j + 1) % 5
                c, d = a + 5, b + 5
                F += [[a, c, b], [b, c, d]]
    V = np.array(V) * 0.5
    return V, np.array(F)


def row_terrain_octopus(seed=7004):
    rng = np.random.default_rng(seed)
    T, h = _terrain(rng)
    V, F = _octopus(rng)
    V = V + np.array([5.0, 5.0, h(5.0, 5.0) - V[:, 2].min() + 0.02])
    q = _mesh(V, [(TRI, F)])
    assert q.n == 4432
    return Row("Terrain vs Octopus", _points(T), q, 100.0, 1000.0, 189.5989, "Points 6591087 / Tris 4432")


def row_bunny_bunny(seed=7005):
    rng = np.random.default_rng(seed)
    V, F = _closed_blob(3485, rng, (0.5, 0.4, 0.45))
    V2 = V + np.array([1.0 + 0.03, 0.0, 0.0])
    return Row("Bunny vs Bunny", _mesh(V, [(TRI, F)]), _mesh(V2, [(TRI, F)]), 200.0, 200.0, 92.5717,
               "Tris 6966 / Tris 6966")


def row_plane_bunny(seed=7006):
    rng = np.random.default_rng(seed)
    n = 21
    x, y = np.meshgrid(np.linspace(-2, 2, n), np.linspace(-2, 2, n), indexing="ij")
    z = 0.1 * np.sin(2 * x) * np.cos(2 * y)
    Vp = np.column_stack([x.ravel(), y.ravel(), z.ravel()])
    F = []
    for i in range(n - 1):
        for j in range(n - 1):
            a, b, c, d = i * n + j, i * n + j + 1, (i + 1) * n + j, (i + 1) * n + j + 1
            F += [[a, c, b], [b, c, d]]
    V, Fb = _closed_blob(3485, rng, (0.5, 0.4, 0.45))
    V = V + np.array([0.0, 0.0, 0.1 - V[:, 2].min() + 0.02])
    return Row("Bumpy Plane vs Bunny", _mesh(Vp, [(TRI, F)]), _mesh(V, [(TRI, Fb)]), 200.0, 200.0, 470.3857,
               "Tris 800 / Tris 6966")


def row_slide_sphere(seed=7007):
    """Slide: 5 parallel curved rails of 123 segments (615 edges); sphere:
    convex hull of 482 points (960 triangles) resting on the rails."""
    rng = np.random.default_rng(seed)
    s = np.linspace(0, 1, 124)
    V, E = [], []
    for k in range(5):
        y = -0.4 + 0.2 * k
        base = len(V)
        for t in s:
            V.append([4 * t, y + 0.05 * (k - 2) ** 2, 2 * (1 - t) ** 2])
        E += [(base + i, base + i + 1) for i in range(123)]
    Vs, Fs = _closed_blob(482, rng, (0.3, 0.3, 0.3), bumps=0.0)
    Vs = Vs + np.array([1.0, 0.0, 2 * (1 - 0.25) ** 2 + 0.35])
    return Row("Slide vs Sphere", _mesh(np.array(V), [(EDGE, E)]), _mesh(Vs, [(TRI, Fs)]), 100.0, 100.0, 33.5601,
               "Edges 615 / Tris 960")


def row_ringtoss_trefoil(seed=7008):
    """Ring toss: 12,400 points on a peg (cylinder) and its base disc;
    trefoil: closed 100-edge trefoil knot around the peg."""
    rng = np.random.default_rng(seed)
    n1 = 6200
    th, z = rng.uniform(0, 2 * math.pi, n1), rng.uniform(0, 1.5, n1)
    peg = np.column_stack([0.1 * np.cos(th), 0.1 * np.sin(th), z])
    r, th2 = 1.2 * np.sqrt(rng.uniform(0, 1, 12400 - n1)), rng.uniform(0, 2 * math.pi, 12400 - n1)
    base = np.column_stack([r * np.cos(th2), r * np.sin(th2), np.zeros_like(r)])
    t = np.arange(100) * 2 * math.pi / 100
    knot = np.column_stack([np.sin(t) + 2 * np.sin(2 * t), np.cos(t) - 2 * np.cos(2 * t), -np.sin(3 * t)]) * 0.12
    knot += np.array([0.0, 0.0, 0.8])
    E = np.stack([np.arange(100), (np.arange(100) + 1) % 100], 1)
    return Row("Ring Toss vs Trefoil", _points(np.concatenate([peg, base])), _mesh(knot, [(EDGE, E)]), 20.0, 20.0,
               1.4727, "Points 12400 / Edges 100")


def row_street_motorcycle(seed=7009):
    """City street: 6,747,648 lidar-like points (road plane + curbs +
    building facades); motorcycle: closed 8800-triangle elongated hull
    resting on the road."""
    rng = np.random.default_rng(seed)
    n = 6747648
    k = rng.uniform(0, 1, n)
    x = rng.uniform(-20, 20, n)
    y = np.where(k < 0.6, rng.uniform(-4, 4, n), np.where(k < 0.8, rng.choice([-6.0, 6.0], n), rng.uniform(-4, 4, n)))
    z = np.where(k < 0.6, 0.0, np.where(k < 0.8, rng.uniform(0, 8, n), 0.15))
    y = np.where(k >= 0.8, np.sign(y + 1e-9) * 4.0 + 0.0 * y, y)
    P = np.column_stack([x, y, z + rng.normal(0, 0.01, n)])
    V, F = _closed_blob(4402, rng, (1.0, 0.3, 0.5))
    V = V + np.array([0.0, 0.0, -V[:, 2].min() + 0.03])
    return Row("City Street vs Motorcycle", _points(P), _mesh(V, [(TRI, F)]), 50.0, 100.0, 581.2362,
               "Points 6747648 / Tris 8800")


ROWS = {
    "bowl_icosphere": row_bowl_icosphere,
    "bowl_spiky": row_bowl_spiky,
    "terrain_bunny": row_terrain_bunny,
    "terrain_octopus": row_terrain_octopus,
    "bunny_bunny": row_bunny_bunny,
    "plane_bunny": row_plane_bunny,
    "slide_sphere": row_slide_sphere,
    "ringtoss_trefoil": row_ringtoss_trefoil,
    "street_motorcycle": row_street_motorcycle,
}
