"""Multi-GPU plumbing for the smooth-distance path (one process per GPU).

Two regimes:

* query sharding (cfg1-4): geometry, weights and tree replicated; every rank
  evaluates its own contiguous block of queries; no data-path collective.
  A fixed batch is split after a Morton sort into contiguous blocks of equal
  estimated BVH cost: shard_queries / balanced_ranges, with
  the per-query cost (popped nodes 2 (leaves + far) - 1) taken from a
  previous evaluation or a strided sample (estimate_query_costs).
* primitive sharding (cfg5): the primitives are split into Morton-contiguous
  shards (one per rank), every rank evaluates ALL queries against its shard
  and produces the unshifted fp64 partial sums (c, grad_c) of the reference
  (smooth.hpp:79-93 restricted to the shard, with the -708 mask applied per
  term); ONE all_reduce(SUM) of 4 doubles per query then gives exactly the
  whole-mesh sums, and result_from_accum (smooth.hpp:147-159) finishes.
  The WeightSet is built on the full mesh (A and sup w~ are global,
  weights.hpp:604,616) and sliced per shard. Instead of the all-reduce the
  ranks can also store their partials straight into the owner's symmetric
  buffer (sd_scatter_partials over peer memory) and each owner finalises
  its block of queries (sd_reduce_owned): owner_blocks gives the blocks.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def query_ranges(n: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced [lo, hi) query blocks, one per rank."""
    b = np.linspace(0, n, world + 1).round().astype(np.int64)
    return [(int(b[r]), int(b[r + 1])) for r in range(world)]


def balanced_ranges(cost, world: int) -> list[tuple[int, int]]:
    """Contiguous [lo, hi) blocks of a cost sequence, one per rank, each
    holding about 1/world of the total cost: rank r starts at the first
    position whose cost prefix reaches r/world of the total (each block's
    cost is within one element's cost of the even share). Zero total cost
    falls back to equal counts."""
    c = np.asarray(cost, np.float64)
    n = len(c)
    if world <= 1 or n == 0:
        return query_ranges(n, max(1, world))
    if (c < 0).any():
        raise ValueError("costs must be non-negative")
    tot = float(c.sum())
    if tot <= 0.0:
        return query_ranges(n, world)
    pre = np.concatenate([[0.0], np.cumsum(c)])  # pre[i] = cost of [0, i)
    b = [0]
    for r in range(1, world):
        # boundary i minimising |pre[i] - r tot / world|, kept monotone
        t = r * tot / world
        i = int(np.searchsorted(pre, t))
        if i > 0 and (i > n or t - pre[i - 1] <= pre[i] - t):
            i -= 1
        b.append(min(max(i, b[-1]), n))
    b.append(n)
    return [(b[r], b[r + 1]) for r in range(world)]


def morton_order(points) -> np.ndarray:
    """Query order along a 63-bit Morton curve over the batch's box (stable)."""
    p = np.asarray(points, np.float64).reshape(-1, 3)
    return np.argsort(_morton63(p), kind="stable") if len(p) else np.zeros(0, np.int64)


def estimate_query_costs(evaluate, points_sorted, stride: int = 64) -> np.ndarray:
    """Per-query BVH cost estimate for a Morton-sorted batch: `evaluate(sub)`
    returns (leaves, far_field) for a query subset (e.g. Engine.smooth_min_dist
    counters); every stride-th query is evaluated and its popped-node count
    2 (L + F) - 1 is given to the stride-long run of neighbours it starts
    (the runs are spatially compact, so the walks are alike)."""
    p = np.asarray(points_sorted, np.float64).reshape(-1, 3)
    n = len(p)
    if n == 0:
        return np.zeros(0)
    idx = np.arange(0, n, max(1, int(stride)))
    leaves, far = evaluate(p[idx])
    pops = np.maximum(2.0 * (np.asarray(leaves, np.float64) + np.asarray(far, np.float64)) - 1.0, 1.0)
    return np.repeat(pops, np.diff(np.append(idx, n)))


def shard_queries(points, world: int, cost=None):
    """Morton order + contiguous blocks of equal estimated cost (equal counts
    without a cost). cost is per query in the ORIGINAL order. Returns (order,
    ranges): rank r evaluates points[order[lo:hi]]."""
    order = morton_order(points)
    if cost is None:
        return order, query_ranges(len(order), world)
    return order, balanced_ranges(np.asarray(cost, np.float64)[order], world)


def _morton63(p: np.ndarray) -> np.ndarray:
    lo, hi = p.min(0), p.max(0)
    span = np.where(hi > lo, hi - lo, 1.0)
    c = np.clip(((p - lo) / span * 2097151.0), 0, 2097151).astype(np.uint64)

    def spread(v):
        v = v & np.uint64(0x1FFFFF)
        v = (v | (v << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
        v = (v | (v << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
        v = (v | (v << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
        v = (v | (v << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
        v = (v | (v << np.uint64(2))) & np.uint64(0x1249249249249249)
        return v

    return (spread(c[:, 0]) << np.uint64(2)) | (spread(c[:, 1]) << np.uint64(1)) | spread(c[:, 2])


@dataclass
class Shard:
    """One rank's primitive shard: a self-contained sub-mesh with its slice
    of the global WeightSet (same polynomial tables, sliced poly_index)."""
    prims: np.ndarray       # global primitive ids of this shard
    vertices: np.ndarray
    simplices: np.ndarray   # re-indexed into `vertices`
    kinds: np.ndarray
    poly_index: np.ndarray


def primitive_shards(vertices, simplices, kinds, poly_index, world: int) -> list[Shard]:
    """Morton-contiguous, equal-count primitive shards (spatially compact, so
    each shard's own tree stays tight)."""
    vertices = np.asarray(vertices, np.float64)
    simplices = np.asarray(simplices, np.int32)
    kinds = np.asarray(kinds, np.uint8)
    n = len(kinds)
    corner = simplices.copy()
    for k in (1, 2):  # unused corners -> the first corner (bbox centre unchanged)
        corner[:, k] = np.where(kinds >= k, simplices[:, k], simplices[:, 0])
    pts = vertices[corner]                                  # (n, 3, 3)
    centre = 0.5 * (pts.min(1) + pts.max(1))               # bbox centre, as bvh.hpp:45
    order = np.argsort(_morton63(centre), kind="stable") if n else np.zeros(0, np.int64)
    out = []
    for lo, hi in query_ranges(n, world):
        ids = np.sort(order[lo:hi])
        s = simplices[ids]
        k = kinds[ids]
        used = np.unique(np.concatenate([s[:, 0], s[k >= 1, 1], s[k >= 2, 2]])) if len(ids) else np.zeros(0, np.int32)
        remap = np.full(len(vertices), -1, np.int64)
        remap[used] = np.arange(len(used))
        s2 = np.where(s >= 0, remap[np.maximum(s, 0)], -1).astype(np.int32)
        out.append(Shard(ids, vertices[used], s2, k, np.asarray(poly_index, np.int32)[ids]))
    return out


def finalize(c: np.ndarray, grad_c: np.ndarray, alpha: float, epsilon: float = 1e-300):
    """result_from_accum (smooth.hpp:147-159) on summed partials (host
    mirror of sd_finalize_device, used by CPU tests)."""
    c = np.asarray(c, np.float64)
    d = np.full(c.shape, np.inf)
    g = np.zeros((len(c), 3))
    ok = c > 0.0
    d[ok] = -np.log(c[ok]) / alpha
    g[ok] = grad_c[ok] / (c[ok] + epsilon)[:, None]
    return d, g


def allreduce_partials(c, grad_c, group=None):
    """The single data-path collective of primitive sharding: SUM of the
    per-query (c, grad_c) partials over ranks. Accepts torch tensors (NCCL
    on GPU tensors, gloo on CPU tensors) and reduces them in place as one
    fused buffer."""
    import torch
    import torch.distributed as dist
    buf = torch.cat([c.reshape(-1, 1), grad_c.reshape(-1, 3)], 1).contiguous()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    c.copy_(buf[:, 0])
    grad_c.copy_(buf[:, 1:].reshape(grad_c.shape))
    return c, grad_c


def owner_blocks(n: int, world: int) -> tuple[int, list[int]]:
    """Peer-memory exchange ownership: query i belongs to rank i // per, per
    = ceil(n / world); returns per and the number of queries each rank owns."""
    per = max(1, -(-n // world))
    return per, [max(0, min(per, n - r * per)) for r in range(world)]


def exchange_reference(partials, per: int):
    """What the owners hold after every rank scattered its partials: for
    owner o, the sum over ranks (in rank order) of (c, grad_c) of its block.
    partials: list over ranks of (c (n,), grad_c (n, 3))."""
    n = len(partials[0][0])
    world = len(partials)
    out = []
    for o in range(world):
        lo, hi = o * per, min(n, (o + 1) * per)
        c = np.zeros(max(0, hi - lo))
        g = np.zeros((max(0, hi - lo), 3))
        for r in range(world):
            c = c + partials[r][0][lo:hi]
            g = g + partials[r][1][lo:hi]
        out.append((c, g))
    return out
