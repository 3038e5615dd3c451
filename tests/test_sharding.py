"""Multi-process (world size 2, gloo, CPU) tests of the multi-GPU host logic:
query sharding is a pure partition; primitive sharding merges per-shard
unshifted fp64 partials with one all_reduce(SUM) and must reproduce the
whole-mesh reference result. Per-shard partials come from the CPU oracle
(exactly the quantities the GPU writes through sd_query_points_device), so
these tests cover the plumbing that the 8-GPU runs use."""
import os
import socket

import numpy as np
import pytest

from paper_2108_10480_b200 import sharding


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_query_ranges_partition():
    for n in (0, 1, 7, 1000, 262144):
        for w in (1, 2, 3, 8):
            r = sharding.query_ranges(n, w)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [hi - lo for lo, hi in r]
            assert max(sizes) - min(sizes) <= 1


def test_balanced_ranges_split_cost_evenly():
    rng = np.random.default_rng(3)
    for n in (1, 5, 100, 10000):
        for w in (1, 2, 3, 8):
            for cost in (np.ones(n), rng.exponential(1.0, n), rng.integers(0, 3, n).astype(float),
                         np.where(np.arange(n) < n // 3, 50.0, 1.0)):
                r = sharding.balanced_ranges(cost, w)
                assert len(r) == w and r[0][0] == 0 and r[-1][1] == n
                assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(r, r[1:]))
                if cost.sum() > 0:
                    share = cost.sum() / w
                    for lo, hi in r:  # within one element of the even share
                        assert abs(cost[lo:hi].sum() - share) <= cost.max() * (1 + 1e-12) * 2
    # uniform costs reproduce the equal-count split up to rounding
    r = sharding.balanced_ranges(np.ones(1000), 8)
    assert [hi - lo for lo, hi in r] == [125] * 8
    assert sharding.balanced_ranges(np.zeros(10), 3) == sharding.query_ranges(10, 3)
    with pytest.raises(ValueError):
        sharding.balanced_ranges(np.array([1.0, -1.0]), 2)


def test_cost_estimate_and_shard_queries(oracle):
    """The strided estimate from the oracle's counters (the GPU returns the
    same counters) balances the measured popped nodes across ranks much
    better than equal counts on a half-near / half-far batch."""
    O = oracle
    m = O.random_scene(11, 300)
    rng = np.random.default_rng(7)
    near = O.QueryStream(77).draw_points(m, 600)
    lo, hi = m.vertices.min(0), m.vertices.max(0)
    span = hi - lo
    # a far cloud off to one side: Morton-contiguous cheap queries
    far = rng.uniform(lo + span * np.array([4.0, 0.0, 0.0]), hi + span * np.array([5.0, 0.0, 0.0]), size=(600, 3))
    q = np.concatenate([near, far])
    w, t = O.Weights.build(m), O.Tree.build(m)
    p = O.Params(alpha=100.0, beta=0.5)
    ref = O.query(m, w, q, p, tree=t)
    true_cost = 2.0 * (ref.leaves + ref.far_field) - 1.0
    order = sharding.morton_order(q)

    def evaluate(sub):
        r = O.query(m, w, sub, p, tree=t)
        return r.leaves, r.far_field

    est_sorted = sharding.estimate_query_costs(evaluate, q[order], stride=8)
    assert est_sorted.shape == (len(q),)
    est = np.empty(len(q))
    est[order] = est_sorted
    o2, ranges = sharding.shard_queries(q, 4, cost=est)
    assert np.array_equal(o2, order)
    assert np.array_equal(np.sort(np.concatenate([order[a:b] for a, b in ranges])), np.arange(len(q)))
    bal = [true_cost[order[a:b]].sum() for a, b in ranges]
    _, eq = sharding.shard_queries(q, 4)
    flat = [true_cost[order[a:b]].sum() for a, b in eq]
    assert max(bal) / np.mean(bal) < max(flat) / np.mean(flat)
    assert max(bal) / np.mean(bal) < 1.25


def test_primitive_shards_cover_mesh(oracle):
    m = oracle.random_scene(5, 200)
    w = oracle.Weights.build(m).table
    shards = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, w.poly_index, 3)
    ids = np.sort(np.concatenate([s.prims for s in shards]))
    assert np.array_equal(ids, np.arange(m.num_simplices))
    for s in shards:
        # the sub-mesh reproduces the global corners of each primitive
        for j, g in enumerate(s.prims):
            for k in range(int(m.kinds[g]) + 1):
                assert np.array_equal(s.vertices[s.simplices[j, k]], m.vertices[m.simplices[g, k]])
        assert np.array_equal(s.poly_index, w.poly_index[s.prims])


def _worker(rank, world, port, seed, beta, results):
    import torch
    import torch.distributed as dist

    import oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = O.random_scene(seed, 200)
    wt = O.Weights.build(m).table  # global WeightSet (A, sup w~ are global)
    shard = sharding.primitive_shards(m.vertices, m.simplices, m.kinds, wt.poly_index, world)[rank]
    sm = O.Mesh.from_arrays(shard.vertices, shard.simplices, shard.kinds)
    sw = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, shard.poly_index))
    q = O.QueryStream(900 + seed).draw_points(m, 120)
    p = O.Params(alpha=100.0, beta=beta)
    tree = O.Tree.build(sm) if beta > 0 else None   # one tree per shard
    r = O.query(sm, sw, q, p, tree=tree)
    c, gc = torch.tensor(r.c), torch.tensor(r.grad_c)
    sharding.allreduce_partials(c, gc)
    d, g = sharding.finalize(c.numpy(), gc.numpy(), p.alpha, p.epsilon)
    if rank == 0:
        results.put((d, g, q))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("seed", [3, 8])
def test_primitive_sharded_merge_gloo(oracle, seed):
    """beta = 0: the merged result equals the whole-mesh flat oracle to fp64
    rounding (sums re-associated across shards)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, 0.0, results)) for r in range(2)]
    for pr in procs:
        pr.start()
    d, g, q = results.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    m = oracle.random_scene(seed, 200)
    w = oracle.Weights.build(m)
    ref = oracle.query(m, w, q, oracle.Params(alpha=100.0, beta=0.0))
    fin = np.isfinite(ref.d_hat)
    assert (np.isfinite(d) == fin).all()
    assert np.abs(d[fin] - ref.d_hat[fin]).max() <= 1e-12 * max(1.0, np.abs(ref.d_hat[fin]).max())
    assert np.abs(g - ref.grad).max() <= 1e-11


def test_primitive_sharded_bvh_is_conservative_gloo(oracle):
    """beta > 0 with one tree per shard (the cfg5 BVH semantics): the merged
    field stays below the exact one (acceptance [1] carried over)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    results = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 4, 0.5, results)) for r in range(2)]
    for pr in procs:
        pr.start()
    d, g, q = results.get(timeout=300)
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    m = oracle.random_scene(4, 200)
    ref = oracle.query(m, oracle.Weights.build(m), q, oracle.Params(alpha=100.0, beta=0.0))
    assert (d <= ref.d_hat + 1e-9).all()



def test_owner_blocks_cover_every_query_once():
    from paper_2108_10480_b200 import sharding
    for n, world in ((0, 1), (1, 8), (7, 8), (1000, 3), (16777216, 8), (5, 2)):
        per, counts = sharding.owner_blocks(n, world)
        assert sum(counts) == n and len(counts) == world
        assert all(0 <= c <= per for c in counts)
        assert per * world >= n
        owners = [i // per for i in range(min(n, 50))]
        assert all(0 <= o < world for o in owners)
