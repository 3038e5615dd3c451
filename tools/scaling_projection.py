"""Projected strong scaling of the BVH leg (cfg4) from ONE GPU: the bench's
own split of the fixed 4,194,304-query batch into N Hilbert-contiguous
blocks of equal estimated cost (sharding.morton_order +
estimate_query_costs + balanced_ranges, exactly as bench.py does at N
ranks), each block timed alone on the GPU (CUDA events, median of 5). The
projection is T(1) / max_r T(block r): what N GPUs would reach if each ran
its block at the single-GPU rate (no collective on this path). Compared
with the interleaved-packet split of sd_query_points_device_shard (rank r
walks packets r, r + N, ... of the whole sorted batch). A projection, not a
multi-GPU measurement.
  python tools/scaling_projection.py [N ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs, sharding  # noqa: E402

Ns = [int(x) for x in sys.argv[1:]] or [2, 4, 8]
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


QD = torch.tensor(q, dtype=torch.float32, device=dev)
D = torch.empty(len(q), dtype=torch.float64, device=dev)
G = torch.empty(len(q), 3, dtype=torch.float64, device=dev)


def time_shard(N, r, reps=5):
    """rank r's interleaved packets of the whole batch (sd_query_points_device_shard)"""
    run = lambda: eng.query_points_device_shard(QD.data_ptr(), len(q), P, N, r, D.data_ptr(), G.data_ptr(),
                                                stream=st.cuda_stream)
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def time_block(qb, reps=5):
    n = len(qb)
    qd = torch.tensor(qb, dtype=torch.float32, device=dev)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    g = torch.empty(n, 3, dtype=torch.float64, device=dev)
    run = lambda: eng.query_points_device(qd.data_ptr(), n, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(),
                                          stream=st.cuda_stream)
    for _ in range(3):
        run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run()
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


t1 = time_block(q)
out = {"workload": "cfg4, 4,194,304 queries, the bench's cost-balanced Hilbert split", "t1_ms": t1, "projection": {}}


def counters(sub):
    r = eng.smooth_min_dist(sub, P)
    return r.leaves, r.far_field


order = sharding.morton_order(q)
est = sharding.estimate_query_costs(counters, q[order], stride=64)
for N in Ns:
    ranges = sharding.balanced_ranges(est, N)
    tb = [time_block(np.ascontiguousarray(q[order[lo:hi]])) for lo, hi in ranges]
    eq = sharding.query_ranges(len(q), N)
    te = [time_block(np.ascontiguousarray(q[order[lo:hi]])) for lo, hi in eq]
    chunks = {}
    for C in (1, 16, 64, 256, 1024):
        os.environ["SDGPU_SHARD_CHUNK"] = str(C)
        tc = [time_shard(N, r) for r in range(N)]
        chunks[C] = {"max_ms": max(tc), "speedup": t1 / max(tc)}
    os.environ.pop("SDGPU_SHARD_CHUNK", None)
    ti = [time_shard(N, r) for r in range(N)]
    out["projection"][N] = {"interleaved_packets": {"rank_ms": ti, "max_ms": max(ti), "speedup": t1 / max(ti),
                                                    "efficiency": t1 / (N * max(ti)), "by_chunk": chunks},
                            "cost_balanced_blocks": {"block_ms": tb, "max_ms": max(tb), "speedup": t1 / max(tb),
                                                     "efficiency": t1 / (N * max(tb))},
                            "equal_count_blocks": {"max_ms": max(te), "speedup": t1 / max(te)}}
    print(N, json.dumps(out["projection"][N]), flush=True)
print(json.dumps(out))
