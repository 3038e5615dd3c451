"""Exact cfg2 end to end through sd_query_points (pinned host buffers):
median seconds per call for SDGPU_PIPELINE chunk settings, interleaved."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2108_10480_b200 as sd
w, v, q, wt = bench.workload(0, 2, None, 0)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
P = sd.SmoothParams(alpha=bench.ALPHA, alpha_u=600.0, beta=0.0)
Q = len(q)
qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
res = sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                       torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy())
times = {}
for rnd in range(3):
    for ch in sys.argv[1:] or ["0", "2"]:
        os.environ["SDGPU_PIPELINE"] = ch
        eng.query_points(qh, P, sd.SD_EXACT, out=res)
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            eng.query_points(qh, P, sd.SD_EXACT, out=res)
            ts.append(time.perf_counter() - t0)
        times.setdefault(ch, []).extend(ts)
for ch, ts in times.items():
    print(f"chunks {ch}: median {np.median(ts) * 1e3:.3f} ms, {Q * len(w.kinds) / np.median(ts):.3e} pair-evals/s")
