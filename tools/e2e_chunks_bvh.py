"""cfg4 BVH end to end through sd_query_points (pinned host buffers):
median seconds per call for SDGPU_PIPELINE chunk settings, interleaved."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
Q = len(q)
qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
res = sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                       torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy())
times = {}
for rnd in range(2):
    for ch in sys.argv[1:] or ["0", "2", "4"]:
        os.environ["SDGPU_PIPELINE"] = ch
        eng.query_points(qh, P, sd.SD_BVH, out=res)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            eng.query_points(qh, P, sd.SD_BVH, out=res)
            ts.append(time.perf_counter() - t0)
        times.setdefault(ch, []).extend(ts)
for ch, ts in times.items():
    print(f"chunks {ch}: median {np.median(ts) * 1e3:.2f} ms, {Q / np.median(ts):.3e} queries/s")
