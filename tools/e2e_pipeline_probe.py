"""Host-API e2e probe: blocking sd_query_points vs sd_query_points_async
(waited per batch, and pipelined) on a BASELINE config.
  python tools/e2e_pipeline_probe.py [cfg=1|2|3|4] [steps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
mode = sd.SD_EXACT
if cfg == 1:
    w, q = configs.cfg1()
    wt = configs.weights_without_triangles(w.simplices, w.kinds, len(w.vertices))
    eng = sd.Engine(0, sd.SD_FP64)
    eng.set_geometry(w.vertices, w.simplices, w.kinds)
    eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
    P = sd.SmoothParams(alpha=50.0, beta=0.0)
elif cfg == 2:
    w, wt, q = bench.cfg2_workload()
    eng = sd.Engine(0, sd.SD_FP32)
    eng.set_geometry(configs.quantize(w.vertices), w.simplices, w.kinds)
    eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
    q = configs.quantize(q)
    P = sd.SmoothParams(alpha=100.0, beta=0.0)
else:
    w, q = configs.cfg4()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    eng = sd.Engine(0, sd.SD_FP32)
    eng.set_geometry(v, w.simplices, w.kinds)
    eng.build_weights()
    eng.build_bvh(sd.SD_BVH_AUTO)
    P = sd.SmoothParams(alpha=200.0, beta=0.5)
    mode = sd.SD_BVH
Q = len(q)
qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
outs = [sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                         torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy()) for _ in range(2)]


def timed(f):
    f(0)
    f(1)
    eng.wait()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        f(i)
    eng.wait()
    torch.cuda.synchronize()
    return 1e3 * (time.perf_counter() - t0) / steps


f0 = lambda i=0: eng.query_points(qh, P, mode, out=outs[0])
f1 = lambda i=0: eng.wait(eng.query_points_async(qh, P, mode, outs[i % 2]))
f2 = lambda i=0: eng.query_points_async(qh, P, mode, outs[i % 2])
for name, f in (("blocking", f0), ("async+wait", f1), ("pipelined", f2)):
    print(f"cfg{cfg} {name:12s} {timed(f):8.3f} ms per batch")
