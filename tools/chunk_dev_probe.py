import os, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32); eng.set_geometry(v, w.simplices, w.kinds); eng.build_weights(); eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
dev = torch.device('cuda', 0); st = torch.cuda.current_stream(dev)
Q = len(q); qd = torch.tensor(q, dtype=torch.float32, device=dev)
d = torch.empty(Q, dtype=torch.float64, device=dev); g = torch.empty(Q, 3, dtype=torch.float64, device=dev)
for nch in (1, 2, 4, 8):
    per = Q // nch
    ts = []
    for k in range(nch):
        run = lambda: eng.query_points_device(qd[k*per:].data_ptr(), per, P, sd.SD_BVH, d[k*per:].data_ptr(), g[k*per:].data_ptr(), stream=st.cuda_stream)
        run(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); run(); e1.record(st); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(nch, 'chunks: per-chunk ms', [round(t, 2) for t in ts], 'sum', round(sum(ts), 2))
