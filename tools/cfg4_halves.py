"""cfg4: K3 time on the uniform half, the near-surface half, and both mixed
(Morton-sorted together) -- does mixing the two populations in a packet cost
lane occupancy?"""
import os, sys
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
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
half = len(q) // 2
def t(sub):
    qd = torch.tensor(sub, dtype=torch.float32, device=dev); n = len(sub)
    d = torch.empty(n, dtype=torch.float64, device=dev); g = torch.empty(n, 3, dtype=torch.float64, device=dev)
    run = lambda: eng.query_points_device(qd.data_ptr(), n, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(), stream=st.cuda_stream)
    for _ in range(2): run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(5): run()
    e1.record(st); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5
a, b, c = t(q[:half]), t(q[half:]), t(q)
print(f"uniform half {a:.2f} ms, near half {b:.2f} ms, sum {a+b:.2f} ms, mixed {c:.2f} ms")
