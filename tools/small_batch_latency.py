"""Per-call latency of small BVH batches through query_points_device (the
re-query loops of the callers): cfg4-like torus, Q in {256, 4096, 65536}."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
v, s = configs.torus(nu=256, nv=128)
k = np.full(len(s), 2, np.uint8)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(configs.quantize(v), s, k)
eng.build_weights()
eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=200.0, alpha_u=600.0, beta=0.5)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
rng = np.random.default_rng(1)
for Q in (256, 4096, 65536):
    q = torch.tensor(configs.quantize(rng.uniform(-1.5, 1.5, size=(Q, 3))), dtype=torch.float32, device=dev)
    d = torch.empty(Q, dtype=torch.float64, device=dev)
    g = torch.empty(Q, 3, dtype=torch.float64, device=dev)
    run = lambda: eng.query_points_device(q.data_ptr(), Q, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(), stream=st.cuda_stream)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        run()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(n):
        run()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"Q={Q}: host issue {1e6 * (t1 - t0) / n:.1f} us/call, wall {1e6 * (t2 - t0) / n:.1f} us/call, "
          f"device {1e3 * e0.elapsed_time(e1) / n:.1f} us/call, launches {eng.last_launch_count()}")
