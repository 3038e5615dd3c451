"""Point-query batch-size crossover between K3 (packet pair traversal, with
the slot split for small batches) and K3F (node-parallel frontier): cfg4
(5.24M triangles, GPU LBVH, beta 0.5, alpha 200), query subsets of growing
size, device-resident queries, CUDA-event timing. Run under gpurun."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
eng.build_bvh(sd.SD_BVH_LBVH)
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
rng = np.random.default_rng(0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
for n in (1024, 4096, 16384, 65536, 262144):
    sub = q[np.sort(rng.choice(len(q), n, replace=False))]
    qd = torch.tensor(sub, dtype=torch.float32, device=dev)
    d = torch.empty(n, dtype=torch.float64, device=dev)
    g = torch.empty(n, 3, dtype=torch.float64, device=dev)
    row = [f"Q={n:7d}"]
    for mode in ("0", "1"):
        os.environ["SDGPU_FRONTIER"] = mode
        for G in (("32", "8") if mode == "1" else ("-",)):
            os.environ["SDGPU_FRONTIER_G"] = G if G != "-" else ""
            run = lambda: eng.query_points_device(qd.data_ptr(), n, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(),
                                                  stream=st.cuda_stream)
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                run()
            e1.record(st)
            torch.cuda.synchronize()
            row.append(f"{'K3' if mode == '0' else 'K3F/G' + G}={e0.elapsed_time(e1) / 10:.3f}ms")
    print(" ".join(row), flush=True)
