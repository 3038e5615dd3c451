"""Where a query-sharded cfg4 call spends its time: rank 0 of N (N = 1, 8)
through sd_query_points_device_shard, CUDA events around the whole call and
(sd_set_kernel_timing) around the traversal launch alone, median of 5 with
L2 flushed. Run bare for the timings, under ncu --metrics
gpu__time_duration.sum for the per-kernel list (sort, traversal, finalize).
  python tools/shard_breakdown.py [N ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

Ns = [int(x) for x in sys.argv[1:]] or [1, 8]
reps = int(os.environ.get("REPS", "5"))
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
eng.set_kernel_timing(True)
out = {}
for N in Ns:
    for r in ([0] if N == 1 else [0, N - 1]):
        run = (lambda: eng.query_points_device(QD.data_ptr(), len(q), P, sd.SD_BVH, D.data_ptr(), G.data_ptr(),
                                               stream=st.cuda_stream)) if N == 1 else \
              (lambda: eng.query_points_device_shard(QD.data_ptr(), len(q), P, N, r, D.data_ptr(), G.data_ptr(),
                                                     stream=st.cuda_stream))
        for _ in range(2):
            run()
        eng.kernel_times()
        tc, tk = [], []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            run()
            b.record(st)
            torch.cuda.synchronize()
            tc.append(a.elapsed_time(b))
            tk.append(sum(eng.kernel_times()))
        out[f"N{N}_r{r}"] = {"call_ms": float(np.median(tc)), "traversal_ms": float(np.median(tk))}
        print(N, r, out[f"N{N}_r{r}"], flush=True)
print(json.dumps(out))
