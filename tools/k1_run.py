"""One exact pass of a BASELINE config on cuda:0 (ncu target for K1):
  python tools/k1_run.py [cfg=3] [alpha=100] [queries]
K1_TIME=reps times it; K1_PRUNE=bits turns the pruned evaluation on."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
alpha = float(sys.argv[2]) if len(sys.argv) > 2 else 100.0
if cfg == 3:
    v, t, k, q = bench.cfg3_workload()
    eng = sd.Engine(0, sd.SD_FP32)
    eng.set_geometry(v, t, k)
    eng.build_weights()
else:
    w, wt, q = bench.cfg2_workload()
    from paper_2108_10480_b200 import configs
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    eng = sd.Engine(0, sd.SD_FP32)
    eng.set_geometry(v, w.simplices, w.kinds)
    eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
if len(sys.argv) > 3:
    q = q[: int(sys.argv[3])]
dev = torch.device("cuda", 0)
qd = torch.tensor(q, dtype=torch.float32, device=dev)
d = torch.empty(len(q), dtype=torch.float64, device=dev)
g = torch.empty(len(q), 3, dtype=torch.float64, device=dev)
P = sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=0.0)
if os.environ.get("K1_PRUNE"):  # sd_set_exact_pruning bits
    eng.set_exact_pruning(float(os.environ["K1_PRUNE"]))
run = lambda: eng.query_points_device(qd.data_ptr(), len(q), P, sd.SD_EXACT, d.data_ptr(), g.data_ptr())
for _ in range(2):
    run()
torch.cuda.synchronize()
if os.environ.get("K1_TIME"):
    reps = int(os.environ["K1_TIME"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cfg{cfg} alpha {alpha:g}: {ms:.3f} ms/step, {len(q) * eng.num_simplices / (ms * 1e-3):.4e} pair-evals/s")
print("ok", float(d[:4].sum()))
