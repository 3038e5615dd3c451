"""fp64 exact triangle kernel (cfg3 torus, weighted) on a query subset:
ms per evaluation for the SDGPU_FP64_QPT / SDGPU_FP64_MINB setting in the
environment. Usage: python tools/fp64_tri_sweep.py [nq]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
nq = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
v, s = configs.torus()
k = np.full(len(s), 2, dtype=np.uint8)
rng = np.random.default_rng(3002)
lo, hi = v.min(0) - 0.5, v.max(0) + 0.5
q = rng.uniform(lo, hi, size=(nq, 3))
eng = sd.Engine(0, sd.SD_FP64)
eng.set_geometry(v, s, k)
eng.build_weights()
P = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=0.0)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
qd = torch.tensor(q, dtype=torch.float64, device=dev)
d = torch.empty(nq, dtype=torch.float64, device=dev)
g = torch.empty(nq, 3, dtype=torch.float64, device=dev)
run = lambda: eng.query_points_device(qd.data_ptr(), nq, P, sd.SD_EXACT, d.data_ptr(), g.data_ptr(), stream=st.cuda_stream)
for _ in range(2):
    run()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(3):
    run()
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
pairs = nq * len(s)
print(f"qpt={os.environ.get('SDGPU_FP64_QPT', '-')} minb={os.environ.get('SDGPU_FP64_MINB', '-')} "
      f"{nq} x {len(s)} tris fp64: {ms:.2f} ms, {pairs / ms * 1e3:.3e} pair-evals/s, dsum {float(d.sum()):.12e}")
