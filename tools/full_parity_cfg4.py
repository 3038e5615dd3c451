"""cfg4 parity on the WHOLE 4,194,304-query batch (not a sample): the GPU
tree walk against the CPU reference (compiled, all host threads) on the
same tree and table; reports both tolerance forms and the worst queries."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP64 if "--fp64" in sys.argv else sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
wt = eng.build_weights()
eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=200.0, beta=0.5)
got = eng.smooth_min_dist(q, P)
arm = bench.CpuArm(v, w.simplices, w.kinds, wt, nodes=eng.export_bvh())
ref = arm.query(q, 200.0, 600.0, 0.5, tree=True)
print("cpu", arm.kind, arm.threads, "threads", f"{ref.seconds:.1f} s")
print("counters equal:", np.array_equal(got.leaves, ref.leaves), np.array_equal(got.far_field, ref.far_field))
s = bench.parity_stats(got.d_hat, got.grad, ref.d_hat, ref.grad, 200.0, "f64" if "--fp64" in sys.argv else "f32")
print(s)
gd = np.linalg.norm(got.grad - ref.grad, axis=1)
gn = np.linalg.norm(ref.grad, axis=1)
e = gd / np.maximum(1.0, gn)
o = np.argsort(-e)[:10]
for i in o:
    print(i, "err", e[i], "|dg|", gd[i], "|g|", gn[i], "d", ref.d_hat[i], "c", ref.c[i], "L", ref.leaves[i], "F",
          ref.far_field[i], "q", q[i])
print("queries over 1e-4 (survey):", int((e > 1e-4).sum()), "over 1e-5:", int((e > 1e-5).sum()))
