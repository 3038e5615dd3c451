import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench, oracle as O
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32); eng.set_geometry(v, w.simplices, w.kinds); wt = eng.build_weights(); eng.build_bvh(sd.SD_BVH_AUTO)
half = len(q)//2
idx = np.concatenate([np.linspace(0, half-1, 32768), np.linspace(half, len(q)-1, 32768)]).astype(np.int64)
P = sd.SmoothParams(alpha=200.0, beta=0.5)
got = eng.smooth_min_dist(q[idx], P)
Om, Ow, Ot = bench.oracle_objects(v, w.simplices, w.kinds, wt, eng.export_bvh())[1:]
ref = O.query(Om, Ow, q[idx], O.Params(alpha=200.0, beta=0.5), tree=Ot)
gd = np.linalg.norm(got.grad - ref.grad, axis=1); gn = np.linalg.norm(ref.grad, axis=1)
e = gd / np.maximum(gn, 1e-3)
o = np.argsort(-e)[:8]
for i in o: print(i, "err", e[i], "|dg|", gd[i], "|g|", gn[i], "d", ref.d_hat[i], "c", ref.c[i], "leaves", ref.leaves[i], "far", ref.far_field[i])
print("grad norm quantiles", np.quantile(gn, [0, 0.001, 0.01, 0.5]))
