import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import bench, paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
idx = np.array([2262542, 935228, 3684761, 3750808, 2436517, 2694089, 2937069, 2634452, 3837356, 3548417])
res = {}
for prec in (sd.SD_FP32, sd.SD_FP64):
    eng = sd.Engine(0, prec); eng.set_geometry(v, w.simplices, w.kinds); wt = eng.build_weights(); eng.build_bvh(sd.SD_BVH_AUTO)
    P = sd.SmoothParams(alpha=200.0, beta=0.5)
    variants = [("default", {})] if prec == sd.SD_FP64 else [("default", {}), ("lanes", {"SDGPU_LEAF_COOP": "0"}), ("inline", {"SDGPU_LEAF_QUEUE": "0"}), ("k3f", {"SDGPU_FRONTIER": "1"})]
    for name, env in variants:
        for k in ("SDGPU_LEAF_COOP", "SDGPU_LEAF_QUEUE", "SDGPU_FRONTIER"): os.environ.pop(k, None)
        os.environ.update(env)
        if name == "k3f":
            r = eng.smooth_min_dist(q[idx], P); g = r.grad
        else:
            r = eng.smooth_min_dist(q, P); g = r.grad[idx]
        res[("fp64" if prec else "fp32") + "_" + name] = g
    arm = bench.CpuArm(v, w.simplices, w.kinds, wt, nodes=eng.export_bvh())
    ref = arm.query(q[idx], 200.0, 600.0, 0.5, tree=True)
for k, g in res.items():
    print(k, np.round(np.linalg.norm(g - ref.grad, axis=1), 8))
