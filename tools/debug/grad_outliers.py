"""Localise the cfg4 fp32 gradient outliers (tools/grad_cancel_cfg4.py):
for the worst queries, fp32 vs fp64 on the tree path (default, per-lane
leaf rounds, inline leaves, K3F) and on the exact path, all against the
compiled reference's tree result (fp64)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
idx = np.array([2262542, 935228, 3750808, 3684761, 2436517, 2694089])
P = sd.SmoothParams(alpha=200.0, alpha_u=600.0, beta=0.5)
P0 = sd.SmoothParams(alpha=200.0, alpha_u=600.0, beta=0.0)
res = {}
for prec in (sd.SD_FP32, sd.SD_FP64):
    tag = "fp64" if prec else "fp32"
    eng = sd.Engine(0, prec)
    eng.set_geometry(v, w.simplices, w.kinds)
    wt = eng.build_weights()
    eng.build_bvh(sd.SD_BVH_AUTO)
    variants = [("tree", {}), ("k3f", {"SDGPU_FRONTIER": "1"})]
    if prec == sd.SD_FP32:
        variants += [("lanes", {"SDGPU_LEAF_COOP": "0"}), ("inline", {"SDGPU_LEAF_QUEUE": "0"})]
    for name, env in variants:
        for k in ("SDGPU_LEAF_COOP", "SDGPU_LEAF_QUEUE", "SDGPU_FRONTIER"):
            os.environ.pop(k, None)
        os.environ.update(env)
        r = eng.smooth_min_dist(q[idx], P) if name == "k3f" else eng.smooth_min_dist(q, P)
        res[f"{tag}_{name}"] = (r.grad if name == "k3f" else r.grad[idx], r.c if name == "k3f" else r.c[idx])
    for k in ("SDGPU_LEAF_COOP", "SDGPU_LEAF_QUEUE", "SDGPU_FRONTIER"):
        os.environ.pop(k, None)
    r = eng.smooth_min_dist_flat(q[idx], P0) if hasattr(eng, "smooth_min_dist_flat") else None
    if r is not None:
        res[f"{tag}_exact"] = (r.grad, r.c)
    if prec == sd.SD_FP64:
        arm = bench.CpuArm(v, w.simplices, w.kinds, wt, nodes=eng.export_bvh())
        ref = arm.query(q[idx], 200.0, 600.0, 0.5, tree=True)
    del eng
print("ref |grad|", np.round(np.linalg.norm(ref.grad, axis=1), 5), "c", np.round(ref.c, 3))
for k, (g, c) in res.items():
    base = ref.grad
    if k.endswith("exact"):
        base = res["fp64_exact"][0]
    print(f"{k:12s} |dg| {np.array2string(np.linalg.norm(g - base, axis=1), precision=2)}"
          f"  dc/c {np.array2string(np.abs(c - (res['fp64_exact'][1] if k.endswith('exact') else ref.c)) / np.abs(ref.c), precision=2)}")
for k in ("fp32_exact", "fp64_exact", "fp64_tree", "fp32_tree"):
    print(k, res[k][0][:3].tolist())
