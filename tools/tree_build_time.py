"""cfg4 (5.24M triangles) tree-build wall times: median (GPU), LBVH, AUTO,
and the first BVH query (device layout upload)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4(nq=4096)
v = configs.quantize(w.vertices)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
for name, m in (("median", sd.SD_BVH_MEDIAN), ("lbvh", sd.SD_BVH_LBVH), ("auto", sd.SD_BVH_AUTO), ("median", sd.SD_BVH_MEDIAN)):
    t0 = time.perf_counter()
    eng.build_bvh(m)
    t1 = time.perf_counter()
    eng.query_points(configs.quantize(q), P, sd.SD_BVH)
    t2 = time.perf_counter()
    eng.query_points(configs.quantize(q), P, sd.SD_BVH)
    t3 = time.perf_counter()
    print(f"{name:7s} build {t1 - t0:.3f} s, first query (upload) {t2 - t1:.3f} s, next query {t3 - t2:.4f} s")
