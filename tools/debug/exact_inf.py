"""fp32 exact path on the cfg4 gradient-outlier queries: raw c / grad_c,
split variants, and the query's distance to the mesh (oracle exact_min)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
idx = np.array([2262542, 935228, 3750808])
P = sd.SmoothParams(alpha=200.0, alpha_u=600.0, beta=0.0)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
for env in ({}, {"SDGPU_EXACT_SPLITS": "1"}, {"SDGPU_EXACT_SPLITS": "7"}):
    for k in ("SDGPU_EXACT_SPLITS",):
        os.environ.pop(k, None)
    os.environ.update(env)
    r = eng.query_points(q[idx], P, sd.SD_EXACT, want_c=True)
    print(env, "d", r.d_hat, "c", r.c)
    print("   grad_c", r.grad_c.tolist())
# nearest primitives of query 0 (numpy brute force over triangle centroids, then exact point-triangle)
tri = w.simplices[w.kinds == 2]
cen = v[tri].mean(axis=1)
for qq in q[idx]:
    dd = np.linalg.norm(cen - qq, axis=1)
    o = np.argsort(dd)[:3]
    print("query", qq.tolist(), "nearest centroid dist", dd[o].tolist())
