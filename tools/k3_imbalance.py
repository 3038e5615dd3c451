"""cfg4: per-packet lane imbalance of the deferred work (leaf and far-field
terms per query) for 32-query packets in a Morton order of the batch --
the utilisation of per-lane rounds is bounded by mean / max per packet."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs, sharding  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
eng.build_bvh(sd.SD_BVH_AUTO)
r = eng.smooth_min_dist(q, sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta))
o = sharding.morton_order(q)
for name, x in (("leaves", r.leaves), ("far", r.far_field)):
    p = x[o][: len(o) // 32 * 32].reshape(-1, 32).astype(np.float64)
    mean, mx = p.mean(1), p.max(1)
    print(f"{name}: per query mean {x.mean():.1f}; per-packet sum(mean)/sum(max) = {mean.sum() / mx.sum():.3f}; "
          f"packets with max 0: {(mx == 0).mean():.3f}")
    half = len(q) // 2
    print(f"   uniform half mean {x[:half].mean():.1f}, near half mean {x[half:].mean():.1f}")
