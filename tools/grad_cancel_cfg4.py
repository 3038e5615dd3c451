"""cfg4 fp32 tree path against the fp64 tree path on the WHOLE 4,194,304-query
batch (the fp64 path matches the compiled reference to ~1e-13): how the
strict relative gradient error (|dg| / max(|g|, 1e-3)) depends on |grad d_hat|,
i.e. how many queries a |grad| < tau refinement rule would re-evaluate and
whether it catches every query over 1e-4.
  python tools/grad_cancel_cfg4.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
res = {}
for prec in (sd.SD_FP32, sd.SD_FP64):
    eng = sd.Engine(0, prec)
    eng.set_geometry(v, w.simplices, w.kinds)
    eng.build_weights()
    eng.build_bvh(sd.SD_BVH_AUTO)
    res[prec] = eng.smooth_min_dist(q, P)
    del eng
a, b = res[sd.SD_FP32], res[sd.SD_FP64]
fin = np.isfinite(b.d_hat)
gn = np.linalg.norm(b.grad, axis=1)
gd = np.linalg.norm(a.grad - b.grad, axis=1)
e = gd / np.maximum(gn, 1e-3)
dd = np.abs(a.d_hat - b.d_hat) / np.maximum(np.abs(b.d_hat), 1.0 / w.alpha)
out = {"n": int(fin.sum()), "over_1e-4": int((e[fin] > 1e-4).sum()), "d_over_1e-5": int((dd[fin] > 1e-5).sum()),
       "grad_norm_quantiles": {str(p): float(np.quantile(gn[fin], p)) for p in (0, 1e-4, 1e-3, 1e-2, 0.05, 0.5)},
       "abs_err_quantiles": {str(p): float(np.quantile(gd[fin], p)) for p in (0.5, 0.99, 0.9999, 1)}}
for tau in (0.02, 0.05, 0.1, 0.2, 0.3, 0.5):
    sel = fin & (gn < tau)
    out[f"tau_{tau}"] = {"flagged": int(sel.sum()), "frac": float(sel.sum() / fin.sum()),
                         "over_1e-4_unflagged": int((fin & ~sel & (e > 1e-4)).sum()),
                         "max_err_unflagged": float(e[fin & ~sel].max())}
worst = np.argsort(-np.where(fin, e, 0))[:10]
out["worst"] = [{"i": int(i), "err": float(e[i]), "abs": float(gd[i]), "gn": float(gn[i]), "d": float(b.d_hat[i]),
                 "leaves": int(b.leaves[i]), "far": int(b.far_field[i])} for i in worst]
print(json.dumps(out, indent=1))
