"""cfg5 exact, all-pairs kernel: queries whose sum loses terms (found by
comparing with the pruned evaluation). Per kind of primitive, c of the GPU
against the oracle for the worst queries.
  python tools/debug/cfg5_lost_term.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

nq = 65536
w, q = configs.cfg5()
v, q = configs.quantize(w.vertices), configs.quantize(q)
q = np.ascontiguousarray(q[np.linspace(0, len(q) - 1, nq).astype(np.int64)])
e = sd.Engine(0, sd.SD_FP32)
e.set_geometry(v, w.simplices, w.kinds)
wt = e.build_weights()
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=0.0)
full = e.query_points(q, P, sd.SD_EXACT, want_c=True)
e.set_exact_pruning(48.0)
got = e.query_points(q, P, sd.SD_EXACT, want_c=True)
e.set_exact_pruning(0.0)
rel = np.abs(got.c - full.c) / np.maximum(got.c, 1e-320)
worst = np.argsort(-rel)[:6]
print("worst rel c diff:", rel[worst], "queries", worst)
O.build()
thr = O.hardware_threads()
qs = q[worst]
for name, sel in (("all", slice(None)), ("triangles", w.kinds == 2), ("edges", w.kinds == 1), ("points", w.kinds == 0)):
    s, k, pi = w.simplices[sel], w.kinds[sel], wt.poly_index[sel]
    om = O.Mesh.from_arrays(v, s, k)
    ow = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, pi))
    r = O.query(om, ow, qs, O.Params(alpha=w.alpha, alpha_u=600.0, beta=0.0), threads=thr)
    e2 = sd.Engine(0, sd.SD_FP32)
    e2.set_geometry(v, s, k)
    e2.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, pi)
    # the worst queries inside their batch neighbourhood (same warps as in the big batch is not guaranteed)
    g = e2.query_points(q, P, sd.SD_EXACT, want_c=True)
    g1 = e2.query_points(qs, P, sd.SD_EXACT, want_c=True)
    for sp in ("1",):
        os.environ["SDGPU_EXACT_SPLITS"] = sp
        gs = e2.query_points(q, P, sd.SD_EXACT, want_c=True)
        del os.environ["SDGPU_EXACT_SPLITS"]
    print(name, "oracle c", r.c, "\n   gpu batch c", g.c[worst], "\n   gpu alone c", g1.c, "\n   gpu 1 split", gs.c[worst])
    e2.close()
