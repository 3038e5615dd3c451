"""cfg5 exact (65,536 evenly spaced queries x 18.8M primitives, one shard):
the pruned evaluation against the all-pairs one, and the oracle on every
query whose finiteness differs plus a strided sample.
  python tools/prune_check_cfg5.py [bits=48] [queries=65536]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

bits = float(sys.argv[1]) if len(sys.argv) > 1 else 48.0
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
w, q = configs.cfg5()
v, q = configs.quantize(w.vertices), configs.quantize(q)
q = np.ascontiguousarray(q[np.linspace(0, len(q) - 1, nq).astype(np.int64)])
e = sd.Engine(0, sd.SD_FP32)
e.set_geometry(v, w.simplices, w.kinds)
wt = e.build_weights()
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=0.0)
full = e.query_points(q, P, sd.SD_EXACT, want_c=True)
e.set_exact_pruning(bits)
got = e.query_points(q, P, sd.SD_EXACT, want_c=True)
ff, fg = np.isfinite(full.d_hat), np.isfinite(got.d_hat)
diff = np.nonzero(ff != fg)[0]
both = ff & fg
print(f"finite: all-pairs {ff.sum()}, pruned {fg.sum()}, differing {len(diff)}")
print(f"max |d_hat diff| {np.abs(got.d_hat[both] - full.d_hat[both]).max():.3g}, "
      f"max |grad diff| {np.abs(got.grad[both] - full.grad[both]).max():.3g}, "
      f"max rel c diff {(np.abs(got.c[both] - full.c[both]) / full.c[both]).max():.3g}")
O.build()
om = O.Mesh.from_arrays(v, w.simplices, w.kinds)
ow = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
idx = np.concatenate([diff[:8], np.linspace(0, nq - 1, 24).astype(np.int64)])
r = O.query(om, ow, q[idx], O.Params(alpha=w.alpha, alpha_u=600.0, beta=0.0), threads=O.hardware_threads())
for j, i in enumerate(idx[: len(diff[:8])]):
    print(f"query {i}: oracle d_hat {r.d_hat[j]!r} c {r.c[j]!r}; all-pairs {full.d_hat[i]!r} c {full.c[i]!r}; "
          f"pruned {got.d_hat[i]!r} c {got.c[i]!r}; alpha*d_hat {w.alpha * r.d_hat[j]!r}")
ok = np.isfinite(r.d_hat)
print("sample: oracle vs pruned max |d_hat diff|", np.abs(got.d_hat[idx][ok] - r.d_hat[ok]).max(),
      "oracle vs all-pairs", np.abs(full.d_hat[idx][ok] - r.d_hat[ok]).max())
