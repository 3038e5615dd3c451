import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import oracle as O
import paper_2108_10480_b200 as sd
for seed in (6, 3):
    m = O.random_scene(seed, 200)
    q = O.QueryStream(31).draw_points(m, 100)
    w = O.Weights.build(m)
    print("seed", seed, "kinds", np.bincount(m.kinds, minlength=3), "polys", len(w.table.edge_a), len(w.table.tri_stored))
    for prec in (1, 0):
        e = sd.Engine(0, prec)
        mm = m if prec else m.quantized()
        qq = q if prec else q.astype(np.float32).astype(float)
        e.set_geometry(mm.vertices, mm.simplices, mm.kinds)
        e.set_weight_table(w.table)
        e.build_bvh(sd.SD_BVH_LBVH)
        ref = e.query_points(qq, sd.SmoothParams(alpha=100.0, beta=0.0), sd.SD_EXACT)
        for beta in (0.0, 1e-9, 0.3):
            r = e.query_points(qq, sd.SmoothParams(alpha=100.0, beta=beta), sd.SD_BVH, want_counters=True)
            err = np.nanmax(np.abs(r.d_hat - ref.d_hat))
            print(f"  prec {prec} beta {beta}: max |d_bvh - d_exact| = {err:.3g}  leaves {r.leaves.mean():.1f} far {r.far_field.mean():.1f}")
