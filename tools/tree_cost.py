import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs, sim_rows
def metrics(nodes):
    e = nodes['hi'] - nodes['lo']
    e = np.maximum(e, 0)
    area = 2 * (e[:, 0] * e[:, 1] + e[:, 1] * e[:, 2] + e[:, 0] * e[:, 2])
    internal = nodes['left'] >= 0
    return dict(diam=float(nodes['diameter'][internal].sum() / nodes['diameter'][0]),
                area=float(area[internal].sum() / max(area[0], 1e-300)))
cases = []
w, _ = configs.cfg4(nq=1); cases.append(("cfg4", configs.quantize(w.vertices), w.simplices, w.kinds))
w, _ = configs.cfg5(nq=1); cases.append(("cfg5", configs.quantize(w.vertices), w.simplices, w.kinds))
for name in ("terrain_octopus", "street_motorcycle", "terrain_bunny"):
    r = sim_rows.ROWS[name](); cases.append((name, configs.quantize(r.data.vertices), r.data.simplices, r.data.kinds))
for name, v, s, k in cases:
    e = sd.Engine(0, sd.SD_FP32); e.set_geometry(v, s, k)
    out = {}
    for t, m in (("median", sd.SD_BVH_MEDIAN), ("lbvh", sd.SD_BVH_LBVH)):
        e.build_bvh(m); out[t] = metrics(e.export_bvh())
    print(name, out, flush=True)
