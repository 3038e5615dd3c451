import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2108_10480_b200 as sd
from paper_2108_10480_b200 import configs
w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP32); eng.set_geometry(v, w.simplices, w.kinds); eng.build_weights(); eng.build_bvh(sd.SD_BVH_AUTO)
P = sd.SmoothParams(alpha=200.0, beta=0.5)
dev = torch.device("cuda", 0); Q = len(q)
qd = torch.tensor(q, dtype=torch.float32, device=dev)
def run(shard, counters):
    d = torch.full((Q,), float("nan"), dtype=torch.float64, device=dev); g = torch.full((Q, 3), float("nan"), dtype=torch.float64, device=dev)
    L = torch.zeros(Q, dtype=torch.int64, device=dev); F = torch.zeros(Q, dtype=torch.int64, device=dev); H = torch.zeros(Q, dtype=torch.int64, device=dev)
    kw = dict(leaves_ptr=L.data_ptr() if counters else None, far_ptr=F.data_ptr() if counters else None, hash_ptr=H.data_ptr() if counters else None)
    if shard: eng.query_points_device_shard(qd.data_ptr(), Q, P, 4, 1, d.data_ptr(), g.data_ptr(), **kw)
    else: eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(), **kw)
    torch.cuda.synchronize(); return d.cpu().numpy(), g.cpu().numpy()
full_c = run(False, True); full = run(False, False); sh_c = run(True, True); sh = run(True, False)
m = ~np.isnan(sh_c[0])
print("rank queries", m.sum(), "shard timed written same", np.array_equal(~np.isnan(sh[0]), m), "grad nan in mine", np.isnan(sh[1][m]).any(), np.isnan(sh_c[1][m]).any())
for name, (d, g) in (("full_counted", full_c), ("shard_counted", sh_c), ("shard", sh)):
    print(name, "d maxdiff vs full", np.nanmax(np.abs(d[m] - full[0][m])), "g maxdiff", np.nanmax(np.abs(g[m] - full[1][m])))
