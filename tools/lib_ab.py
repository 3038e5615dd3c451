"""A/B timing of libsdgpu.so builds (tools/build_ab.sh) on the bench's BVH
leg (cfg4, 4,194,304 queries, L2 flushed, CUDA events, median of REPS;
AB_SHARD=W: rank 0's share of a W-way sharded call; AB_CFG=3 / 2 / 1: exact cfg3 / cfg2 / cfg1 (fp64); AB_PREC=64: fp64):
  python tools/lib_ab.py ablibs/base ablibs/x[:ENV=VAL,...] ...   (rounds alternate)
Each variant runs in its own process (one library per process)."""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, HERE)
import paper_2108_10480_b200 as sd
sd.LIB_PATH = os.path.join(LIBDIR, "libsdgpu.so")
from paper_2108_10480_b200 import configs
cfg = os.environ.get("AB_CFG", "4")
dev = torch.device("cuda", 0); st = torch.cuda.current_stream(dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
if cfg == "4":
    w, q = configs.cfg4(); mode = sd.SD_BVH
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
elif cfg == "2":
    import bench
    w, wt, q = bench.cfg2_workload(); mode = sd.SD_EXACT
    P = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=0.0)
elif cfg == "1":
    w, q = configs.cfg1(); mode = sd.SD_EXACT
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=0.0)
else:
    import bench
    v, T, K, q = bench.cfg3_workload(); mode = sd.SD_EXACT
    q = q[: int(os.environ.get("AB_NQ", "131072"))]
    P = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=0.0)
    w = type("W", (), {"vertices": v, "simplices": T, "kinds": K})
prec = sd.SD_FP64 if os.environ.get("AB_PREC") == "64" or cfg == "1" else sd.SD_FP32
v = w.vertices if prec == sd.SD_FP64 else configs.quantize(w.vertices)
q = q if prec == sd.SD_FP64 else configs.quantize(q)
eng = sd.Engine(0, prec); eng.set_geometry(v, w.simplices, w.kinds)
if cfg == "1": wt = configs.weights_without_triangles(w.simplices, w.kinds, len(w.vertices))
if cfg in ("1", "2"): eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
else: eng.build_weights()
if mode == sd.SD_BVH: eng.build_bvh(sd.SD_BVH_AUTO)
QD = torch.tensor(q, dtype=torch.float64 if prec == sd.SD_FP64 else torch.float32, device=dev)
D = torch.empty(len(q), dtype=torch.float64, device=dev); G = torch.empty(len(q), 3, dtype=torch.float64, device=dev)
W = int(os.environ.get("AB_SHARD", "1"))  # > 1: rank 0's share of a W-way query-sharded call
if W > 1:
    run = lambda: eng.query_points_device_shard(QD.data_ptr(), len(q), P, W, 0, D.data_ptr(), G.data_ptr(), stream=st.cuda_stream)
else:
    run = lambda: eng.query_points_device(QD.data_ptr(), len(q), P, mode, D.data_ptr(), G.data_ptr(), stream=st.cuda_stream)
for _ in range(3): run()
ts = []
for _ in range(int(os.environ.get("REPS", "9"))):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st); run(); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(json.dumps({"lib": LIBDIR, "ms": float(np.median(ts)), "min": float(min(ts))}))
'''

libs = sys.argv[1:]
rounds = int(os.environ.get("ROUNDS", "2"))
res = {l: [] for l in libs}
for r in range(rounds):
    for l in (libs if r % 2 == 0 else libs[::-1]):
        path, _, envs = l.partition(":")  # "ablibs/x:NAME=VAL,NAME2=VAL2" sets an environment per variant
        env = dict(os.environ, **dict(kv.split("=", 1) for kv in envs.split(",") if kv))
        code = CHILD.replace("HERE", repr(HERE)).replace("LIBDIR", repr(os.path.abspath(path)))
        out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
        if out.returncode != 0:
            print(l, "failed", out.stderr[-2000:], flush=True)
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        res[l].append(d["ms"])
        print(json.dumps(d), flush=True)
print(json.dumps({l: sorted(v) for l, v in res.items()}))
