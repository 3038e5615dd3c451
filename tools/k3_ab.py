"""A/B of K3 variants on cfg4 (BASELINE configs[3]) in ONE process: the tree
and queries are built once, each variant (a set of SDGPU_* environment
switches read per launch) is timed with CUDA events (L2 flushed between
steps) and checked against the first variant: identical decision hashes and
counters, d_hat within 1e-5 relative.
  python tools/k3_ab.py "SDGPU_LEAF_QUEUE=0" "SDGPU_LEAF_QUEUE=1" [--steps 10] [--reps 2]"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_10480_b200 as sd  # noqa: E402
from paper_2108_10480_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="+")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--fp64", action="store_true")
ap.add_argument("--tree", default="auto")
args = ap.parse_args()

w, q = configs.cfg4()
v, q = configs.quantize(w.vertices), configs.quantize(q)
eng = sd.Engine(0, sd.SD_FP64 if args.fp64 else sd.SD_FP32)
eng.set_geometry(v, w.simplices, w.kinds)
eng.build_weights()
eng.build_bvh({"median": sd.SD_BVH_MEDIAN, "lbvh": sd.SD_BVH_LBVH}.get(args.tree, sd.SD_BVH_AUTO))
P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
Q = len(q)
qd = torch.tensor(q, dtype=torch.float64 if args.fp64 else torch.float32, device=dev)
d = torch.empty(Q, dtype=torch.float64, device=dev)
g = torch.empty(Q, 3, dtype=torch.float64, device=dev)
L = torch.empty(Q, dtype=torch.int64, device=dev)
F = torch.empty(Q, dtype=torch.int64, device=dev)
H = torch.empty(Q, dtype=torch.int64, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def setenv(spec):
    for k in [k for k in os.environ if k.startswith("SDGPU_")]:
        del os.environ[k]
    for kv in spec.split("+"):
        if "=" in kv:
            k, val = kv.split("=", 1)
            os.environ[k] = val


def run(counters=False):
    eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_BVH, d.data_ptr(), g.data_ptr(),
                            leaves_ptr=L.data_ptr() if counters else None, far_ptr=F.data_ptr() if counters else None,
                            hash_ptr=H.data_ptr() if counters else None, stream=st.cuda_stream)


base = None
for rep in range(args.reps):
    for spec in args.variants:
        setenv(spec)
        run(True)
        torch.cuda.synchronize()
        res = (d.cpu().numpy().copy(), L.cpu().numpy().copy(), F.cpu().numpy().copy(), H.cpu().numpy().copy())
        for _ in range(3):
            run()
        eng.kernel_times()
        eng.set_kernel_timing(True)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize()
        for a, b in evs:
            flush.zero_()
            a.record(st)
            run()
            b.record(st)
        torch.cuda.synchronize()
        kt = eng.kernel_times()
        eng.set_kernel_timing(False)
        ms = np.mean([a.elapsed_time(b) for a, b in evs])
        note = ""
        if base is None:
            base = res
        else:
            same = all(np.array_equal(x, y) for x, y in zip(res[1:], base[1:]))
            fin = np.isfinite(base[0])
            err = np.abs(res[0][fin] - base[0][fin]) / np.maximum(1.0, np.abs(base[0][fin]))
            note = f"decisions {'identical' if same else 'DIFFER'}, max d_hat diff {err.max():.2e}"
        print(f"{spec:50s} step {ms:7.3f} ms  kernel {np.mean(kt):7.3f} ms  {note}", flush=True)
