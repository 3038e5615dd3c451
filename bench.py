#!/usr/bin/env python
"""Benchmark of the B200 smooth-distance engine (exact path, BASELINE cfg2).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one exact pass of d_hat + grad over the workload's queries
(smooth_min_dist_flat for every query, smooth.hpp:189-198): BASELINE.json
configs[1], the helix polyline (20,000 edges) against 262,144 queries per
GPU, alpha = 100, fp32. Multi-GPU runs shard queries (each rank its own
block of the same query distribution) with the geometry replicated: no
collective on the data path, "scaling": "weak". One JSON line on rank 0.

--impl reference times the reference CPU evaluator of the same path on this
host's cores: the reference cannot be built here (Eigen3/GTest/CLI11 are
absent), so its line-faithful fp64 restatement in oracle/ stands in
("kind": "port"). Only that leg and the cpu_baseline leg execute oracle/.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FLOPS_PER_EDGE_PAIR = 62      # SURVEY 8(d) canonical count, S != 1
FLOPS_PER_TRI_PAIR = 192
FLOPS_BOX_TEST, FLOPS_FAR_TERM = 10, 12
BYTES_NODE, BYTES_LEAF = 32, 100  # fp32 traversal node record; leaf record (96 B) + meta
MUFU_PER_EDGE_PAIR = 3            # rsqrt, lg2, ex2 (no reciprocal on certified-positive weights)
QUERIES_PER_GPU = 262144
ALPHA = 100.0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# Tree builder (BENCH_TREE=median|lbvh|auto, default auto): SD_BVH_AUTO
# builds the reference's median-split tree (build_bvh, bvh.hpp:34-91, on the
# device by median.cu) and the GPU LBVH and keeps the smaller surface-area
# cost -- the median tree on single surfaces (cfg4 28.4 ms vs 29.7 ms:
# 1152 vs 1335 popped nodes per query; Terrain 8.2 vs 15.6 ms), the LBVH on
# clustered scenes whose Morton splits follow the gaps between objects (cfg5
# 35 vs 62 ms, City Street 22 vs 38 ms).
def tree_method(sd):
    t = os.environ.get("BENCH_TREE") or "auto"
    return {"median": sd.SD_BVH_MEDIAN, "lbvh": sd.SD_BVH_LBVH}.get(t, sd.SD_BVH_AUTO)


def tree_name():
    t = os.environ.get("BENCH_TREE") or "auto"
    return {"median": "reference median-split tree built on the GPU", "lbvh": "GPU LBVH"}.get(
        t, "GPU tree (median split or LBVH, smaller surface-area cost)")


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a thread (nvidia-smi -lms 200 as the
    fallback when pynvml is unavailable)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.nvml = pynvml

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:  # noqa: BLE001 -- sampling must never break a run
                        break
                    names = [n for n, bit in self.BITS.items() if r & bit]
                    self.lines.append((float(sm), float(smax), names))
                    time.sleep(0.002)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            f = [x.strip() for x in line.strip().split(",")]
            if len(f) < 9:
                continue
            try:
                sm, smax = float(f[1]), float(f[2])
            except ValueError:
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            self.lines.append((sm, smax, [n for n, v in zip(names, f[5:9]) if v.lower() == "active"]))

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [x[0] for x in self.lines]
        smax = [x[1] for x in self.lines]
        reasons = set(n for x in self.lines for n in x[2])
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def measure_peaks(device: int = 0):
    L = ctypes.CDLL(os.path.join(ROOT, "paper_2108_10480_b200", "libsdpeaks.so"))
    L.sd_peaks_set_device.argtypes = [ctypes.c_int]
    if L.sd_peaks_set_device(device) != 0:
        return None
    f, d, m = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    L.sd_measure_peaks.argtypes = [ctypes.POINTER(ctypes.c_double)] * 3
    if L.sd_measure_peaks(ctypes.byref(f), ctypes.byref(d), ctypes.byref(m)) != 0:
        return None
    out = {"ffma_tflops": f.value / 1e12, "dfma_tflops": d.value / 1e12, "mufu_tops": m.value / 1e12}
    f2 = ctypes.c_double()
    L.sd_measure_ffma2.argtypes = [ctypes.POINTER(ctypes.c_double)]
    if L.sd_measure_ffma2(ctypes.byref(f2)) == 0:
        out["ffma2_tflops"] = f2.value / 1e12
    return out


def workload(block: int, cfg: int = 2, alpha: float | None = None, device: int = 0):
    """cfg2 (headline) or cfg3 (triangles, --config 3): mesh, fp32-rounded
    vertices and queries, and the WeightSet table."""
    from paper_2108_10480_b200 import configs
    if cfg == 1:
        w, q = configs.cfg1()
        q = np.random.default_rng([1002, block]).uniform(-2, 2, q.shape)
        wt = configs.weights_without_triangles(w.simplices, w.kinds, len(w.vertices))
        return w, w.vertices, q, wt  # fp64 config: no rounding
    if cfg == 2:
        w, q = configs.cfg2(QUERIES_PER_GPU, block=block)
        wt = configs.weights_without_triangles(w.simplices, w.kinds, len(w.vertices))
    else:
        V, T = configs.torus()
        rng = np.random.default_rng([3002, block])
        lo, hi = V.min(0) - 0.5, V.max(0) + 0.5
        q = rng.uniform(lo, hi, (1048576, 3))
        w = configs.Workload("cfg3 torus 262,144 triangles, exact LSE", V, T, np.full(len(T), 2, np.uint8),
                             alpha=alpha or 100.0)
        import paper_2108_10480_b200 as sd
        e = sd.Engine(device, sd.SD_FP32)
        e.set_geometry(configs.quantize(V), T, w.kinds)
        wt = e.build_weights()
        e.close()
    return w, configs.quantize(w.vertices), configs.quantize(q), wt


def cpu_sample(v, s, k, wt, q, threads, target_s=12.0):
    """Times the oracle port on a bounded prefix of the queries, sized from a
    pilot so that the sample takes about target_s seconds."""
    import oracle as O
    m = O.Mesh.from_arrays(v, s, k)
    w = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
    p = O.Params(alpha=ALPHA, alpha_u=600.0, beta=0.0)
    pilot = max(threads * 2, 64)
    r = O.query(m, w, q[:pilot], p, threads=threads)
    n = int(min(len(q), max(pilot, pilot * target_s / max(r.seconds, 1e-3))))
    r = O.query(m, w, q[:n], p, threads=threads)
    return n, r.seconds, r


def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle as O
    O.build()
    w, v, q, wt = workload(0)
    threads = O.hardware_threads()
    N = len(w.kinds)
    n, secs, _ = cpu_sample(v, w.simplices, w.kinds, wt, q, threads, target_s=3.0)
    import oracle as O2  # noqa: F401  (same module; warm-up steps below)
    m = O.Mesh.from_arrays(v, w.simplices, w.kinds)
    ws = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
    p = O.Params(alpha=ALPHA, alpha_u=600.0, beta=0.0)
    for i in range(args.warmup):
        O.query(m, ws, q[:n], p, threads=threads)
    times = []
    for i in range(args.steps):
        lo = (i * n) % max(1, len(q) - n)
        r = O.query(m, ws, q[lo:lo + n], p, threads=threads)
        times.append(r.seconds)
    t = float(np.mean(times))
    value = n * N / t
    line = {
        "impl": "reference", "metric": "exact pair-evals/s (value+grad)", "value": value, "unit": "pair-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg2: helix polyline 20,000 edges, exact LSE, alpha=100 (BASELINE configs[1])",
                   "queries_per_step": n, "primitives": N, "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": threads, "kind": "port",
                         "sample": f"{n} of {QUERIES_PER_GPU} cfg2 queries x {N} edges per step"},
        "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_bvh:
        line["bvh"] = reference_bvh(threads)
    print(json.dumps(line), flush=True)


def reference_bvh(threads, target_s=10.0):
    """The reference's own CPU path for the BVH metric: the oracle port builds
    the WeightSet and the median-split tree of cfg4 on the host
    (build_weight_set / build_bvh restated) and evaluates a bounded query
    sample (both halves of the distribution) on all host threads."""
    import oracle as O
    from paper_2108_10480_b200 import configs
    t0 = time.perf_counter()
    w, q = configs.cfg4()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    m = O.Mesh.from_arrays(v, w.simplices, w.kinds)
    ws = O.Weights.build(m)
    tree = O.Tree.build(m)
    setup = time.perf_counter() - t0
    p = O.Params(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
    half = len(q) // 2
    pick = lambda n: np.concatenate([q[:n // 2], q[half:half + n - n // 2]])
    pilot = max(threads * 16, 1024)
    r = O.query(m, ws, pick(pilot), p, tree=tree, threads=threads)  # also warms the tree pages
    n = int(min(262144, max(pilot, pilot * target_s / max(r.seconds, 1e-3))))
    r = O.query(m, ws, pick(n), p, tree=tree, threads=threads)
    return {"metric": "BVH queries/s (value+grad)", "value": n / r.seconds, "unit": "queries/s",
            "workload": "cfg4 (BASELINE configs[3]): icosphere(9), 5,242,880 triangles, alpha=200, beta=0.5, "
                        "host-built median tree and WeightSet",
            "cpu_baseline": {"value": n / r.seconds, "unit": "queries/s", "cores": threads, "kind": "port",
                             "sample": f"{n} cfg4 queries (half from each half of the distribution), "
                                       f"{r.seconds:.1f} s"},
            "setup_s": setup}


def measure_bvh(args, rank, world, local, eng_cls, dev, stream, flush, peaks):
    """Secondary line item: BVH far-field queries/s on BASELINE configs[3]
    (cfg4: icosphere(9), 5,242,880 triangles, 4,194,304 queries per GPU,
    alpha 200, beta 0.5), the reference's median tree built on the GPU + fp32
    traversal."""
    import torch
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import configs
    t0 = time.perf_counter()
    strong = args.bvh_strong
    # weak (default): every rank its own cfg4 batch; strong: ONE batch split
    # into Morton-contiguous blocks of equal estimated cost
    w, q = configs.cfg4(block=0 if strong else rank)
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    Q_total = len(q) * (1 if strong else world)
    bvh64 = args.fp64 and args.config == 2  # --fp64: the BVH leg in fp64 too
    eng = sd.Engine(local, sd.SD_FP64 if bvh64 else sd.SD_FP32)
    eng.set_geometry(v, w.simplices, w.kinds)
    tw = time.perf_counter()
    eng.build_weights()
    tw = time.perf_counter() - tw
    tb = time.perf_counter()
    # BENCH_TREE=median builds the reference's median-split tree instead (A/B)
    eng.build_bvh(tree_method(sd))
    tb = time.perf_counter() - tb
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
    balance = None
    if strong:
        from paper_2108_10480_b200 import sharding

        def counters(sub):
            r = eng.smooth_min_dist(sub, P)
            return r.leaves, r.far_field

        order = sharding.morton_order(q)
        est = sharding.estimate_query_costs(counters, q[order], stride=64)
        ranges = sharding.balanced_ranges(est, world)
        lo, hi = ranges[rank]
        q = np.ascontiguousarray(q[order[lo:hi]])
        balance = {"ranges": ranges, "estimated_cost_share": [float(est[a:b].sum() / est.sum()) for a, b in ranges],
                   "estimate": "strided sample (1/64) of the Morton-sorted batch, popped nodes 2(L+F)-1"}
    Q = len(q)
    qd = torch.tensor(q, dtype=torch.float64 if bvh64 else torch.float32, device=dev)
    d_hat = torch.empty(Q, dtype=torch.float64, device=dev)
    grad = torch.empty(Q, 3, dtype=torch.float64, device=dev)
    leaves = torch.empty(Q, dtype=torch.int64, device=dev)
    far = torch.empty(Q, dtype=torch.int64, device=dev)

    def step(counters=False):
        eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_BVH, d_hat.data_ptr(), grad.data_ptr(),
                                leaves_ptr=leaves.data_ptr() if counters else None,
                                far_ptr=far.data_ptr() if counters else None, stream=stream.cuda_stream)

    step(counters=True)  # also uploads the traversal layout
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    L = leaves.double().sum().item()
    F = far.double().sum().item()
    for _ in range(max(3, args.warmup)):
        step()
    launches = eng.last_launch_count()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        evs[i][0].record(stream)
        step()
        evs[i][1].record(stream)
    torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    # end to end through the public host API: pinned fp64 host queries in,
    # d_hat + gradient out (H2D, Morton sort, traversal, finalize, D2H)
    qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
    res = sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                           torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy())
    eng.query_points(qh, P, sd.SD_BVH, out=res)
    e2e_times = []
    for _ in range(max(3, args.steps)):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        eng.query_points(qh, P, sd.SD_BVH, out=res)
        e2e_times.append(time.perf_counter() - t1)
    te = torch.tensor([float(np.mean(e2e_times))], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e = {"value": Q_total / float(te.item()), "unit": "queries/s", "h2d_bytes_per_step": Q * 24,
           "d2h_bytes_per_step": Q * 32}
    if world > 1:  # counters summed over ranks (per-query means below are whole-job)
        lf = torch.tensor([L, F, float(Q)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(lf)
        L, F, Qsum = (float(x) for x in lf.tolist())
    else:
        Qsum = float(Q)
    pops = 2 * (L + F) - Qsum
    # algorithmic work per GPU per step (whole-job / ranks), over the
    # max-over-ranks step time: the roofline is a per-GPU figure
    flops = (FLOPS_BOX_TEST * pops + FLOPS_FAR_TERM * F + FLOPS_PER_TRI_PAIR * L) / world
    nbytes = (BYTES_NODE * pops + BYTES_LEAF * L) / world
    out = {"metric": "BVH queries/s (value+grad)", "value": Q_total / (ms * 1e-3), "unit": "queries/s",
           "scaling": "strong" if strong else "weak", "e2e": e2e,
           "ms_per_step": ms, "queries_per_gpu": Q, "primitives": len(w.kinds),
           "workload": "cfg4: icosphere(9) with radial displacement, 5,242,880 triangles, 4,194,304 queries "
                       "per GPU (half uniform in [-1.5,1.5]^3, half within 0.02 of the surface), alpha=200, "
                       f"beta=0.5, {'fp64' if bvh64 else 'fp32'}, {tree_name()} (BASELINE configs[3])",
           "dtype": "f64" if bvh64 else "f32",
           "per_query": {"leaves": L / Qsum, "far_field": F / Qsum, "nodes_popped": pops / Qsum},
           "setup_s": {"total": setup_s, "build_weights": tw, "build_tree": tb},
           "gpu_launches": launches * args.steps,
           "roofline": {"achieved_tflops": flops / (ms * 1e-3) / 1e12, "touched_gbs": nbytes / (ms * 1e-3) / 1e9,
                        "hbm_peak_gbs": 6542.4, "algorithmic": "10 flop/popped node + 12/far term + 192/exact "
                        "tri leaf; 32 B/popped node + 100 B/leaf (from this run's counters)"}}
    if balance:
        out["balance"] = balance
    if peaks:
        out["roofline"]["frac_fp32"] = out["roofline"]["achieved_tflops"] / peaks["ffma_tflops"]
    # the touched bytes are served from L1/L2 (ncu of pair_kernel: DRAM 0.9 % of
    # peak, L2 hit 88 %, L1 hit 57 %); the kernel is issue-bound (76 % of issue
    # slots, profiles/r1_pair_bvh_summary.md)
    out["roofline"]["bound"] = "issue (L1/L2-resident tree)"
    out["roofline"]["touched_frac_of_hbm_peak"] = out["roofline"]["touched_gbs"] / 6542.4
    # the issue-slot bound, from the committed ncu capture of this kernel (not
    # measured in this run): warp instructions per launch and issue-slot use
    out["roofline"]["ncu_issue"] = {"issue_slots_busy": 0.768, "ipc": 3.05, "warp_instructions": 2.009e10,
                                    "avg_active_lanes": 17.0, "source": "profiles/r1_pair_bvh_details.csv, "
                                    "profiles/r1_k3_source_breakdown.md (fp32, median tree)"}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = bvh_cpu_sample(eng, v, w, q, P)
    eng.close()
    return out


def bvh_cpu_sample(eng, v, w, q, P, target_s=10.0):
    """The oracle port (fp64, all host threads) on a bounded query subset of
    cfg4, traversing the SAME tree (the GPU-built tree exported in the reference
    layout) with the same WeightSet table."""
    import oracle as O
    O.build()
    threads = O.hardware_threads()
    wt = eng.weight_table()
    m = O.Mesh.from_arrays(v, w.simplices, w.kinds)
    ws = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
    t = O.Tree.from_nodes(eng.export_bvh())
    p = O.Params(alpha=P.alpha, alpha_u=P.alpha_u, beta=P.beta)
    # both halves of the query distribution (uniform box / near surface)
    half = len(q) // 2
    pick = lambda n: np.concatenate([q[:n // 2], q[half:half + n - n // 2]])
    pilot = max(threads * 16, 1024)
    r = O.query(m, ws, pick(pilot), p, tree=t, threads=threads)
    n = int(min(65536, max(pilot, pilot * target_s / max(r.seconds, 1e-3))))
    r = O.query(m, ws, pick(n), p, tree=t, threads=threads)
    return {"value": n / r.seconds, "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"{n} cfg4 queries (half from each half of the distribution) on the exported GPU-built tree, "
                      f"fp64 oracle port, {r.seconds:.1f} s"}


def run_cfg5(args, rank, world, local):
    """BASELINE configs[4]: mixed scene (16.8M triangles + 1M edges + 1M
    points), 16,777,216 queries, alpha 100, beta 0.5, PRIMITIVE-sharded over
    the ranks (Morton-contiguous shards, one GPU-built tree per shard, global
    WeightSet), per-query fp64 partials merged with ONE NCCL all-reduce,
    then sd_finalize_device. Strong scaling (fixed total work)."""
    import torch
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import configs, sharding
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.perf_counter()
    w, q = configs.cfg5()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    tg = time.perf_counter() - t0
    eg = sd.Engine(local, sd.SD_FP32)  # host-side: global WeightSet on the full mesh
    eg.set_geometry(v, w.simplices, w.kinds)
    tw = time.perf_counter()
    wt = eg.build_weights()
    tw = time.perf_counter() - tw
    eg.close()
    sh = sharding.primitive_shards(v, w.simplices, w.kinds, wt.poly_index, world)[rank]
    eng = sd.Engine(local, sd.SD_FP32)
    eng.set_geometry(sh.vertices, sh.simplices, sh.kinds)
    eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, sh.poly_index)
    tb = time.perf_counter()
    # BENCH_TREE=median builds the reference's median-split tree instead (A/B)
    eng.build_bvh(tree_method(sd))
    tb = time.perf_counter() - tb
    Q = len(q)
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
    qd = torch.tensor(q, dtype=torch.float32, device=dev)
    buf = torch.empty(4 * Q, dtype=torch.float64, device=dev)  # [c | grad_c AoS]: one all-reduce
    d_hat = torch.empty(Q, dtype=torch.float64, device=dev)
    grad = torch.empty(Q, 3, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    launches = [0]

    # merge: one NCCL all_reduce of the partials (default), or the peer-memory
    # exchange (--exchange peer): every rank stores its partials into the
    # owners' symmetric buffers (torch symmetric memory), a device barrier,
    # and each owner finalises its block of queries
    exchange = args.exchange
    per, counts = sharding.owner_blocks(Q, world)
    hdl = None
    if exchange == "peer":
        try:
            if world > 1:
                import torch.distributed._symmetric_memory as symm_mem
                sbuf = symm_mem.empty(world * 4 * per, dtype=torch.float64, device=dev)
                hdl = symm_mem.rendezvous(sbuf, torch.distributed.group.WORLD.group_name)
                ptrs = list(hdl.buffer_ptrs)
            else:
                sbuf = torch.zeros(world * 4 * per, dtype=torch.float64, device=dev)
                ptrs = [sbuf.data_ptr()]
            table = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        except Exception as ex:  # noqa: BLE001 -- fall back to the all-reduce
            exchange = f"nccl (peer exchange unavailable: {type(ex).__name__}: {ex})"

    def step():
        if exchange == "peer":
            # evaluation with the stores into the owners' buffers fused into
            # its finalize epilogue (sd_query_points_scatter)
            eng.query_points_scatter(qd.data_ptr(), Q, P, sd.SD_BVH, table.data_ptr(), world, rank, per,
                                     stream=stream.cuda_stream)
            launches[0] = eng.last_launch_count()
            if hdl is not None:
                hdl.barrier(channel=0)
            eng.reduce_owned(sbuf.data_ptr(), per, counts[rank], world, P, d_hat.data_ptr(), grad.data_ptr(),
                             stream=stream.cuda_stream)
            if hdl is not None:  # owners done reading before the next step's stores
                hdl.barrier(channel=1)
            launches[0] += 1
            return
        eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_BVH, d_hat.data_ptr(), c_ptr=buf.data_ptr(),
                                grad_c_ptr=buf.data_ptr() + 8 * Q, stream=stream.cuda_stream)
        launches[0] = eng.last_launch_count() + 1  # + the finalize kernel below
        if world > 1:
            torch.distributed.all_reduce(buf, op=torch.distributed.ReduceOp.SUM)
        eng.finalize_device(buf.data_ptr(), buf.data_ptr() + 8 * Q, Q, P, d_hat.data_ptr(), grad.data_ptr(),
                            stream=stream.cuda_stream)

    step()
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for _ in range(max(3, args.warmup) - 1):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    ms = float(np.mean([a.elapsed_time(b) for a, b in evs]))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    nres = counts[rank] if exchange == "peer" else Q  # peer exchange: this rank's block of results
    fin = float(torch.isfinite(d_hat[:nres]).double().mean().item())
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the oracle port on 4,096 of the queries, same tree and table
        import oracle as O
        O.build()
        threads = O.hardware_threads()
        om = O.Mesh.from_arrays(v, w.simplices, w.kinds)
        ow = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
        ot = O.Tree.from_nodes(eng.export_bvh())
        sample = np.linspace(0, Q - 1, 4096).astype(np.int64)
        r = O.query(om, ow, q[sample], O.Params(alpha=w.alpha, alpha_u=600.0, beta=w.beta), tree=ot, threads=threads)
        got = d_hat[torch.as_tensor(sample, device=dev)].cpu().numpy()
        ok = np.isfinite(r.d_hat)
        cpu = {"value": 4096 / r.seconds, "unit": "queries/s", "cores": threads, "kind": "port",
               "sample": f"4,096 evenly spaced cfg5 queries on the exported GPU-built tree, fp64 oracle port, {r.seconds:.2f} s",
               "max_abs_d_hat_diff": float(np.abs(got[ok] - r.d_hat[ok]).max()) if ok.any() else 0.0}
        del om, ow, ot
    if rank == 0:
        line = {"metric": "BVH queries/s (value+grad), primitive-sharded", "value": Q / (ms * 1e-3),
                "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": "cfg5: 64 rotated cfg3 tori (16,777,216 triangles) + 1M edges + 1M points, "
                                       "16,777,216 queries uniform in the scene AABB, alpha=100, beta=0.5, fp32 "
                                       "(BASELINE configs[4])",
                           "parallelism": f"primitive-sharded x{world} (Morton shards, {tree_name()} per shard), "
                                          + ("partials stored into the owners' symmetric buffers over peer memory "
                                             "by the evaluation's own finalize epilogue (sd_query_points_scatter), "
                                             "owner-side reduce + finalize" if exchange == "peer" else
                                             f"one NCCL all_reduce(SUM) of 4 fp64 per query; exchange={exchange}"),
                           "primitives_per_gpu": len(sh.kinds), "l2": "flushed between timed steps"},
                "finite_fraction": fin, "gpu_launches": launches[0] * args.steps, "cpu_baseline": cpu,
                "setup_s": {"total": setup, "generate": tg, "build_weights": tw, "build_tree": tb},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_m2m(args, rank, world, local):
    """Mesh-to-mesh smooth distance d_hat(M, Mq) (smooth_mesh_dist,
    smooth.hpp:212-255) on seeded stand-ins for every row of the paper's
    timing table (average evaluation time on 28 CPU
    threads; sim_rows.py has the shapes, with each row's primitive types,
    counts, alpha and alpha_q). One step = one evaluation through the public
    host API (query mesh H2D, inner BVH queries -- points on the fp32 point
    path, edges / triangles on the fp64 simplex path -- outer LogSumExp,
    vertex gradients D2H); the data mesh's weights and tree are built
    once per row. The oracle port evaluates the same row once on the host
    threads (cpu_ms) and its d_hat checks ours."""
    import torch
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import configs, sim_rows
    torch.cuda.set_device(local)
    names = args.rows.split(",") if args.rows else list(sim_rows.ROWS)
    rows = []
    with ClockSampler(local) as clk:
        for name in names:
            r = sim_rows.ROWS[name]()
            dv = configs.quantize(r.data.vertices)
            qv = configs.quantize(r.query.vertices)
            eng = sd.Engine(local, sd.SD_FP32)
            t0 = time.perf_counter()
            eng.set_geometry(dv, r.data.simplices, r.data.kinds)
            eng.build_weights()
            eng.build_bvh(tree_method(sd))
            setup = time.perf_counter() - t0
            P = sd.SmoothParams(alpha=r.alpha, alpha_u=600.0, beta=0.5, alpha_q=r.alpha_q)
            run = lambda: eng.smooth_mesh_dist_general(qv, r.query.simplices, r.query.kinds, P)
            for _ in range(max(3, args.warmup)):
                md = run()
            launches = eng.last_launch_count()
            times = []
            for _ in range(args.steps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                md = run()
                times.append(time.perf_counter() - t0)
            ms = 1e3 * float(np.mean(times))
            row = {"row": r.name, "types": r.types, "alpha": r.alpha, "alpha_q": r.alpha_q, "gpu_ms": ms,
                   "gpu_ms_min": 1e3 * float(np.min(times)), "paper_ms": r.paper_ms, "speedup_vs_paper": r.paper_ms / ms,
                   "d_hat": md.d_hat, "setup_s": setup, "gpu_launches": launches}
            if not args.no_cpu:
                import oracle as O
                O.build()
                threads = O.hardware_threads()
                om = O.Mesh.from_arrays(dv, r.data.simplices, r.data.kinds)
                # same table and tree as the GPU run
                wt = eng.weight_table()
                ow = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
                ot = O.Tree.from_nodes(eng.export_bvh())
                oq = O.Mesh.from_arrays(qv, r.query.simplices, r.query.kinds)
                t0 = time.perf_counter()
                ref = O.mesh_dist(om, ow, oq, O.Params(alpha=r.alpha, beta=0.5, alpha_q=r.alpha_q), tree=ot,
                                  threads=threads)
                row.update({"cpu_ms": 1e3 * (time.perf_counter() - t0), "cpu_threads": threads,
                            "cpu_d_hat": ref.d_hat, "d_hat_abs_err": abs(ref.d_hat - md.d_hat),
                            "leaves_per_query": ref.leaves / r.query.n, "far_per_query": ref.far_field / r.query.n})
            eng.close()
            rows.append(row)
            print(json.dumps(row), file=sys.stderr, flush=True)
    tot = sum(x["gpu_ms"] for x in rows)
    paper = sum(x["paper_ms"] for x in rows)
    cpu = None
    if not args.no_cpu:
        cpu = {"value": sum(x["cpu_ms"] for x in rows), "unit": "ms", "cores": rows[0]["cpu_threads"], "kind": "port",
               "sample": "one evaluation of every row, fp64 oracle port on the host threads, same weights and tree"}
    line = {"metric": "mesh-to-mesh d_hat(M, Mq) + vertex gradients, sum of avg evaluation times over the paper's "
                      "timing table", "value": tot, "unit": "ms", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot, "higher_is_better": False, "scaling": "none",
            "vs_baseline": tot / paper, "dtype": "f32 points / f64 simplices", "data": "synthetic stand-ins",
            "config": {"workload": f"{len(rows)} rows of PAPER.md:1378-1397 (sim_rows.py stand-ins), beta=0.5, "
                                   f"{tree_name()}, e2e through sd_mesh_dist", "paper_total_ms": paper},
            "rows": rows, "cpu_baseline": cpu, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_render(args, rank, world, local):
    """The reference's batched callers on their acceptance workloads:
    beta_ablation (bench.hpp:94-145) of the sphere tracer (render.hpp:77-134)
    on uv_torus (7,200 triangles) in the benchmark frame, 256 x 256, alpha
    200, alpha_u 1200, beta in {0, 0.2, 0.5} (acceptance [6],
    T/acceptance.cpp:367-390), and grid_benchmark (bench.hpp:29-70) at 64^3
    on the same mesh. GPU: sd_render / sd_grid_benchmark (device time of
    the whole call); CPU: the oracle port's render on the host threads."""
    import torch
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import callers, configs
    torch.cuda.set_device(local)
    V, T = configs.torus(0.35, 0.15, 60, 60, jitter=False)
    V = configs.benchmark_frame(V)
    K = np.full(len(T), 2, np.uint8)
    e = V.max(0) - V.min(0)
    diag = float(np.sqrt((e[0] * e[0] + e[1] * e[1]) + e[2] * e[2]))
    eng = sd.Engine(local, sd.SD_FP64 if args.fp64 else sd.SD_FP32)
    eng.set_geometry(V, T, K)
    eng.build_weights()
    eng.build_bvh(tree_method(sd))
    P = sd.SmoothParams(alpha=200.0, alpha_u=1200.0)
    for _ in range(max(1, args.warmup)):
        eng.render(sd.SmoothParams(alpha=200.0, alpha_u=1200.0, beta=0.2))
    with ClockSampler(local) as clk:
        rows = [callers.beta_ablation(eng, P, [0.0, 0.2, 0.5], diag) for _ in range(max(1, args.steps))]
        grids = [eng.grid_benchmark(sd.SmoothParams(alpha=100.0, beta=0.3), 64) for _ in range(max(1, args.steps))]
    # per-beta median over the repetitions
    med = []
    for k, beta in enumerate((0.0, 0.2, 0.5)):
        rs = [r[k] for r in rows]
        secs = float(np.median([r.seconds for r in rs]))
        med.append({"beta": beta, "seconds": secs, "mean_disp_rel": rs[0].mean_disp_rel,
                    "max_disp_rel": rs[0].max_disp_rel, "mismatched_hits": rs[0].mismatched_hits,
                    "leaves": rs[0].leaves})
    for m in med:
        m["speedup_vs_beta0"] = med[0]["seconds"] / m["seconds"]
    grid_s = float(np.median([g[3] for g in grids]))
    cpu = None
    if not args.no_cpu:
        import oracle as O
        O.build()
        threads = O.hardware_threads()
        wt = eng.weight_table()
        om = O.Mesh.from_arrays(V, T, K)
        ow = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
        ot = O.Tree.from_nodes(eng.export_bvh())
        r = O.render(om, ow, ot, O.Params(alpha=200.0, alpha_u=1200.0, beta=0.2), O.render_config(), threads)
        g = eng.render(sd.SmoothParams(alpha=200.0, alpha_u=1200.0, beta=0.2))
        cpu = {"value": r.seconds, "unit": "s", "cores": threads, "kind": "port",
               "sample": "the beta = 0.2 render (256 x 256) on the same tree and weights, fp64 oracle port",
               "hits": r.hits, "gpu_hits": g.hits,
               "hit_mismatch": int(((r.hit_t >= 0) != (g.hit_t >= 0)).sum())}
    line = {"metric": "sphere-traced render time (256x256, beta 0.2) -- acceptance [6] workload", "value": med[1]["seconds"],
            "unit": "s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * med[1]["seconds"],
            "higher_is_better": False, "scaling": "none", "vs_baseline": None,
            "dtype": "f64" if args.fp64 else "f32", "data": "synthetic (uv_torus 60x60, benchmark frame)",
            "config": {"workload": "render.hpp:77-134 via sd_render, beta_ablation {0, 0.2, 0.5}, alpha 200, "
                                   f"alpha_u 1200, {tree_name()}; grid_benchmark 64^3 alpha 100 beta 0.3"},
            "ablation": med, "acceptance_6": {"speedup_beta02": med[1]["speedup_vs_beta0"],
                                              "pass": med[1]["speedup_vs_beta0"] >= 5.0
                                              and med[1]["mean_disp_rel"] < 0.04 and med[2]["mean_disp_rel"] < 0.04},
            "grid_64_seconds": grid_s, "cpu_baseline": cpu, "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local):
    import torch
    import paper_2108_10480_b200 as sd

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w, v, q, wt = workload(rank, args.config, args.alpha, local)
    global ALPHA, FLOPS_PER_EDGE_PAIR, MUFU_PER_EDGE_PAIR
    if args.config == 3:
        ALPHA = w.alpha
        FLOPS_PER_EDGE_PAIR, MUFU_PER_EDGE_PAIR = FLOPS_PER_TRI_PAIR, 3
    if args.config == 1:
        ALPHA = w.alpha
        FLOPS_PER_EDGE_PAIR, MUFU_PER_EDGE_PAIR = 20, 2
    fp64 = args.config == 1 or args.fp64
    prec = sd.SD_FP64 if fp64 else sd.SD_FP32
    N, Q = len(w.kinds), len(q)
    eng = sd.Engine(local, prec)
    eng.set_geometry(v, w.simplices, w.kinds)
    eng.set_weights(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index)
    P = sd.SmoothParams(alpha=ALPHA, alpha_u=600.0, beta=0.0)

    dev = torch.device("cuda", local)
    qd = torch.tensor(q, dtype=torch.float64 if fp64 else torch.float32, device=dev)
    d_hat = torch.empty(Q, dtype=torch.float64, device=dev)
    grad = torch.empty(Q, 3, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_EXACT, d_hat.data_ptr(), grad.data_ptr(),
                                stream=stream.cuda_stream)

    peaks = measure_peaks(local) if rank == 0 else None  # only rank 0 reports the roofline
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    launches_per_step = eng.last_launch_count()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = float(np.mean(step_ms))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(t.item())
    pairs_per_rank = Q * N
    value = world * pairs_per_rank / (ms_max * 1e-3)

    # end to end through the public host API: pinned host q in, d_hat+grad out
    qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
    res = sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                           torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy())
    e2e_times = []
    barrier()
    eng.query_points(qh, P, sd.SD_EXACT, out=res)  # warm the host-path buffers
    for i in range(max(3, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.query_points(qh, P, sd.SD_EXACT, out=res)
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.mean(e2e_times))
    te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
    e2e_value = world * pairs_per_rank / float(te.item())

    bvh = None if args.no_bvh else measure_bvh(args, rank, world, local, sd.Engine, dev, stream, flush, peaks)
    if rank == 0:
        achieved = pairs_per_rank * FLOPS_PER_EDGE_PAIR / (ms_max * 1e-3) / 1e12
        # dram read + write of the dominant launch, from the committed ncu
        # capture of this workload (cfg2 fp32, tile-bound kernel):
        # profiles/r1_v6_exact_edge_details.csv (132.6 MB read + 68.2 MB written,
        # the fp64 per-query partial state of the 8 primitive splits)
        traffic = 2.008e8 if (args.config == 2 and not fp64) else None
        roof = {"bound": "fp64-fma" if fp64 else "fp32-fma", "achieved": achieved, "unit": "TFLOP/s",
                "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
                "algorithmic_bytes": Q * 12 + N * 48,
                "kernel": (f"exact_kernel<{'double' if fp64 else 'float'}, "
                           + {1: "point>", 2: "edge, poly> x3 segment launches", 3: "triangle, poly>"}[args.config]
                           + " + finalize (step time)"),
                "algorithmic": f"{FLOPS_PER_EDGE_PAIR} flop x {pairs_per_rank} pairs per step (SURVEY 8d)"}
        if peaks:
            pk = peaks["dfma_tflops"] if fp64 else peaks["ffma_tflops"]
            roof.update({"peak": pk, "frac": achieved / pk,
                         "peak_source": f"in-run {'DFMA' if fp64 else 'FFMA'} microbenchmark (libsdpeaks.so); "
                                        "MEASURED_PEAKS.json has no FP32/FP64 entry",
                         "mufu_frac": pairs_per_rank * MUFU_PER_EDGE_PAIR / (ms_max * 1e-3) / 1e12 / peaks["mufu_tops"],
                         "peaks": peaks})
            # bound-aware roofline = max(flops / P_fma, mufu / P_mufu)
            roof["bound_aware_frac"] = max(roof["frac"], roof["mufu_frac"])
        cpu = None
        if world == 1 and not args.no_cpu:
            import oracle as O
            O.build()
            threads = O.hardware_threads()
            n, secs, _ = cpu_sample(v, w.simplices, w.kinds, wt, q, threads)
            cpu = {"value": n * N / secs, "unit": "pair-evals/s", "cores": threads, "kind": "port",
                   "sample": f"first {n} of {Q} cfg{args.config} queries x {N} primitives ({secs:.1f} s, "
                             f"fp64 oracle port)"}
        line = {
            "metric": "exact pair-evals/s (value+grad)", "value": value, "unit": "pair-evals/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64" if fp64 else "f32", "data": "synthetic",
            "config": {"workload": "cfg1: 4,096 unit-sphere points x 65,536 queries per GPU, exact LSE, alpha=50, fp64 "
                                   "(BASELINE configs[0])" if args.config == 1 else ("cfg2: helix polyline 20,000 edges x 262,144 queries per GPU, exact LSE, "
                                    f"alpha=100, {'fp64' if fp64 else 'fp32'} (BASELINE configs[1])") if args.config == 2 else
                                   (f"cfg3: torus 262,144 triangles x 1,048,576 queries per GPU, exact LSE, "
                                    f"alpha={ALPHA:g}, fp32 (BASELINE configs[2])"),
                       "queries_per_gpu": Q, "primitives": N, "l2": "flushed between timed steps (256 MiB write)",
                       "parallelism": f"query-sharded x{world}, geometry replicated"},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "pair-evals/s", "h2d_bytes_per_step": Q * 3 * 8,
                    "d2h_bytes_per_step": Q * 4 * 8},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "bvh": bvh,
            "step_ms_all": step_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-bvh", action="store_true", help="skip the secondary BVH (cfg4) measurement")
    ap.add_argument("--bvh-strong", action="store_true",
                    help="BVH leg: split ONE cfg4 batch across the ranks by estimated cost (strong scaling)")
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 5],
                    help="exact workload: 2 = BASELINE configs[1] (headline), 1 = configs[0] fp64 points, "
                         "3 = configs[2] torus triangles, 5 = configs[4] primitive-sharded BVH")
    ap.add_argument("--fp64", action="store_true", help="fp64 arithmetic for --config 2")
    ap.add_argument("--m2m", action="store_true", help="mesh-to-mesh evaluations of the paper's timing table rows")
    ap.add_argument("--rows", default="", help="comma-separated sim_rows names for --m2m (default: all)")
    ap.add_argument("--render", action="store_true", help="sphere tracer beta ablation + grid benchmark (callers)")
    ap.add_argument("--exchange", choices=["nccl", "peer"], default="nccl",
                    help="--config 5 merge: NCCL all-reduce or stores into the owners' buffers over peer memory")
    ap.add_argument("--alpha", type=float, default=None, help="alpha for --config 3 (10, 100 or 1000)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == 5:
        run_cfg5(args, rank, world, local)
    elif args.m2m:
        if rank == 0:
            run_m2m(args, rank, world, local)
    elif args.render:
        if rank == 0:
            run_render(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
