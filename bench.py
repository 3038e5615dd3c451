#!/usr/bin/env python
"""Benchmark of the B200 smooth-distance engine.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (`metric` "exact pair-evals/s (value+grad)"): BASELINE.json
configs[2], the jittered torus (262,144 triangles) against its 1,048,576
queries, alpha = 100, fp32: a step is one exact pass of d_hat + grad over the
batch (smooth_min_dist_flat for every query, smooth.hpp:189-198). The same
JSON line carries, as extra keys, cfg3 at alpha 10 and 1000, cfg2 (helix,
20,000 edges x 262,144 queries) in fp32 and fp64, and the BVH far-field
metric on configs[3] (cfg4: icosphere(9), 5,242,880 triangles, 4,194,304
queries, alpha 200, beta 0.5), plus a `parity` object: the timed outputs of
every leg checked against the CPU oracle on config-scale samples, and cfg4
Barnes-Hut against exact on 65,536 queries.

Multi-GPU: one process per GPU. Without torchrun, --gpus N > 1 re-launches
this script under torch.distributed.run with N ranks; the world size must
equal --gpus. The BASELINE batch is fixed and split across the ranks
("scaling": "strong"): exact legs by equal contiguous query blocks (uniform
queries, uniform per-pair work), the BVH leg by Hilbert-contiguous blocks of
equal estimated traversal cost (sharding.balanced_ranges). No collective on
the data path (geometry replicated, queries sharded); the BVH leg also
reports the weak-scaling variant (every rank a full cfg4 batch) at N > 1.

--impl reference times the reference CPU evaluator of the same path on this
host's cores: the reference cannot be installed as a package here (a CMake
header library, no Eigen), so its line-faithful fp64 restatement in oracle/
stands in ("kind": "port"). Only that leg, the cpu_baseline legs and the
parity checker execute oracle/.
"""
from __future__ import annotations

import argparse
import ctypes
import glob
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# SURVEY 8(d) canonical algorithmic flops per pair evaluation (S != 1)
FLOPS_PER_PAIR = {0: 20, 1: 62, 2: 192}
FLOPS_BOX_TEST, FLOPS_FAR_TERM = 10, 12
BYTES_NODE, BYTES_LEAF = 32, 100  # fp32 traversal node record; leaf record (96 B) + meta
MUFU_PER_PAIR = {0: 2, 1: 3, 2: 3}  # rsqrt, lg2, ex2 (no reciprocal on certified-positive weights)
SMS = 148
TOL = {"f32": (1e-5, 1e-4), "f64": (1e-10, 1e-9)}  # north_star: relative d_hat / gradient


# ------------------------------------------------------------- processes
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> bool:
    """--gpus N > 1 outside torchrun: run this script under
    torch.distributed.run with N ranks (127.0.0.1 rendezvous) and return
    True (the caller exits with its status)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    sys.exit(rc)


class Run:
    """Process group plumbing: barrier, max / sum over ranks, all-gather of
    small objects (NCCL on GPUs, gloo in --stub runs)."""

    def __init__(self, rank, world, local, backend):
        self.rank, self.world, self.local = rank, world, local
        self.backend = backend
        import torch
        self.torch = torch
        if world > 1:
            import torch.distributed as dist
            if backend == "nccl":
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            else:
                dist.init_process_group("gloo")
            self.dist = dist
        self.dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def reduce(self, xs, op="max"):
        xs = [float(x) for x in (xs if isinstance(xs, (list, tuple)) else [xs])]
        if self.world > 1:
            t = self.torch.tensor(xs, dtype=self.torch.float64, device=self.dev)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
            xs = [float(v) for v in t.cpu().tolist()]
        return xs

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            self.dist.barrier()
            self.dist.destroy_process_group()


def strong_blocks(n: int, world: int):
    """Equal contiguous [lo, hi) blocks of a fixed batch (exact legs)."""
    from paper_2108_10480_b200 import sharding
    return sharding.query_ranges(n, world)


# ------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled DURING the timed
    region: NVML polled every 2 ms from a thread (nvidia-smi -lms 200 as the
    fallback when pynvml is unavailable)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason* bits
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}
    ALL = []  # every sample of the run (the top-level "clocks")

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
        ClockSampler.ALL.extend(self.lines)

    @staticmethod
    def summarize(lines, source="nvml"):
        sm = [x[0] for x in lines]
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(x[1] for x in lines),
                "reasons": sorted(set(n for x in lines for n in x[2])), "samples": len(sm), "source": source}

    def summary(self):
        return self.summarize(self.lines, "nvml" if self.nvml is not None else "nvidia-smi")


# ---------------------------------------------------------------- peaks
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


def compute_peak(peaks, sm_mhz, fp64: bool):
    """Roofline denominator: the largest of the in-run probes and the
    nominal pipe rate at the sampled SM clock (148 SMs x 128 FP32 / 64 FP64
    lanes x 2 flop per FMA)."""
    clk = (sm_mhz or 1965.0) * 1e6
    nominal = SMS * (64 if fp64 else 128) * 2 * clk / 1e12
    cands = {"nominal_at_sampled_clock": nominal}
    if peaks:
        if fp64:
            cands["dfma_probe"] = peaks["dfma_tflops"]
        else:
            cands["ffma_probe"] = peaks["ffma_tflops"]
            if "ffma2_tflops" in peaks:
                cands["ffma2_probe"] = peaks["ffma2_tflops"]
    src = max(cands, key=cands.get)
    return cands[src], src, cands


# the CUDA sources each stamped kernel is built from
STAMP_SOURCES = {
    "exact": ("exact.cu", "exact.h", "pair.cuh", "pair2.cuh", "device_common.cuh", "api.cu", "context.h"),
    "bvh": ("bvh.cu", "traverse.cuh", "layout.cu", "pair.cuh", "pair2.cuh", "device_common.cuh", "api.cu",
            "context.h", "exact.h"),
}


def source_hash(kind: str | None = None) -> str:
    """Hash of the CUDA sources of a kernel family (all of csrc/ without
    `kind`): ncu figures stamped with another hash are stale and not
    reported."""
    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2108_10480_b200", "csrc")
    names = STAMP_SOURCES[kind] if kind else sorted(os.path.basename(p) for p in glob.glob(os.path.join(csrc, "*")))
    for n in names:
        if n.endswith((".cu", ".cuh", ".h", ".cpp")):
            with open(os.path.join(csrc, n), "rb") as f:
                h.update(n.encode() + f.read())
    return h.hexdigest()[:16]


def ncu_stamp(kernel_key: str):
    """Per-launch ncu figures of `kernel_key` (profiles/ncu_stamps.json,
    written by tools/ncu_stamp.py from a capture of the same sources), or
    None when the capture is of different sources."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_stamps.json")) as f:
            st = json.load(f)
    except (OSError, ValueError):
        return None
    e = st.get(kernel_key)
    if not e or e.get("src_sha") != source_hash(kernel_key.split("_")[0]):
        return None
    return e


# ------------------------------------------------------------- timing
def time_device(run, step, stream, flush, steps, warmup, eng=None):
    """W >= 3 untimed steps, then exactly K steps between CUDA events on the
    launching stream with an L2 flush (256 MiB write) before each; barrier
    + synchronize on both sides; max over ranks. With `eng`, the engine's
    own event pairs around its dominant launches are read as well."""
    torch = run.torch
    for _ in range(max(3, warmup)):
        step()
    torch.cuda.synchronize()
    if eng is not None:
        eng.kernel_times()
        eng.set_kernel_timing(True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    run.barrier()
    torch.cuda.synchronize()
    with ClockSampler(run.local) as clk:
        for i in range(steps):
            flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    run.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    kern = None
    if eng is not None:
        kern = eng.kernel_times()
        eng.set_kernel_timing(False)
    ms, kms = run.reduce([float(np.mean(step_ms)), float(np.mean(kern)) if kern is not None and len(kern) else 0.0])
    return {"ms": ms, "step_ms": step_ms, "kernel_ms": kms if kern is not None else None,
            "kernel_launch_groups": int(len(kern)) if kern is not None else 0, "clocks": clk.summary()}


def time_e2e_pipelined(run, eng, qh, P, mode, outs, steps):
    """End to end through the pipelined host API (sd_query_points_async):
    `steps` batches submitted back to back (two in flight, alternating
    pinned output buffers), each with its own H2D of the queries and D2H of
    d_hat + grad; wall clock over all of them, max over ranks."""
    torch = run.torch
    for k in range(2):  # both pipeline slots allocate their buffers before the timing
        eng.query_points_async(qh, P, mode, outs[k])
    eng.wait()
    run.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(steps):
        eng.query_points_async(qh, P, mode, outs[i % 2])
    eng.wait()
    return run.reduce((time.perf_counter() - t0) / steps)[0]


def time_e2e(run, call, steps):
    """End to end through the public host API, wall clock per call (the call
    is blocking: H2D + evaluation + D2H), max over ranks."""
    torch = run.torch
    call()
    times = []
    run.barrier()
    for _ in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    return run.reduce(float(np.mean(times)))[0]


# ------------------------------------------------------------- workloads
def cfg3_workload():
    """BASELINE configs[2]: torus 512 x 256 (262,144 triangles) with vertex
    jitter, 1,048,576 queries uniform in the AABB expanded by 0.5; fp32
    inputs (rounded before the GPU and the oracle see them)."""
    from paper_2108_10480_b200 import configs
    V, T = configs.torus()
    rng = np.random.default_rng([3002, 0])
    lo, hi = V.min(0) - 0.5, V.max(0) + 0.5
    q = rng.uniform(lo, hi, (1048576, 3))
    return configs.quantize(V), T, np.full(len(T), 2, np.uint8), configs.quantize(q)


def cfg2_workload():
    from paper_2108_10480_b200 import configs
    w, q = configs.cfg2(262144, block=0)
    wt = configs.weights_without_triangles(w.simplices, w.kinds, len(w.vertices))
    return w, wt, q


def oracle_objects(v, s, k, wt, nodes=None):
    import oracle as O
    O.build()
    m = O.Mesh.from_arrays(v, s, k)
    ws = O.Weights.from_table(O.WeightTable(wt.A, wt.sup_wtilde, wt.edge_a, wt.tri_stored, wt.poly_index))
    t = O.Tree.from_nodes(nodes) if nodes is not None else None
    return O, m, ws, t


class CpuArm:
    """The CPU implementation of the path timed beside ours: the reference
    itself (oracle/_ref: its unmodified headers compiled with the Eigen
    shim; kind "reference") when that library is present, else the oracle
    restatement (kind "port"). The WeightSet table is fed in (the shim has
    no SVD for the triangle polynomials); the tree is given or built."""

    def __init__(self, v, s, k, wt, nodes=None, build_tree=False):
        from oracle import reference as R
        self.threads = os.cpu_count() or 1
        if R.available():
            self.kind = "reference"
            self.sc = R.Scene(v, s, k, wt)
            if nodes is not None or build_tree:
                self.sc.set_bvh(nodes)
            self.run = lambda q, p, tree: self.sc.query(q, p, tree=tree, threads=self.threads)
        else:
            O, m, ws, t = oracle_objects(v, s, k, wt, nodes)
            if build_tree and t is None:
                t = O.Tree.build(m)
            self.kind, self.threads = "port", O.hardware_threads()
            self.run = lambda q, p, tree: O.query(m, ws, q, p, tree=t if tree else None, threads=self.threads)

    def query(self, q, alpha, alpha_u=600.0, beta=0.0, tree=False):
        import oracle as O
        return self.run(np.ascontiguousarray(q), O.Params(alpha=alpha, alpha_u=alpha_u, beta=beta), tree)


# ------------------------------------------------------------- parity
def parity_stats(got_d, got_g, ref_d, ref_g, alpha, dtype):
    """Both tolerance forms of north_star's relative bound on the same pairs:
    the survey's (error / max(1, |ref|)) and the strict relative one with a
    1/alpha floor for d_hat (|d_hat| < 1/alpha is below the LSE's own
    resolution) and a 1e-3 floor for the gradient norm. +inf must agree."""
    td, tg = TOL[dtype]
    got_d, ref_d = np.asarray(got_d, np.float64), np.asarray(ref_d, np.float64)
    fr, fg = np.isfinite(ref_d), np.isfinite(got_d)
    both = fr & fg
    dd = np.abs(got_d[both] - ref_d[both])
    rd = np.abs(ref_d[both])
    out = {"n": int(len(ref_d)), "finite": int(both.sum()), "inf_mismatch": int((fr != fg).sum()),
           "tol_d_hat": td, "tol_grad": tg}
    if dd.size:
        e1 = dd / np.maximum(1.0, rd)
        e2 = dd / np.maximum(rd, 1.0 / alpha)
        out.update({"d_hat_max_err_survey": float(e1.max()), "d_hat_max_err_strict": float(e2.max()),
                    "d_hat_over_tol_strict": int((e2 > td).sum()), "d_hat_max_abs": float(dd.max())})
    if got_g is not None and ref_g is not None and dd.size:
        gd = np.linalg.norm(np.asarray(got_g)[both] - np.asarray(ref_g)[both], axis=1)
        gn = np.linalg.norm(np.asarray(ref_g)[both], axis=1)
        g1 = gd / np.maximum(1.0, gn)
        g2 = gd / np.maximum(gn, 1e-3)
        out.update({"grad_max_err_survey": float(g1.max()), "grad_max_err_strict": float(g2.max()),
                    "grad_over_tol_strict": int((g2 > tg).sum())})
    out["pass_survey"] = bool(out["inf_mismatch"] == 0 and out.get("d_hat_max_err_survey", 0.0) <= td
                              and out.get("grad_max_err_survey", 0.0) <= tg)
    out["pass_strict"] = bool(out["inf_mismatch"] == 0 and out.get("d_hat_over_tol_strict", 0) == 0
                              and out.get("grad_over_tol_strict", 0) == 0)
    return out


# ------------------------------------------------------------ exact legs
def exact_leg(run, eng, q, prec, N, kind, P, steps, warmup, flush, stream, peaks, e2e_steps=0, q_total=None,
              stamp_key=None):
    """Times one exact configuration on this rank's query block q (fp32 /
    fp64 device buffer, inputs resident), optionally end to end through
    sd_query_points with pinned host buffers. Returns the result dict and
    this rank's (d_hat, grad) of the timed steps (host copies)."""
    import paper_2108_10480_b200 as sd
    torch = run.torch
    fp64 = prec == sd.SD_FP64
    Q = len(q)
    q_total = q_total or Q * run.world
    dev = run.dev
    qd = torch.tensor(q, dtype=torch.float64 if fp64 else torch.float32, device=dev)
    d_hat = torch.empty(Q, dtype=torch.float64, device=dev)
    grad = torch.empty(Q, 3, dtype=torch.float64, device=dev)

    def step():
        eng.query_points_device(qd.data_ptr(), Q, P, sd.SD_EXACT, d_hat.data_ptr(), grad.data_ptr(),
                                stream=stream.cuda_stream)

    t = time_device(run, step, stream, flush, steps, warmup, eng)
    launches = eng.last_launch_count()
    pairs_rank = Q * N
    out = {"value": q_total * N / (t["ms"] * 1e-3), "unit": "pair-evals/s", "ms_per_step": t["ms"],
           "queries": q_total, "queries_per_gpu": Q, "primitives": N, "dtype": "f64" if fp64 else "f32",
           "alpha": P.alpha, "gpu_launches": launches * steps, "clocks": t["clocks"]}
    kms = t["kernel_ms"]
    if kms:
        achieved = FLOPS_PER_PAIR[kind] * pairs_rank / (kms * 1e-3) / 1e12
        peak, src, cands = compute_peak(peaks, t["clocks"].get("sm_mhz"), fp64)
        out["roofline"] = {
            "bound": "fp64-fma" if fp64 else "fp32-fma", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "peak_source": src, "peak_candidates": cands,
            "kernel_ms": kms, "step_ms": t["ms"], "kernel_share_of_step": kms / t["ms"],
            "algorithmic": f"{FLOPS_PER_PAIR[kind]} flop/pair x {pairs_rank} pairs per launch group (SURVEY 8d); "
                           "kernel time = CUDA events on the launching stream around the exact segment launches "
                           "(sd_set_kernel_timing), query sort and finalize excluded",
            "kernel": f"exact_kernel<{'double' if fp64 else 'float'}, {['point', 'edge', 'triangle'][kind]}>"}
        if peaks and not fp64:
            out["roofline"]["mufu_frac"] = MUFU_PER_PAIR[kind] * pairs_rank / (kms * 1e-3) / 1e12 / peaks["mufu_tops"]
        # bytes per launch: the queries in, the primitive records once per
        # query block (staged through shared memory), the outputs out
        out["roofline"]["algorithmic_bytes"] = Q * 12 + N * 4 * [4, 12, 24][kind] + Q * 32
        out["roofline"]["traffic"] = None
        st = ncu_stamp(f"exact_{stamp_key}") if stamp_key else None
        if st:
            out["roofline"]["traffic"] = st.get("dram_bytes")
            out["roofline"]["ncu"] = st
    if e2e_steps:
        qh = torch.tensor(q, dtype=torch.float64).pin_memory().numpy()
        outs = [sd.SmoothResults(torch.empty(Q, dtype=torch.float64).pin_memory().numpy(),
                                 torch.empty(Q, 3, dtype=torch.float64).pin_memory().numpy()) for _ in range(2)]
        tp = time_e2e_pipelined(run, eng, qh, P, sd.SD_EXACT, outs, e2e_steps)
        te = time_e2e(run, lambda: eng.query_points(qh, P, sd.SD_EXACT, out=outs[0]), e2e_steps)
        out["e2e"] = {"value": q_total * N / tp, "unit": "pair-evals/s", "h2d_bytes_per_step": Q * 3 * 8,
                      "d2h_bytes_per_step": Q * 4 * 8, "steps": e2e_steps,
                      "api": "sd_query_points_async (pinned host fp64 queries in, d_hat + grad out; batches "
                             "submitted back to back, two in flight)",
                      "blocking_call": {"value": q_total * N / te, "api": "sd_query_points"}}
    return out, d_hat.cpu().numpy(), grad.cpu().numpy()


PRUNE_BITS = 48.0


def pruned_leg(run, eng, q, prec, N, kind, P, steps, flush, stream, peaks, q_total, full, base_ms, bits=PRUNE_BITS):
    """The same exact configuration with sd_set_exact_pruning(48): an extra
    key, never the headline. Tiles whose terms are below 2^-48 of a lower
    bound of the query's sum are skipped, so `value` is the all-pairs
    EQUIVALENT rate (Q x N / time, skipped pairs counted); every timed
    answer of this rank is compared with the all-pairs kernel's."""
    eng.set_exact_pruning(bits)
    try:
        r, d, g = exact_leg(run, eng, q, prec, N, kind, P, steps, 3, flush, stream, peaks, q_total=q_total)
    finally:
        eng.set_exact_pruning(0.0)
    if "roofline" in r:
        r["roofline_all_pairs"] = r.pop("roofline")
        r["roofline_all_pairs"]["note"] = "counts skipped pairs too; not a pipe utilisation"
    r["unit"] = "pair-evals/s (all-pairs equivalent)"
    r["pruning_bits"] = bits
    r["speedup_over_all_pairs"] = base_ms / r["ms_per_step"]
    d0, g0 = full
    fin = np.isfinite(d0)
    r["vs_all_pairs_kernel"] = {
        "n": int(len(d0)), "inf_mismatch": int((np.isfinite(d) != fin).sum()),
        "d_hat_max_abs": float(np.abs(d[fin] - d0[fin]).max()) if fin.any() else 0.0,
        "grad_max_abs": float(np.abs(g[fin] - g0[fin]).max()) if fin.any() else 0.0,
        "bound": f"relative error of c < N 2^-{bits:g} = {N * 2.0 ** -bits:.1e} (include/sdgpu.h); the rest "
                 "is regrouping of the tile sums (another tile order)"}
    return r, d, g


def cpu_exact_sample(arm, q, alpha, target_s):
    """The CPU arm on a bounded prefix of the queries, sized by a pilot so
    the sample takes about target_s seconds."""
    pilot = max(arm.threads * 2, 32)
    arm.query(q[:pilot], alpha)  # first touch of the scene
    r = arm.query(q[:pilot], alpha)
    n = int(min(len(q), max(pilot, pilot * target_s / max(r.seconds, 1e-3))))
    return n, arm.query(q[:n], alpha)


def run_exact_headline(args, run, peaks, stream, flush, line):
    """cfg3 (BASELINE configs[2]) alpha 100 = the headline; alpha 10 / 1000,
    cfg2 fp32 / fp64 as extra keys; parity of every leg's timed outputs."""
    import paper_2108_10480_b200 as sd
    rank, world = run.rank, run.world
    par = line.setdefault("parity", {})
    # ---- cfg3 torus
    v3, t3, k3, q3 = cfg3_workload()
    eng = sd.Engine(run.local, sd.SD_FP32)
    eng.set_geometry(v3, t3, k3)
    wt3 = eng.build_weights()
    lo, hi = strong_blocks(len(q3), world)[rank]
    qb = q3[lo:hi]
    N3 = len(k3)
    P = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=0.0)
    head, d100, g100 = exact_leg(run, eng, qb, sd.SD_FP32, N3, 2, P, args.steps, args.warmup, flush, stream, peaks,
                                 e2e_steps=max(3, min(args.steps, 10)), q_total=len(q3),
                                 stamp_key="cfg3_f32" if run.world == 1 else None)
    extra = {}
    outs = {100.0: (d100, g100)}
    for alpha in (10.0, 1000.0):
        Pa = sd.SmoothParams(alpha=alpha, alpha_u=600.0, beta=0.0)
        r, d, g = exact_leg(run, eng, qb, sd.SD_FP32, N3, 2, Pa, max(1, min(args.steps, 3)), 3, flush, stream, peaks,
                            q_total=len(q3))
        if alpha >= 1000.0 and "roofline" in r:
            # tiles whose every term is below the -708 mask are skipped (exact,
            # not an approximation): the all-pairs flop rate exceeds the pipe
            r["roofline_all_pairs"] = r.pop("roofline")
            r["roofline_all_pairs"]["note"] = ("counts every pair the reference evaluates; tiles whose terms are all "
                                               "masked (alpha d > 708) are skipped exactly, so frac > 1 is expected")
        extra[f"exact_cfg3_alpha{alpha:g}"] = r
        outs[alpha] = (d, g)
    rp, dp, gp = pruned_leg(run, eng, qb, sd.SD_FP32, N3, 2, P, max(1, min(args.steps, 5)), flush, stream, peaks,
                            len(q3), (d100, g100), head["ms_per_step"])
    extra["exact_cfg3_pruned"] = rp
    outs["pruned"] = (dp, gp)
    eng.close()
    threads = None
    if rank == 0 and not args.no_cpu:
        import oracle as O
        O.build()
        threads = O.hardware_threads()
        # parity: strided samples of the timed outputs (this rank's block)
        _, m, w, _ = oracle_objects(v3, t3, k3, wt3)
        for alpha, nq in ((100.0, 512), (10.0, 256), (1000.0, 256)):
            idx = np.linspace(0, len(qb) - 1, nq).astype(np.int64)
            ref = O.query(m, w, qb[idx], O.Params(alpha=alpha, alpha_u=600.0, beta=0.0), threads=threads)
            d, g = outs[alpha]
            par[f"cfg3_alpha{alpha:g}"] = parity_stats(d[idx], g[idx], ref.d_hat, ref.grad, alpha, "f32")
            par[f"cfg3_alpha{alpha:g}"]["sample"] = f"{nq} evenly spaced timed queries of rank 0's block"
            if alpha == 100.0:
                d, g = outs["pruned"]
                par["cfg3_alpha100_pruned"] = parity_stats(d[idx], g[idx], ref.d_hat, ref.grad, alpha, "f32")
                par["cfg3_alpha100_pruned"]["sample"] = f"the same {nq} queries, sd_set_exact_pruning({PRUNE_BITS:g})"
        if world == 1:
            arm = CpuArm(v3, t3, k3, wt3)
            n, r = cpu_exact_sample(arm, qb, 100.0, 10.0)
            line["cpu_baseline"] = {"value": n * N3 / r.seconds, "unit": "pair-evals/s", "cores": arm.threads,
                                    "kind": arm.kind, "sample": f"first {n} of {len(qb)} cfg3 queries x {N3} "
                                    f"triangles, alpha 100 ({r.seconds:.1f} s, fp64, {arm.kind})"}
    line.update({"metric": "exact pair-evals/s (value+grad)", "value": head["value"], "unit": "pair-evals/s",
                 "ms_per_step": head["ms_per_step"], "dtype": "f32",
                 "config": {"workload": "cfg3: torus R=1 r=0.3, 512x256 grid (262,144 triangles), vertex jitter, "
                                        "1,048,576 queries uniform in the AABB expanded by 0.5, exact LSE, alpha=100, "
                                        "fp32 (BASELINE configs[2])",
                            "queries": len(q3), "queries_per_gpu": len(qb), "primitives": N3,
                            "l2": "flushed between timed steps (256 MiB write)",
                            "parallelism": f"query-sharded x{world} (equal contiguous blocks of the fixed batch), "
                                           "geometry replicated"},
                 "roofline": head.get("roofline"), "e2e": head.get("e2e"), "gpu_launches": head["gpu_launches"],
                 "clocks": head["clocks"]})
    line.update(extra)
    # ---- cfg2 helix (BASELINE configs[1]), fp32 and fp64
    w2, wt2, q2 = cfg2_workload()
    from paper_2108_10480_b200 import configs
    v2, q2 = configs.quantize(w2.vertices), configs.quantize(q2)
    lo, hi = strong_blocks(len(q2), world)[rank]
    qb2 = q2[lo:hi]
    N2 = len(w2.kinds)
    P2 = sd.SmoothParams(alpha=100.0, alpha_u=600.0, beta=0.0)
    res2 = {}
    for prec, key in ((sd.SD_FP32, "exact_cfg2"), (sd.SD_FP64, "exact_cfg2_fp64")):
        e = sd.Engine(run.local, prec)
        e.set_geometry(v2, w2.simplices, w2.kinds)
        e.set_weights(wt2.A, wt2.sup_wtilde, wt2.edge_a, wt2.tri_stored, wt2.poly_index)
        r, d, g = exact_leg(run, e, qb2, prec, N2, 1, P2, args.steps, args.warmup, flush, stream, peaks,
                            e2e_steps=3, q_total=len(q2),
                            stamp_key=(f"cfg2_{'f64' if prec == sd.SD_FP64 else 'f32'}" if run.world == 1 else None))
        r["workload"] = ("cfg2: helix polyline 20,000 edges x 262,144 queries, exact LSE, alpha=100 "
                         "(BASELINE configs[1])")
        line[key] = r
        res2[prec] = (d, g)
        if prec == sd.SD_FP32:
            rp, dp, gp = pruned_leg(run, e, qb2, prec, N2, 1, P2, args.steps, flush, stream, peaks, len(q2), (d, g),
                                    r["ms_per_step"])
            line["exact_cfg2_pruned"] = rp
            res2["pruned"] = (dp, gp)
        else:  # the reference's precision: 64 bits keep the fp64 path's 1e-10 bound
            rp, dp, gp = pruned_leg(run, e, qb2, prec, N2, 1, P2, max(1, min(args.steps, 5)), flush, stream, peaks,
                                    len(q2), (d, g), r["ms_per_step"], bits=64.0)
            line["exact_cfg2_fp64_pruned"] = rp
            res2["pruned64"] = (dp, gp)
        e.close()
    # ---- cfg1 point cloud (BASELINE configs[0]), fp64 as specified
    from paper_2108_10480_b200 import configs as cf
    w1, q1 = cf.cfg1()
    lo, hi = strong_blocks(len(q1), world)[rank]
    qb1 = q1[lo:hi]
    wt1 = cf.weights_without_triangles(w1.simplices, w1.kinds, len(w1.vertices))
    e1 = sd.Engine(run.local, sd.SD_FP64)
    e1.set_geometry(w1.vertices, w1.simplices, w1.kinds)
    e1.set_weights(wt1.A, wt1.sup_wtilde, wt1.edge_a, wt1.tri_stored, wt1.poly_index)
    P1 = sd.SmoothParams(alpha=w1.alpha, alpha_u=600.0, beta=0.0)
    r1, d1, g1 = exact_leg(run, e1, qb1, sd.SD_FP64, len(w1.kinds), 0, P1, args.steps, args.warmup, flush, stream, peaks,
                           e2e_steps=3, q_total=len(q1))
    r1["workload"] = "cfg1: 4,096 unit-sphere points x 65,536 queries, exact LSE, alpha=50, fp64 (BASELINE configs[0])"
    line["exact_cfg1_fp64"] = r1
    e1.close()
    if rank == 0 and not args.no_cpu:
        arm1 = CpuArm(w1.vertices, w1.simplices, w1.kinds, wt1)
        n1, rr1 = cpu_exact_sample(arm1, qb1, w1.alpha, 4.0)
        par["exact_cfg1_fp64"] = parity_stats(d1[:n1], g1[:n1], rr1.d_hat, rr1.grad, w1.alpha, "f64")
        par["exact_cfg1_fp64"]["sample"] = f"first {n1} timed queries of rank 0's block"
        cpu1 = {"value": n1 * len(w1.kinds) / rr1.seconds, "unit": "pair-evals/s", "cores": arm1.threads,
                "kind": arm1.kind, "sample": f"first {n1} cfg1 queries x 4,096 points ({rr1.seconds:.1f} s, fp64)"}
        line["exact_cfg1_fp64"]["cpu_baseline"] = cpu1
        if world == 1:
            line["exact_cfg1_fp64"]["vs_cpu_baseline"] = r1["value"] / cpu1["value"]
    if rank == 0 and not args.no_cpu:
        # the oracle port on a ~7 s prefix of the timed cfg2 queries: the cfg2
        # cpu baseline at the reference's precision and the parity reference
        arm = CpuArm(v2, w2.simplices, w2.kinds, wt2)
        n, r = cpu_exact_sample(arm, qb2, 100.0, 7.0)
        cpu2 = {"value": n * N2 / r.seconds, "unit": "pair-evals/s", "cores": arm.threads, "kind": arm.kind,
                "sample": f"first {n} of {len(qb2)} cfg2 queries x {N2} edges ({r.seconds:.1f} s, fp64, {arm.kind})"}
        for prec, key, dt in ((sd.SD_FP32, "exact_cfg2", "f32"), (sd.SD_FP64, "exact_cfg2_fp64", "f64"),
                              ("pruned", "exact_cfg2_pruned", "f32"), ("pruned64", "exact_cfg2_fp64_pruned", "f64")):
            d, g = res2[prec]
            par[key] = parity_stats(d[:n], g[:n], r.d_hat, r.grad, 100.0, dt)
            par[key]["sample"] = f"first {n} timed queries of rank 0's block"
            line[key]["cpu_baseline"] = cpu2
            line[key]["vs_cpu_baseline"] = line[key]["value"] / cpu2["value"] if world == 1 else None
            if "e2e" in line[key] and world == 1:
                line[key]["e2e_vs_cpu_baseline"] = line[key]["e2e"]["value"] / cpu2["value"]


# ------------------------------------------------------------- BVH leg
def tree_method(sd):
    """BENCH_TREE=median|lbvh|auto (default auto): SD_BVH_AUTO builds the
    reference's median-split tree (build_bvh, bvh.hpp:34-91, on the device)
    and the GPU LBVH and keeps the smaller surface-area cost."""
    t = os.environ.get("BENCH_TREE") or "auto"
    return {"median": sd.SD_BVH_MEDIAN, "lbvh": sd.SD_BVH_LBVH}.get(t, sd.SD_BVH_AUTO)


def tree_name():
    t = os.environ.get("BENCH_TREE") or "auto"
    return {"median": "reference median-split tree built on the GPU", "lbvh": "GPU LBVH"}.get(
        t, "GPU tree (median split or LBVH, smaller surface-area cost)")


def measure_bvh(args, run, stream, flush, peaks, fp64=False):
    """BASELINE configs[3] (cfg4): BVH far-field queries/s. The fixed
    4,194,304-query batch is shared by the ranks (strong scaling): every
    rank holds the whole batch and walks its share of the library's
    32-query packets -- chunks of packets of the Hilbert-sorted batch dealt
    round robin (sd_query_points_device_shard: regional locality within a
    chunk, balance across chunks, no cost model, no collective). The timed
    outputs are then checked against the oracle on 65,536 queries (decision
    hash, counters, d_hat, grad) and Barnes-Hut against exact on the same
    queries. --shard-world W --shard-rank R runs one rank's share on a
    single GPU (tests of the sharded path; the value is that rank's rate)."""
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import configs, sharding
    torch = run.torch
    rank, world = run.rank, run.world
    W, R = (world, rank) if world > 1 else (max(1, args.shard_world), args.shard_rank)
    sharded = W > 1
    t0 = time.perf_counter()
    w, q = configs.cfg4()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    Q_total = len(q)
    eng = sd.Engine(run.local, sd.SD_FP64 if fp64 else sd.SD_FP32)
    eng.set_geometry(v, w.simplices, w.kinds)
    tw = time.perf_counter()
    wt = eng.build_weights()
    tw = time.perf_counter() - tw
    tb = time.perf_counter()
    eng.build_bvh(tree_method(sd))
    tb = time.perf_counter() - tb
    P = sd.SmoothParams(alpha=w.alpha, alpha_u=600.0, beta=w.beta)
    qd = torch.tensor(q, dtype=torch.float64 if fp64 else torch.float32, device=run.dev)
    d_hat = torch.full((Q_total,), float("nan"), dtype=torch.float64, device=run.dev)
    grad = torch.empty(Q_total, 3, dtype=torch.float64, device=run.dev)
    leaves = torch.zeros(Q_total, dtype=torch.int64, device=run.dev)
    far = torch.zeros(Q_total, dtype=torch.int64, device=run.dev)
    hsh = torch.zeros(Q_total, dtype=torch.int64, device=run.dev)

    def step(counters=False):
        kw = dict(leaves_ptr=leaves.data_ptr() if counters else None, far_ptr=far.data_ptr() if counters else None,
                  hash_ptr=hsh.data_ptr() if counters else None, stream=stream.cuda_stream)
        if sharded:
            eng.query_points_device_shard(qd.data_ptr(), Q_total, P, W, R, d_hat.data_ptr(), grad.data_ptr(), **kw)
        else:
            eng.query_points_device(qd.data_ptr(), Q_total, P, sd.SD_BVH, d_hat.data_ptr(), grad.data_ptr(), **kw)

    step(counters=True)  # also uploads the traversal layout; counters + decision hash of the batch
    torch.cuda.synchronize()
    counted = (d_hat.cpu().numpy(), leaves.cpu().numpy(), far.cpu().numpy(), hsh.cpu().numpy().view(np.uint64))
    mine = ~np.isnan(counted[0]) if sharded else np.ones(Q_total, bool)  # this rank's queries (cfg4 has no NaN)
    Q = int(mine.sum())
    setup_s = time.perf_counter() - t0
    L, F = float(counted[1][mine].sum()), float(counted[2][mine].sum())
    t = time_device(run, step, stream, flush, args.steps, args.warmup, eng)
    launches = eng.last_launch_count()
    ms, kms = t["ms"], t["kernel_ms"]
    got_d, got_g = d_hat.cpu().numpy(), grad.cpu().numpy()
    # end to end through the pipelined host API; with several ranks each
    # takes an equal contiguous block of the Morton-sorted batch (the host
    # API has no packet-sharded form)
    if sharded:
        order = sharding.morton_order(q)
        lo, hi = sharding.query_ranges(Q_total, W)[R]
        qe = np.ascontiguousarray(q[order[lo:hi]])
    else:
        qe = q
    qh = torch.tensor(qe, dtype=torch.float64).pin_memory().numpy()
    outs = [sd.SmoothResults(torch.empty(len(qe), dtype=torch.float64).pin_memory().numpy(),
                             torch.empty(len(qe), 3, dtype=torch.float64).pin_memory().numpy()) for _ in range(2)]
    ne2e = max(3, min(args.steps, 10))
    tp = time_e2e_pipelined(run, eng, qh, P, sd.SD_BVH, outs, ne2e)
    te = time_e2e(run, lambda: eng.query_points(qh, P, sd.SD_BVH, out=outs[0]), ne2e)
    q_job = Q_total if world > 1 or not sharded else Q  # a virtual shard reports its own rate
    e2e = {"value": q_job / tp, "unit": "queries/s", "h2d_bytes_per_step": len(qe) * 24,
           "d2h_bytes_per_step": len(qe) * 32, "steps": ne2e,
           "api": "sd_query_points_async (pinned host fp64 queries in, d_hat + grad out; batches submitted back "
                  "to back, two in flight)" + ("; per rank an equal Morton block of the batch" if sharded else ""),
           "blocking_call": {"value": q_job / te, "api": "sd_query_points"}}
    L, F, Qs = run.reduce([L, F, float(Q)], "sum")
    pops = 2 * (L + F) - Qs
    flops = (FLOPS_BOX_TEST * pops + FLOPS_FAR_TERM * F + FLOPS_PER_PAIR[2] * L) / world
    nbytes = (BYTES_NODE * pops + BYTES_LEAF * L) / world
    out = {"metric": "BVH queries/s (value+grad)", "value": q_job / (ms * 1e-3), "unit": "queries/s",
           "scaling": "strong", "e2e": e2e, "ms_per_step": ms, "queries": Q_total, "queries_per_gpu": Q,
           "primitives": len(w.kinds),
           "workload": "cfg4: icosphere(9) with radial displacement, 5,242,880 triangles, 4,194,304 queries "
                       "(half uniform in [-1.5,1.5]^3, half within 0.02 of the surface), alpha=200, "
                       f"beta=0.5, {'fp64' if fp64 else 'fp32'}, {tree_name()} (BASELINE configs[3])",
           "dtype": "f64" if fp64 else "f32", "clocks": t["clocks"],
           "per_query": {"leaves": L / Qs, "far_field": F / Qs, "nodes_popped": pops / Qs},
           "setup_s": {"total": setup_s, "build_weights": tw, "build_tree": tb},
           "gpu_launches": launches * args.steps}
    if sharded:
        out["sharding"] = {"world": W, "rank": R, "virtual": world == 1,
                           "split": "chunks of 32-query packets of the Hilbert-sorted batch dealt round robin "
                                    "(sd_query_points_device_shard)"}
    if kms:
        peak, src, cands = compute_peak(peaks, t["clocks"].get("sm_mhz"), fp64)
        achieved = flops / (kms * 1e-3) / 1e12
        roof = {"bound": "issue (L1/L2-resident tree; see ncu)", "achieved": achieved, "unit": "TFLOP/s",
                "peak": peak, "peak_source": src, "frac": achieved / peak, "kernel_ms": kms,
                "kernel_share_of_step": kms / ms,
                "algorithmic": "10 flop/popped node + 12/far term + 192/exact tri leaf (this run's counters); "
                               "kernel time = CUDA events around the traversal launch (sort and finalize excluded)",
                "modelled_l1l2_bytes_per_launch": nbytes,
                "modelled_l1l2_gbs": nbytes / (kms * 1e-3) / 1e9,
                "modelled_bytes": "32 B per popped node + 100 B per exact leaf, served from L1/L2, not DRAM",
                "traffic": None}
        st = ncu_stamp("bvh_cfg4_f64" if fp64 else "bvh_cfg4_f32") if not sharded else None
        if st:
            roof["traffic"] = st.get("dram_bytes")
            roof["ncu"] = st
        out["roofline"] = roof
    par = None
    if rank == 0 and not args.no_cpu:
        par = bvh_parity(eng, v, w, wt, q, np.nonzero(mine)[0], counted, got_d, got_g, P, not sharded)
        if world == 1 and not sharded:
            out["cpu_baseline"] = par.pop("cpu_baseline")
    if world > 1 and not args.no_weak:
        # weak scaling variant: every rank a full cfg4 batch of its own
        _, qw = configs.cfg4(block=rank)
        qw = configs.quantize(qw)
        qwd = torch.tensor(qw, dtype=torch.float64 if fp64 else torch.float32, device=run.dev)
        dw = torch.empty(len(qw), dtype=torch.float64, device=run.dev)
        gw = torch.empty(len(qw), 3, dtype=torch.float64, device=run.dev)
        tw2 = time_device(run, lambda: eng.query_points_device(qwd.data_ptr(), len(qw), P, sd.SD_BVH, dw.data_ptr(),
                                                                gw.data_ptr(), stream=stream.cuda_stream),
                          stream, flush, args.steps, args.warmup)
        out["weak"] = {"value": world * len(qw) / (tw2["ms"] * 1e-3), "unit": "queries/s", "scaling": "weak",
                       "ms_per_step": tw2["ms"], "queries_per_gpu": len(qw)}
    eng.close()
    return out, par


def bvh_parity(eng, v, w, wt, q, sel, counted, got_d, got_g, P, full_batch, n_sample=65536):
    """cfg4 at config scale: the oracle port on the SAME tree (exported in
    the reference layout) and table, on n_sample queries (half from each
    half of the distribution at N=1): decision hash and counters of every
    query, d_hat / grad of the timed outputs, plus Barnes-Hut against the
    GPU exact path on the same queries (acceptance [1]: d_hat_BH <= d_hat
    + tol) and GPU exact against the oracle's exact on a 32-query subset."""
    import paper_2108_10480_b200 as sd
    O, m, ws, t = oracle_objects(v, w.simplices, w.kinds, wt, eng.export_bvh())
    threads = O.hardware_threads()
    Q = len(q)
    qb = q  # sample indices address the whole batch; sel = this rank's queries
    if full_batch:
        half = Q // 2
        idx = np.concatenate([np.linspace(0, half - 1, n_sample // 2), np.linspace(half, Q - 1, n_sample // 2)])
    else:
        idx = sel[np.linspace(0, len(sel) - 1, min(n_sample, len(sel))).astype(np.int64)]
    idx = np.unique(idx.astype(np.int64))
    p = O.Params(alpha=P.alpha, alpha_u=P.alpha_u, beta=P.beta)
    ref = O.query(m, ws, qb[idx], p, tree=t, threads=threads)
    cd, cl, cf, ch = counted
    out = {"n": int(len(idx)), "sample": "32,768 evenly spaced queries from each half of the distribution"
           if full_batch else f"{len(idx)} evenly spaced queries of rank 0's block",
           "hash_mismatch": int((ch[idx] != ref.decision_hash).sum()),
           "leaves_mismatch": int((cl[idx] != ref.leaves).sum()),
           "far_field_mismatch": int((cf[idx] != ref.far_field).sum()),
           "timed_equals_counted_run": bool(np.array_equal(cd[idx], got_d[idx], equal_nan=True))}
    out.update(parity_stats(got_d[idx], got_g[idx], ref.d_hat, ref.grad, P.alpha, "f32"))
    arm = CpuArm(v, w.simplices, w.kinds, wt, nodes=eng.export_bvh())
    rr = arm.query(qb[idx], P.alpha, P.alpha_u, P.beta, tree=True)
    if arm.kind == "reference":  # the oracle restatement against the reference itself on the same sample
        out["oracle_equals_reference"] = bool(all(np.array_equal(getattr(ref, f), getattr(rr, f), equal_nan=True)
                                                  for f in ("d_hat", "grad", "leaves", "far_field")))
    # the CPU baseline proper: a ~8 s sample of the same batch (both halves)
    n = int(min(Q, max(len(idx), len(idx) * 8.0 / max(rr.seconds, 1e-3))))
    half = Q // 2
    big = np.concatenate([qb[:n // 2], qb[half:half + n - n // 2]])
    rb = arm.query(big, P.alpha, P.alpha_u, P.beta, tree=True)
    out["cpu_baseline"] = {"value": len(big) / rb.seconds, "unit": "queries/s", "cores": arm.threads,
                           "kind": arm.kind,
                           "sample": f"{len(big)} cfg4 queries (both halves) on the exported GPU-built tree, "
                                     f"fp64, {arm.kind}, {rb.seconds:.1f} s"}
    # Barnes-Hut vs exact on the same queries (GPU exact, checked below)
    ex = eng.query_points(qb[idx], sd.SmoothParams(alpha=P.alpha, alpha_u=P.alpha_u, beta=0.0), sd.SD_EXACT)
    fin = np.isfinite(ex.d_hat) & np.isfinite(got_d[idx])
    diff = got_d[idx][fin] - ex.d_hat[fin]
    out["bvh_minus_exact"] = {"n": int(fin.sum()), "max": float(diff.max()), "mean": float(diff.mean()),
                              "min": float(diff.min()), "violations_bh_le_exact_plus_1e-5": int((diff > 1e-5).sum()),
                              "criterion": "acceptance [1] (T/acceptance.cpp:76-115): d_hat_BH <= d_hat_exact + tol"}
    sub = idx[np.linspace(0, len(idx) - 1, 32).astype(np.int64)]
    rex = O.query(m, ws, qb[sub], O.Params(alpha=P.alpha, alpha_u=P.alpha_u, beta=0.0), threads=threads)
    pos = np.searchsorted(idx, sub)
    out["gpu_exact_vs_oracle_exact"] = parity_stats(ex.d_hat[pos], ex.grad[pos], rex.d_hat, rex.grad, P.alpha, "f32")
    out["gpu_exact_vs_oracle_exact"]["sample"] = "32 of the sample queries x 5,242,880 triangles"
    if eng.precision == sd.SD_FP32:
        # every timed output of this rank against the fp64 tree path on the
        # same tree (pinned to the reference by the sample above at fp64:
        # test_config4_parity_65536_queries), decisions included
        e64 = sd.Engine(eng.device, sd.SD_FP64)
        e64.set_geometry(v, w.simplices, w.kinds)
        e64.set_weight_table(wt)
        e64.set_bvh(eng.export_bvh())
        r64 = e64.smooth_min_dist(qb[sel], P)
        e64.close()
        wb = parity_stats(got_d[sel], got_g[sel], r64.d_hat, r64.grad, P.alpha, "f32")
        wb.update({"n": int(len(sel)), "hash_mismatch": int((ch[sel] != r64.decision_hash).sum()),
                   "sample": "every timed query of this rank (whole batch at N=1) vs the fp64 GPU tree path"})
        out["whole_batch_vs_fp64"] = wb
    return out


# ----------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch
    torch.cuda.set_device(local)
    run = Run(rank, world, local, "nccl")
    dev = run.dev
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    peaks = measure_peaks(local)
    line = {"metric": "exact pair-evals/s (value+grad)", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "data": "synthetic (seeded generators of BASELINE configs[1..3])"}
    t0 = time.perf_counter()
    run_exact_headline(args, run, peaks, stream, flush, line)
    if not args.no_bvh:
        bvh, par = measure_bvh(args, run, stream, flush, peaks)
        line["bvh"] = bvh
        if par is not None:
            line.setdefault("parity", {})["cfg4_bvh"] = par
    if peaks:
        line["peaks_probe"] = peaks
    line["clocks_all"] = ClockSampler.summarize(ClockSampler.ALL)
    line["bench_seconds"] = time.perf_counter() - t0
    if rank == 0:
        line["gpu_launches_note"] = "libsdgpu.so kernels launched inside the headline's timed region"
        print(json.dumps(line), flush=True)
    run.close()


# ------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The reference's own CPU path, on our headline's config, metric and
    unit: the reference itself (oracle/_ref, its unmodified headers
    compiled with the Eigen shim; else the oracle port), fp64, on all host
    threads, a bounded query sample per step. The cfg3 WeightSet is the
    reference construction restated by the oracle (the shim has no SVD);
    the `bvh` object does the same for cfg4 on the reference's own
    build_bvh tree."""
    if rank != 0:
        return
    import oracle as O
    O.build()
    v3, t3, k3, q3 = cfg3_workload()
    m = O.Mesh.from_arrays(v3, t3, k3)
    wt = O.Weights.build(m).table
    arm = CpuArm(v3, t3, k3, wt)
    N = len(k3)
    pilot = max(arm.threads * 2, 32)
    arm.query(q3[:pilot], 100.0)  # first touch of the scene
    r = arm.query(q3[:pilot], 100.0)
    n = int(min(len(q3), max(pilot, pilot * 2.0 / max(r.seconds, 1e-3))))  # ~2 s per step
    for i in range(args.warmup):
        arm.query(q3[:n], 100.0)
    times = []
    for i in range(args.steps):
        lo = (i * n) % max(1, len(q3) - n)
        times.append(arm.query(q3[lo:lo + n], 100.0).seconds)
    t = float(np.mean(times))
    value = n * N / t
    line = {
        "impl": "reference", "metric": "exact pair-evals/s (value+grad)", "value": value, "unit": "pair-evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generators of BASELINE configs[1..3])",
        "config": {"workload": "cfg3: torus 262,144 triangles, 1,048,576 queries, exact LSE, alpha=100 "
                               "(BASELINE configs[2]); a bounded sample of the batch per step",
                   "queries_per_step": n, "primitives": N, "parallelism": f"{arm.threads} host threads",
                   "implementation": ("the reference's smooth_min_dist_flat (smooth.hpp:189-198) batched by its "
                                      "parallel_for, unmodified headers compiled with an Eigen-subset shim "
                                      "(oracle/_ref)") if arm.kind == "reference" else
                                     "the oracle's fp64 restatement of the reference (oracle/)"},
        "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": arm.threads, "kind": arm.kind,
                         "sample": f"{n} of {len(q3)} cfg3 queries x {N} triangles per step"},
        "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_bvh:
        line["bvh"] = reference_bvh()
    print(json.dumps(line), flush=True)


def reference_bvh(target_s=10.0):
    """The reference's own CPU path for the BVH metric on cfg4: its
    build_bvh tree (built here by the reference, or by the oracle port),
    the WeightSet from the oracle's restated construction, a bounded query
    sample (both halves of the distribution) on all host threads."""
    import oracle as O
    from paper_2108_10480_b200 import configs
    t0 = time.perf_counter()
    w, q = configs.cfg4()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    m = O.Mesh.from_arrays(v, w.simplices, w.kinds)
    wt = O.Weights.build(m).table
    del m
    arm = CpuArm(v, w.simplices, w.kinds, wt, build_tree=True)
    setup = time.perf_counter() - t0
    half = len(q) // 2
    pick = lambda n: np.concatenate([q[:n // 2], q[half:half + n - n // 2]])
    pilot = max(arm.threads * 16, 1024)
    r = arm.query(pick(pilot), w.alpha, 600.0, w.beta, tree=True)  # also warms the tree pages
    n = int(min(262144, max(pilot, pilot * target_s / max(r.seconds, 1e-3))))
    r = arm.query(pick(n), w.alpha, 600.0, w.beta, tree=True)
    return {"metric": "BVH queries/s (value+grad)", "value": n / r.seconds, "unit": "queries/s",
            "workload": "cfg4 (BASELINE configs[3]): icosphere(9), 5,242,880 triangles, alpha=200, beta=0.5, "
                        "the reference's build_bvh tree, WeightSet from the restated construction",
            "cpu_baseline": {"value": n / r.seconds, "unit": "queries/s", "cores": arm.threads, "kind": arm.kind,
                             "sample": f"{n} cfg4 queries (half from each half of the distribution), "
                                       f"{r.seconds:.1f} s"},
            "setup_s": setup}


# ------------------------------------------------------------ stub arm
def run_stub(args, rank, world, local):
    """CPU stand-in for the multi-GPU plumbing (tests/test_bench_spawn.py):
    the same spawn path, process group (gloo), strong split of a fixed
    batch, max-over-ranks timing and all-gathered result checksum, with a
    numpy exact LSE over a tiny point cloud as the evaluator."""
    run = Run(rank, world, local, "gloo")
    rng = np.random.default_rng(7)
    pts = rng.standard_normal((64, 3))
    q = rng.uniform(-2, 2, (4096, 3))
    lo, hi = strong_blocks(len(q), world)[rank]

    def evaluate(qs, alpha=50.0):
        d = np.linalg.norm(qs[:, None, :] - pts[None], axis=2)
        m = d.min(1)
        return m - np.log(np.exp(-alpha * (d - m[:, None])).sum(1)) / alpha

    for _ in range(max(3, args.warmup)):
        evaluate(q[lo:hi])
    run.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = evaluate(q[lo:hi])
    ms = run.reduce(1e3 * (time.perf_counter() - t0) / max(1, args.steps))[0]
    parts = run.gather({"rank": rank, "lo": lo, "hi": hi, "sum": float(out.sum())})
    if rank == 0:
        full = float(evaluate(q).sum())
        print(json.dumps({"metric": "stub exact pair-evals/s", "value": len(q) * len(pts) / (ms * 1e-3),
                          "unit": "pair-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": ms, "scaling": "strong", "blocks": [(p["lo"], p["hi"]) for p in parts],
                          "checksum": sum(p["sum"] for p in parts), "checksum_single": full,
                          "backend": run.backend}), flush=True)
    run.close()


# ------------------------------------------------------ other configs
def run_cfg5(args, rank, world, local):
    """BASELINE configs[4]: mixed scene (16.8M triangles + 1M edges + 1M
    points), 16,777,216 queries, alpha 100, beta 0.5, PRIMITIVE-sharded over
    the ranks (Morton-contiguous shards, one GPU-built tree per shard, global
    WeightSet), per-query fp64 partials merged with ONE NCCL all-reduce,
    then sd_finalize_device. Strong scaling (fixed total work). --exact: the
    exact path (smooth_min_dist_flat, smooth.hpp:189-198) over the same
    primitive shards and merge, on an evenly spaced subset of the queries
    (--exact-queries, default 65,536: the whole batch would be 3.2e14 pair
    evaluations per step)."""
    import torch
    import paper_2108_10480_b200 as sd
    from paper_2108_10480_b200 import configs, sharding
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    run = Run(rank, world, local, "nccl")
    t0 = time.perf_counter()
    w, q = configs.cfg5()
    v, q = configs.quantize(w.vertices), configs.quantize(q)
    exact = args.exact
    mode = sd.SD_EXACT if exact else sd.SD_BVH
    if exact:
        q = np.ascontiguousarray(q[np.linspace(0, len(q) - 1, args.exact_queries).astype(np.int64)])
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
    if exact and args.prune > 0:
        eng.set_exact_pruning(args.prune)
    tb = time.perf_counter()
    # BENCH_TREE=median builds the reference's median-split tree instead (A/B)
    if not exact:
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
            eng.query_points_scatter(qd.data_ptr(), Q, P, mode, table.data_ptr(), world, rank, per,
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
        eng.query_points_device(qd.data_ptr(), Q, P, mode, d_hat.data_ptr(), c_ptr=buf.data_ptr(),
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
        ot = None if exact else O.Tree.from_nodes(eng.export_bvh())
        nsamp = (64 if args.prune > 0 else 16) if exact else 4096
        sample = np.linspace(0, Q - 1, nsamp).astype(np.int64)
        r = O.query(om, ow, q[sample], O.Params(alpha=w.alpha, alpha_u=600.0, beta=0.0 if exact else w.beta),
                    tree=None if exact else ot, threads=threads)
        got = d_hat[torch.as_tensor(sample, device=dev)].cpu().numpy()
        ok = np.isfinite(r.d_hat)
        NP = len(w.kinds)
        cpu = {"value": (nsamp * NP if exact else nsamp) / r.seconds, "unit": "pair-evals/s" if exact else "queries/s",
               "cores": threads, "kind": "port",
               "sample": f"{nsamp} evenly spaced cfg5 queries "
                         + ("x all primitives (exact)" if exact else "on the exported GPU-built tree")
                         + f", fp64 oracle port, {r.seconds:.2f} s",
               "max_abs_d_hat_diff": float(np.abs(got[ok] - r.d_hat[ok]).max()) if ok.any() else 0.0,
               "parity": parity_stats(got, None, r.d_hat, None, w.alpha, "f32")}
        del om, ow, ot
    if rank == 0:
        NP = len(w.kinds)
        line = {"metric": ("exact pair-evals/s (value+grad), primitive-sharded" if exact else
                           "BVH queries/s (value+grad), primitive-sharded"),
                "value": (Q * NP if exact else Q) / (ms * 1e-3),
                "unit": "pair-evals/s" if exact else "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": {"workload": "cfg5: 64 rotated cfg3 tori (16,777,216 triangles) + 1M edges + 1M points, "
                                       + (f"{Q:,} evenly spaced of the 16,777,216 queries, exact LSE" if exact else
                                          "16,777,216 queries uniform in the scene AABB, beta=0.5")
                                       + ", alpha=100, fp32 (BASELINE configs[4])",
                           "parallelism": f"primitive-sharded x{world} (Morton shards, {tree_name()} per shard), "
                                          + ("partials stored into the owners' symmetric buffers over peer memory "
                                             "by the evaluation's own finalize epilogue (sd_query_points_scatter), "
                                             "owner-side reduce + finalize" if exchange == "peer" else
                                             f"one NCCL all_reduce(SUM) of 4 fp64 per query; exchange={exchange}"),
                           "primitives_per_gpu": len(sh.kinds), "l2": "flushed between timed steps"},
                "pruning_bits": (args.prune if exact else None),
                "finite_fraction": fin, "gpu_launches": launches[0] * args.steps, "cpu_baseline": cpu,
                "setup_s": {"total": setup, "generate": tg, "build_weights": tw, "build_tree": tb},
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    run.close()



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



def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline and oracle parity legs")
    ap.add_argument("--no-bvh", action="store_true", help="skip the BVH (cfg4) leg")
    ap.add_argument("--no-weak", action="store_true", help="N > 1: skip the weak-scaling BVH variant")
    ap.add_argument("--config", type=int, default=0, choices=[0, 5],
                    help="0 = the default line (cfg3 headline + cfg2 + cfg4), 5 = configs[4] primitive-sharded")
    ap.add_argument("--exact", action="store_true", help="--config 5: the exact path instead of the BVH path")
    ap.add_argument("--exact-queries", type=int, default=65536, help="--config 5 --exact: evenly spaced queries")
    ap.add_argument("--prune", type=float, default=0.0,
                    help="--config 5 --exact: sd_set_exact_pruning bits (0 = every pair, the default)")
    ap.add_argument("--bvh-fp64", action="store_true", help="run only the BVH leg, in fp64")
    ap.add_argument("--fp64", action="store_true", help="--render in fp64")
    ap.add_argument("--m2m", action="store_true", help="mesh-to-mesh evaluations of the paper's timing table rows")
    ap.add_argument("--rows", default="", help="comma-separated sim_rows names for --m2m (default: all)")
    ap.add_argument("--render", action="store_true", help="sphere tracer beta ablation + grid benchmark (callers)")
    ap.add_argument("--exchange", choices=["nccl", "peer"], default="nccl",
                    help="--config 5 merge: NCCL all-reduce or stores into the owners' buffers over peer memory")
    ap.add_argument("--stub", action="store_true", help="CPU stand-in evaluator over gloo (plumbing tests)")
    ap.add_argument("--shard-world", type=int, default=1, help=argparse.SUPPRESS)  # one rank's share on 1 GPU (tests)
    ap.add_argument("--shard-rank", type=int, default=0, help=argparse.SUPPRESS)
    args = ap.parse_args()
    maybe_spawn(args)
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    if args.stub:
        run_stub(args, rank, world, local)
    elif args.impl == "reference":
        run_reference(args, rank, world)
    elif args.config == 5:
        run_cfg5(args, rank, world, local)
    elif args.m2m:
        if rank == 0:
            run_m2m(args, rank, world, local)
    elif args.render:
        if rank == 0:
            run_render(args, rank, world, local)
    elif args.bvh_fp64:
        import torch
        torch.cuda.set_device(local)
        run = Run(rank, world, local, "nccl")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device=run.dev)
        out, par = measure_bvh(args, run, torch.cuda.current_stream(run.dev), flush, measure_peaks(local), fp64=True)
        if rank == 0:
            out.update({"n_gpus": world, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                        "vs_baseline": None, "data": "synthetic", "parity": par})
            print(json.dumps(out), flush=True)
        run.close()
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
