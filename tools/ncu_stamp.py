"""Stamp the per-launch ncu figures of one capture into profiles/ncu_stamps.json
under a key bench.py looks up (roofline.traffic and the issue figures), with
the hash of the CUDA sources the capture was taken of: bench.py reports a
stamp only while the sources still hash the same.
  python tools/ncu_stamp.py <capture.ncu-rep> <key> [kernel-substring]
keys: exact_cfg3_f32, exact_cfg2_f32, bvh_cfg4_f32, ..."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

rep, key = sys.argv[1], sys.argv[2]
sub = sys.argv[3] if len(sys.argv) > 3 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
units = dict(zip(h, rows[1]))
sel = [dict(zip(h, r)) for r in rows[2:] if sub in r[h.index("Kernel Name")]]
if not sel:
    raise SystemExit(f"no kernel matching {sub!r} in {rep}")
d = sel[0]


def val(name, scale=1.0):
    v = d.get(name)
    if v in (None, "", "n/a"):
        return None
    x = float(v.replace(",", ""))
    u = units.get(name, "")
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "msecond": 1e-3, "ms": 1e-3,
            "usecond": 1e-6, "us": 1e-6, "nsecond": 1e-9, "ns": 1e-9, "second": 1, "s": 1}.get(u, 1)
    return x * mult * scale


stamp = {
    "kernel": d["Kernel Name"],
    "src_sha": bench.source_hash(key.split("_")[0]),
    "capture": os.path.relpath(rep, ROOT),
    "duration_s": val("gpu__time_duration.sum"),
    "dram_bytes": (val("dram__bytes_read.sum") or 0) + (val("dram__bytes_write.sum") or 0),
    "dram_read_bytes": val("dram__bytes_read.sum"),
    "dram_write_bytes": val("dram__bytes_write.sum"),
    "l2_hit_pct": val("lts__t_sector_hit_rate.pct"),
    "l1_hit_pct": val("l1tex__t_sector_hit_rate.pct"),
    "warp_instructions": val("smsp__inst_executed.sum"),
    "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "avg_active_lanes": val("smsp__thread_inst_executed_per_inst_executed.ratio"),
    "fma_pipe_pct": val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": val("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
    "xu_inst_pct": val("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "registers": val("launch__registers_per_thread"),
    "warps_active_pct": val("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "note": "one ncu --set full --clock-control none capture (cold cache, serialised): shares and bytes per launch, "
            "not absolute times",
}
path = os.path.join(ROOT, "profiles", "ncu_stamps.json")
stamps = json.load(open(path)) if os.path.exists(path) else {}
stamps[key] = stamp
with open(path, "w") as f:
    json.dump(stamps, f, indent=1, sort_keys=True)
print(json.dumps({key: stamp}, indent=1))
