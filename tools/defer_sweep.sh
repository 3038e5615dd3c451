#!/bin/bash
# Deferred-tail threshold sweep for the K3 packet walk (cfg4 BVH leg of
# bench.py); run under gpurun, 1 GPU. SDGPU_DEFER = 0 is the plain packet walk.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for T in ${DEFER_LIST:-0 4 8 12 16 24}; do
  for CAP in ${CAP_LIST:-64}; do
    SDGPU_DEFER=$T SDGPU_DEFER_CAP=$CAP timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/defer_${T}_${CAP}.log 2>&1
    python - "$T" "$CAP" gpurun_out/defer_${T}_${CAP}.log <<'PY'
import json, sys
line = [l for l in open(sys.argv[3]) if l.startswith("{")]
if not line: print("T", sys.argv[1], "cap", sys.argv[2], "FAILED"); sys.exit()
b = json.loads(line[-1])["bvh"]
print(f"T {sys.argv[1]:>2} cap {sys.argv[2]:>3}: {b['ms_per_step']:.2f} ms  {b['value']:.3e} q/s  pops {b['per_query']['nodes_popped']:.1f} far {b['per_query']['far_field']:.1f}")
PY
  done
done
