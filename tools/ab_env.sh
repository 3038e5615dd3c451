#!/bin/bash
# A/B of traversal switches on the cfg4 BVH leg of bench.py (run under
# gpurun, 1 GPU). Usage: AB="SDGPU_LEAF_QUEUE=0 SDGPU_LEAF_QUEUE=1" tools/ab_env.sh
# (each word is one run's environment; '+' joins several variables).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for cfg in ${AB:-SDGPU_LEAF_QUEUE=0 SDGPU_LEAF_QUEUE=1}; do
  for rep in $(seq ${REPS:-1}); do
    log=gpurun_out/ab_${cfg//[^A-Za-z0-9_]/_}_$rep.log
    env ${cfg//+/ } timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu ${BENCH_ARGS} > $log 2>&1
    python - "$cfg" $log <<'PY'
import json, sys
line = [l for l in open(sys.argv[2]) if l.startswith("{")]
if not line: print(sys.argv[1], "FAILED"); sys.exit()
j = json.loads(line[-1]); b = j.get("bvh") or {}
print(f"{sys.argv[1]:40s} exact {j['ms_per_step']:.3f} ms | bvh {b.get('ms_per_step', float('nan')):.2f} ms {b.get('value', 0):.3e} q/s e2e {b.get('e2e', {}).get('value', 0):.3e}")
PY
  done
done
