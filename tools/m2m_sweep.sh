#!/bin/bash
# A/B of the few-query traversal modes on the paper-table rows (gpurun, 1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ROWS=${ROWS:-bowl_icosphere,ringtoss_trefoil,bowl_spiky,bunny_bunny,terrain_bunny}
for mode in "FRONTIER=1" "FRONTIER=0 SPLIT=" "FRONTIER=0 SPLIT=4" "FRONTIER=0 SPLIT=8"; do
  env $(echo $mode | sed 's/\([A-Z]*=\)/SDGPU_\1/g') timeout 600 python bench.py --m2m --no-cpu --rows $ROWS --steps 5 --warmup 2 2>/dev/null \
    | python -c "import sys,json; l=json.loads(sys.stdin.read()); print('$mode', ' '.join(f\"{r['row'].split(' vs ')[1][:8]}={r['gpu_ms']:.3f}\" for r in l['rows']))"
done
