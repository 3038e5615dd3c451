#!/bin/bash
# A/B of the few-query traversal modes on the paper-table rows (gpurun, 1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ROWS=${ROWS:-bowl_icosphere,ringtoss_trefoil,bowl_spiky,bunny_bunny,terrain_bunny,terrain_octopus}
MODES=${MODES:-"FRONTIER=1,FRONTIER_G=4 FRONTIER=1,FRONTIER_G=8 FRONTIER=1,FRONTIER_G=16 FRONTIER=1,FRONTIER_G=32 FRONTIER=0,SPLIT="}
for mode in $MODES; do
  env $(echo $mode | tr ',' ' ' | sed 's/\([A-Z_]*=\)/SDGPU_\1/g') timeout 600 python bench.py --m2m --no-cpu --rows $ROWS --steps 5 --warmup 2 2>/dev/null \
    | python -c "import sys,json; l=json.loads(sys.stdin.read()); print('$mode', ' '.join(f\"{r['row'].split(' vs ')[1][:8]}={r['gpu_ms']:.3f}\" for r in l['rows']))"
done
