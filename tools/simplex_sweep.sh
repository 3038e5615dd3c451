#!/bin/bash
# A/B of the simplex-query kernels on the paper-table rows (gpurun, 1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
ROWS=${ROWS:-bowl_icosphere,bowl_spiky,terrain_octopus,bunny_bunny,plane_bunny,slide_sphere,ringtoss_trefoil,street_motorcycle}
for k in ${KERNELS:-warp frontier}; do
  for gw in ${GWS:-16}; do
    SDGPU_SIMPLEX_GW=$gw SDGPU_SIMPLEX_KERNEL=$k timeout 900 python bench.py --m2m --no-cpu --rows $ROWS --steps 5 \
      --warmup 2 2>/dev/null | TAG="$k$gw" python -c "
import os, sys, json
l = json.loads(sys.stdin.read())
print(os.environ['TAG'], ' '.join(f\"{r['row'].split(' vs ')[1][:8]}={r['gpu_ms']:.3f}\" for r in l['rows']))"
  done
done
