#!/bin/bash
# ncu --set full of one K3 launch (cfg4, tools/k3_ab.py, the non-hash
# traversal of the first warm-up step); run under gpurun, 1 GPU.
#   VARIANT="SDGPU_LEAF_QUEUE=1" KREGEX=pair_kernel tools/k3_ncu.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python tools/k3_ab.py ${VARIANT:-SDGPU_LEAF_QUEUE=1} --steps 1 --reps 1"
$CMD > gpurun_out/k3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-pair_kernel} -s 1 -c 1 \
    -o gpurun_out/${OUT:-prof_k3} $CMD > gpurun_out/k3_ncu.log 2>&1; echo "ncu rc=$?"
