#!/bin/bash
# ncu evidence for the BVH leg (cfg4 traversal); run under gpurun, 1 GPU.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu"
$CMD > gpurun_out/plain_bvh.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_bvh.log; exit 1; }
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bvh.csv $CMD > gpurun_out/ncu_launches_bvh.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:pair_kernel -s 2 -c 1 -o gpurun_out/prof_bvh $CMD > gpurun_out/ncu_full_bvh.log 2>&1; echo "full rc=$?"
true
