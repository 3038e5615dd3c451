#!/bin/bash
# Round evidence on one GPU (run under gpurun): the default bench line, the
# launch list of a short bench, and one ncu --set full capture each of the
# exact triangle kernel (cfg3, 262,144 queries) and the K3 traversal (cfg4).
# Every ncu command runs only after the same command exited 0 without ncu.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
[ -n "$SKIP_BENCH" ] || { python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; }
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
if [ -z "$SKIP_LAUNCHES" ]; then
  $CMD > gpurun_out/short.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv $CMD \
    > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
fi
# the full headline launch (cfg3: 1,048,576 queries x 262,144 triangles)
python tools/k1_run.py 3 100 > gpurun_out/k1_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:exact_kernel -s 1 -c 1 -o gpurun_out/prof_k1 \
  python tools/k1_run.py 3 100 > gpurun_out/k1_ncu.log 2>&1; echo "k1 rc=$?"
[ -n "$SKIP_K3" ] || tools/k3_ncu.sh
