#!/bin/bash
# ncu evidence for the bench workload (run under gpurun, 1 GPU):
# plain run first (must exit 0), then the launch list and one full capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-cpu ${BENCH_ARGS}"
$CMD > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain.log; exit 1; }
[ -n "$SKIP_LAUNCHES" ] || ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-exact_kernel} -s ${SKIP:-3} -c ${COUNT:-3} -o gpurun_out/${PROF:-prof_exact} $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
