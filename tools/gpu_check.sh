#!/bin/bash
# One GPU verification pass (run under gpurun): smoke, GPU parity tests, bench.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/smoke.log; tail -15 gpurun_out/pytest_gpu.log; tail -c 2500 gpurun_out/bench.log
