for b in 0 32 40 48 64; do K1_TIME=3 K1_PRUNE=$b python tools/k1_run.py 3 100 2>&1 | grep ms/step | sed "s/^/prune $b: /"; done
K1_TIME=3 python tools/k1_run.py 3 100000 2>&1 | grep ms/step | sed "s/^/floor (all masked): /"
K1_TIME=3 K1_PRUNE=48 python tools/k1_run.py 3 10 2>&1 | grep ms/step | sed "s/^/prune 48: /"
K1_TIME=3 K1_PRUNE=48 python tools/k1_run.py 3 1000 2>&1 | grep ms/step | sed "s/^/prune 48: /"
for b in 0 32 48; do K1_TIME=20 K1_PRUNE=$b python tools/k1_run.py 2 100 2>&1 | grep ms/step | sed "s/^/prune $b: /"; done
python -m pytest tests/test_gpu_parity.py -x -q -k "prun" 2>&1 | tail -2
