#!/bin/bash
# fp64 exact-kernel sweep: queries per thread x launch-bounds CTA floor,
# cfg1 (points) and cfg2 --fp64 (edges). Output: gpurun_out/fp64_sweep.txt
mkdir -p gpurun_out
out=gpurun_out/fp64_sweep.txt
: > $out
for q in 1 2 4; do for mb in 1 2; do
  for cfg in "--config 1" "--config 2 --fp64"; do
    r=$(SDGPU_FP64_QPT=$q SDGPU_FP64_MINB=$mb timeout 300 python bench.py $cfg --no-bvh --no-cpu --steps 5 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), '%.3e' % d['value'])")
    echo "qpt=$q minb=$mb $cfg -> $r" >> $out
  done
done; done
cat $out
for q in 1 2 4; do for mb in 1 2; do
  SDGPU_FP64_QPT=$q SDGPU_FP64_MINB=$mb timeout 300 python tools/fp64_tri_sweep.py 32768 >> $out 2>&1
done; done
cat $out
