#!/bin/bash
# Build libsdgpu.so variants for A/B timing on the GPU box:
#   tools/build_ab.sh NAME [git-rev|-] [EXTRA nvcc flags]
# copies paper_2108_10480_b200/ (at the working tree, or at git-rev) to a
# scratch dir, builds it with EXTRA, and leaves ablibs/NAME/libsdgpu.so
# (git-ignored, travels with gpurun). tools/lib_ab.py times them.
set -e
cd "$(dirname "$0")/.."
NAME=$1; REV=${2:--}; shift 2 || true
T=$(mktemp -d)
if [ "$REV" = "-" ]; then cp -r paper_2108_10480_b200 include "$T/"; else git archive "$REV" paper_2108_10480_b200 include | tar -x -C "$T"; fi
rm -rf "$T/paper_2108_10480_b200/build"
make -s -C "$T/paper_2108_10480_b200" -j8 libsdgpu.so EXTRA="$*" > "$T/log" 2>&1 || { cat "$T/log"; exit 1; }
mkdir -p ablibs/$NAME && cp "$T/paper_2108_10480_b200/libsdgpu.so" ablibs/$NAME/
grep -A4 "Compiling entry function '_ZN5sdgpu13pair_kernel_qIfNS_10PointVisitIfEELb0ELb0ELb1E" "$T/paper_2108_10480_b200/build/bvh.ptxas.log" | grep -i "used" | sed "s/^/$NAME: /"
rm -rf "$T"
