#!/bin/bash
# Builds the A/B inputs the ab*.sh scripts compare, from the tree alone:
#   scripts/ab_build.sh A <git-rev>   -> abtest/liblfe_A.so built from <git-rev>'s csrc/ + include/
#   scripts/ab_build.sh B             -> abtest/liblfe_B.so built from the working tree
# and, for the per-source-line scripts (ncu_lines.py, sass_range.py), abtest/kf.sass:
#   the SASS of the working tree's fused kernel with line info (nvdisasm -c -g).
# abtest/ is scratch (git-ignored, but it travels to the GPU box with gpurun).
set -e
cd "$(dirname "$0")/.."
mkdir -p abtest
tag=${1:?usage: ab_build.sh A|B [git-rev]}
src=$PWD
if [ -n "$2" ]; then
  src=$(mktemp -d)
  git archive "$2" paper_1304_3992_b200/csrc include | tar -x -C "$src"
fi
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared"
nvcc $FLAGS -I "$src/include" -I "$src/paper_1304_3992_b200/csrc" -o "abtest/liblfe_$tag.so" \
  "$src"/paper_1304_3992_b200/csrc/*.cu
if [ -z "$2" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -cubin -I include \
    -I paper_1304_3992_b200/csrc -o abtest/kernel_fused.sm_100a.cubin paper_1304_3992_b200/csrc/kernel_fused_v0.cu
  nvdisasm -c -g abtest/kernel_fused.sm_100a.cubin > abtest/kf.sass
fi
echo "built abtest/liblfe_$tag.so from ${2:-the working tree}"
