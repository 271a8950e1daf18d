#!/bin/bash
# usage: tools/build_variant.sh NAME [-DMACRO=V ...] -- compile a variant .so into _lib/variants/
set -e
cd "$(dirname "$0")/.."
N=$1; shift
mkdir -p paracut_b200/_lib/variants
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode=arch=compute_100a,code=sm_100a -lineinfo -fmad=false \
  -Xcompiler -fPIC -shared "$@" -o paracut_b200/_lib/variants/$N.so paracut_b200/csrc/paracut_b200.cu
