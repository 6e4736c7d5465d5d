#!/bin/bash
# Builds a variant of the product library with extra -D flags into
# tools/libconvgpu_<tag>.so (select it with CONVGPU_LIB=... for A/B timing).
# usage: tools/build_variant.sh tag -DCVG_TILE_CHUNK=8 ...
tag=$1; shift
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC "$@" \
  -o tools/libconvgpu_${tag}.so paper_1711_00289_b200/csrc/convgpu.cu
