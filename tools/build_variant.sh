#!/bin/bash
# Tools only: build libsrlg.so with detect.cu compiled under extra -D flags,
# for A/B runs against the default build (SRLG_TOOLS_LIB=<out>, tools/libswap.py).
# Usage: tools/build_variant.sh <tag> -DNAME=VALUE ...   -> gpurun_in/libsrlg_<tag>.so
set -e
tag=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
lib=$root/paper_1805_09246_b200/_lib
out=$root/gpurun_in
mkdir -p "$out"
nvcc=/usr/local/cuda/bin/nvcc
arch="-gencode arch=compute_100a,code=sm_100a"
$nvcc $arch -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off \
  "$@" -I "$root/include" -I "$root/paper_1805_09246_b200/csrc" \
  -c "$root/paper_1805_09246_b200/csrc/detect.cu" -o "$out/detect_$tag.o"
$nvcc $arch -shared -o "$out/libsrlg_$tag.so" "$lib/kernels.o" "$out/detect_$tag.o" "$lib/capi.o" \
  "$lib/exact.o" -Xlinker -z,defs -lcudart_static -lrt -lpthread -ldl
echo "$out/libsrlg_$tag.so"
