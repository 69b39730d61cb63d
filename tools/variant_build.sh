#!/bin/bash
# Timing-diagnostic variants of libsrlg.so (detect.cu with -D<FLAG>) for A/B
# runs through tools/libswap.py: tools/variant_build.sh FLAG OUT.so
set -e
L=paper_1805_09246_b200/_lib
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC,-ffp-contract=off -I include -I paper_1805_09246_b200/csrc -D$1 \
  -c paper_1805_09246_b200/csrc/detect.cu -o /tmp/detect_$1.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $2 $L/kernels.o /tmp/detect_$1.o $L/capi.o \
  $L/exact.o -Xlinker -z,defs -lcudart_static -lrt -lpthread -ldl
