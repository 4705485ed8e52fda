#!/bin/bash
# Build an experimental variant of the library with extra -D flags:
#   scripts/build_variant.sh NAME -DFOO -DBAR  ->  paper_1711_08604_b200/lib/ab/NAME.so
name=$1; shift
mkdir -p paper_1711_08604_b200/lib/ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -shared -Xcompiler -fPIC "$@" -o paper_1711_08604_b200/lib/ab/$name.so paper_1711_08604_b200/csrc/afd_capi.cu
