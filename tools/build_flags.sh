#!/bin/bash
# Build the device library with extra nvcc flags into variants/<name>.so
# (kernel experiments; select at run time with PPPC_LIB=variants/<name>.so).
#   tools/build_flags.sh stages4 -DPPPC_STAGES=4
set -e
name=$1; shift
mkdir -p variants
/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v "$@" -I include paper_1905_13076_b200/csrc/kernels.cu \
  paper_1905_13076_b200/csrc/spectral.cu paper_1905_13076_b200/csrc/capi.cu paper_1905_13076_b200/csrc/builders.cpp \
  -o variants/$name.so 2> variants/$name.ptxas.log
