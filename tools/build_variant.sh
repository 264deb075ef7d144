#!/bin/bash
# Build the device library from an alternative kernels.cu (and optionally an
# alternative pppc_internal.h, $3) into variants/<name>.so (kernel experiments;
# select at run time with PPPC_LIB=variants/<name>.so).
set -e
name=$1; src=$2; hdr=$3
mkdir -p variants/tmp_$name
cp paper_1905_13076_b200/csrc/*.cu paper_1905_13076_b200/csrc/*.cpp paper_1905_13076_b200/csrc/*.h paper_1905_13076_b200/csrc/*.cuh variants/tmp_$name/
cp "$src" variants/tmp_$name/kernels.cu
[ -n "$hdr" ] && cp "$hdr" variants/tmp_$name/pppc_internal.h
sed -i 's@#include "../../include/pppc_b200.h"@#include "pppc_b200.h"@' variants/tmp_$name/pppc_internal.h
/usr/local/cuda/bin/nvcc -ccbin /usr/bin/g++ -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v -I include variants/tmp_$name/kernels.cu variants/tmp_$name/spectral.cu \
  variants/tmp_$name/capi.cu variants/tmp_$name/builders.cpp -o variants/$name.so 2> variants/$name.ptxas.log
grep -A2 "propagate_kernelILb0ELi3" variants/$name.ptxas.log | grep "spill\|registers"
rm -rf variants/tmp_$name
