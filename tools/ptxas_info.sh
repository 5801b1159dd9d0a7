#!/bin/bash
# usage: tools/ptxas_info.sh [extra nvcc flags]  -- registers / spills of the pricing kernels
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xptxas -v -I include -I paper_1205_0106_b200/csrc "$@" -c paper_1205_0106_b200/csrc/kernels.cu -o /tmp/ptxas_info.o 2>&1 |
  grep -A3 "Compiling entry function '_ZN4qmcg.*\(price_kernel\|gen_z\)" | grep -o "price_kernelILi[^N]*\|gen_z_kernelILb[^E]*\|Used [0-9]* registers\|[0-9]* bytes spill stores" | paste - - - | head -24
