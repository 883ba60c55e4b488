#!/bin/bash
# Build the CUDA library with extra nvcc flags into paper_2510_05485_b200/lib_<name>.so (A/B runs).
# usage: tools/build_variant.sh <name> [nvcc flags...]
cd "$(dirname "$0")/../paper_2510_05485_b200/csrc"
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --threads 0 "$@" \
  tb_runtime.cu tb_kernel_sparse.cu tb_kernel_pair.cu tb_kernel_multi.cu tb_kernel_group.cu plugin.cu \
  -o ../lib_$name.so
