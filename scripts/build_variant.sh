#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...] -> paper_1907_13428_b200/lib/libfdg_NAME.so
set -e
name=$1; shift
cd "$(dirname "$0")/.."
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  --diag-suppress 177 "$@" -o paper_1907_13428_b200/lib/libfdg_$name.so \
  paper_1907_13428_b200/csrc/fdg_kernels.cu paper_1907_13428_b200/csrc/fdg_api.cu
