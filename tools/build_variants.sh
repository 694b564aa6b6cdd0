#!/bin/bash
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants; mkdir -p tools/variants
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -diag-suppress 177,550 "$@" -o tools/variants/libnfgpu_$name.so paper_2509_00774_b200/csrc/nfgpu.cu &
}
build exact
build noreduce -DNFGPU_EXACT_REDUCE=0
wait
