#!/bin/bash
# Build tuning variants of libnfgpu.so into tools/variants/ (select one with NFGPU_LIB=...).
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants; mkdir -p tools/variants
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -diag-suppress 177,550 "$@" -o tools/variants/libnfgpu_$name.so paper_2509_00774_b200/csrc/nfgpu.cu &
}
build base
build w1 -DNFGPU_FWD_WARPS=1 -DNFGPU_ADJ_WARPS=1 -DNFGPU_MINB_FWD=16 -DNFGPU_MINB_ADJ=16
build w2 -DNFGPU_FWD_WARPS=2 -DNFGPU_ADJ_WARPS=2 -DNFGPU_MINB_FWD=8 -DNFGPU_MINB_ADJ=8
wait
ls tools/variants
