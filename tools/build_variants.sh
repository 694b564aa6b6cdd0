#!/bin/bash
# Build tuning variants of libnfgpu.so into tools/variants/.
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants; mkdir -p tools/variants
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -diag-suppress 177,550 "$@" -o tools/variants/libnfgpu_$name.so paper_2509_00774_b200/csrc/nfgpu.cu &
}
build pair0 -DNFGPU_FWD_PAIR=0
build pair1_mb4 -DNFGPU_FWD_PAIR=1 -DNFGPU_MINB_FWD=4
build pair1_mb3 -DNFGPU_FWD_PAIR=1 -DNFGPU_MINB_FWD=3
build pair1_mb3_tree -DNFGPU_FWD_PAIR=1 -DNFGPU_MINB_FWD=3 -DNFGPU_FWD_TREE=1
wait
