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
build base_tree0 -DNFGPU_FWD_TREE=0
build tree1
build tree1_mb5 -DNFGPU_MINB_FWD=4 -DNFGPU_MINB_ADJ=5
build tree1_mb6 -DNFGPU_MINB_FWD=5 -DNFGPU_MINB_ADJ=6
build tree1_t8tg3_mb5 -DNFGPU_TBR=8 -DNFGPU_TG=3 -DNFGPU_MINB_FWD=5 -DNFGPU_MINB_ADJ=5
wait
for f in tools/variants/*.so; do echo $f; done
