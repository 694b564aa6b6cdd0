#!/bin/bash
# Build tuning variants of libnfgpu.so into tools/variants/ (name:flags pairs).
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants; mkdir -p tools/variants
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -diag-suppress 177,550 "$@" -o tools/variants/libnfgpu_$name.so paper_2509_00774_b200/csrc/nfgpu.cu &
}
build v8tg4u2t16 -DNFGPU_TG=4 -DNFGPU_TBR=16
build v8tg4u2t8 -DNFGPU_TG=4 -DNFGPU_TBR=8
build v8tg3u2t8 -DNFGPU_TG=3 -DNFGPU_TBR=8
build v8tg3u2t8w2 -DNFGPU_TG=3 -DNFGPU_TBR=8 -DNFGPU_FWD_WARPS=2 -DNFGPU_ADJ_WARPS=2
build v8tg4u2t8w1 -DNFGPU_TG=4 -DNFGPU_TBR=8 -DNFGPU_FWD_WARPS=1 -DNFGPU_ADJ_WARPS=1
build v8tg5u2t8 -DNFGPU_TG=5 -DNFGPU_TBR=8
build v4tg6u2t16 -DNFGPU_V=4 -DNFGPU_TG=6 -DNFGPU_TBR=16
build v8tg4u4t16 -DNFGPU_TG=4 -DNFGPU_UNROLL=4
wait
ls tools/variants
