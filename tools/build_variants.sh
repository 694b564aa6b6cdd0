#!/bin/bash
# Build tuning variants of libnfgpu.so into tools/variants/ (select one with NFGPU_LIB=...).
#   tools/build_variants.sh name "-DFLAG=.. -DFLAG2=.." [name "-D..."]...   (default: a base build)
set -e
cd "$(dirname "$0")/.."
rm -rf tools/variants; mkdir -p tools/variants
build() {
  name=$1; shift
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
       -diag-suppress 177,550 "$@" -o tools/variants/libnfgpu_$name.so paper_2509_00774_b200/csrc/nfgpu.cu &
}
if [ $# -eq 0 ]; then set -- base ""; fi
while [ $# -ge 2 ]; do
  # shellcheck disable=SC2086
  build "$1" $2
  shift 2
done
wait
ls tools/variants
