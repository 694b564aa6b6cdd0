#!/bin/bash
# A/B timing of the in-tree library against tools/variants/*.so (run on the GPU box).
# usage: tools/ab.sh "large medium" "0 8"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for wl in ${1:-large}; do
  for z in ${2:-0}; do
    for rep in 1 2; do
      for so in paper_2509_00774_b200/libnfgpu.so tools/variants/*.so; do
        echo -n "$so $wl z=$z: "
        NFGPU_LIB=$so timeout 300 python tools/time_kernels.py --workload $wl --zslab $z 2>>gpurun_out/ab.err | tail -1
      done
    done
  done
done
