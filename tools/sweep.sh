#!/bin/bash
# Time every tools/variants/*.so on the given workloads (run on the GPU box).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for wl in ${WORKLOADS:-large medium}; do
  for so in tools/variants/*.so; do
    NFGPU_LIB=$so timeout 300 python tools/time_kernels.py --workload $wl 2>>gpurun_out/sweep.err
  done
done
