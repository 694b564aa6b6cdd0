#!/bin/bash
# Sweep the forward/adjoint warp-unit targets at several slab sizes (run on the GPU box).
cd "$(dirname "$0")/.."
for z in ${ZSLABS:-8 16 0}; do
  for t in ${TARGETS:-1184 2368 4736 9472 14208 18944 28416}; do
    NFGPU_FWD_TARGET=$t NFGPU_ADJ_TARGET=$t python tools/time_kernels.py --workload ${WL:-large} --zslab $z | sed "s/^{/{\"target\": $t, /"
  done
done
