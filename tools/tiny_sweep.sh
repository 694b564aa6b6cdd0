#!/bin/bash
# tiny_loop_kernel work split sweep on BASELINE Small (NFGPU_TINY_JC channels per forward item, NFGPU_TINY_CC
# channel chunks per voxel block in the adjoint)
for jc in 1 2 4; do for cc in 4 9 18 32; do
  echo -n "jc=$jc cc=$cc "; NFGPU_TINY_JC=$jc NFGPU_TINY_CC=$cc python tools/loop_rate.py --workload small --iters 2000 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['loop_us_per_iter'],2))"
done; done
