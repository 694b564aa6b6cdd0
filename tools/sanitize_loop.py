#!/usr/bin/env python3
"""Small persistent-loop launches for compute-sanitizer (memcheck / racecheck / synccheck): both loop kernels,
both dtypes, table and device samplers, a tolerance stop and a time-budget stop."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import ArrayGeometry, FrequencyGrid, ImagingScenario, Vec3, VoxelGrid  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402
import os  # noqa: E402

rng = np.random.default_rng(1)
tx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (5, 2)), np.zeros(5)])
rx = tuple(Vec3(*p) for p in np.c_[rng.uniform(-0.1, 0.1, (7, 2)), np.zeros(7)])
scn = ImagingScenario(array=ArrayGeometry(tx, rx), frequencies=FrequencyGrid(57e9, 64e9, 6),
                      voxels=VoxelGrid(center=Vec3(0, 0, 0.35), extent=(0.1, 0.06, 0.05), dims=(21, 10, 6)))
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
for tiny in ("1", "0"):
    os.environ["NFGPU_TINY"] = tiny
    for dtype in ("c64", "c128"):
        plan = DevicePlan(scn, dtype=dtype, device="cuda:0", max_batch=40)
        eng = SPGMEngine(plan, y, 1e-3, 1e-6)
        tab = np.stack([np.sort(rng.choice(scn.n_channels, 40, replace=False)) for _ in range(3)])
        eng.run_loop(3, table=tab, tol=0.0)
        print(tiny, dtype, eng.loop_result())
        eng.run_loop(4, table=None, seed=3, iter0=1, batch=33, tol=1e9)
        print(tiny, dtype, eng.loop_result())
        eng.run_loop(5, table=None, seed=3, iter0=1, batch=17, tol=0.0, time_budget_s=0.0)
        print(tiny, dtype, eng.loop_result())
        torch.cuda.synchronize()
