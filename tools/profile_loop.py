#!/usr/bin/env python3
"""Two launches of the persistent SPGM loop on a BASELINE workload (for ncu -k regex:spgm_loop -s 1 -c 1):
a warm-up launch, then the profiled one.

    python tools/profile_loop.py --workload medium --iters 20
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="medium")
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7, initial=configs.make_scene(w))
for _ in range(2):
    eng.run_loop(a.iters, table=None, seed=0, iter0=1, batch=w.batch, tol=0.0)
    torch.cuda.synchronize()
print(a.workload, eng.loop_result())
