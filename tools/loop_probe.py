#!/usr/bin/env python3
"""One persistent-loop launch (a few iterations) and one per-launch step on a workload, for ncu comparisons
of spgm_loop_kernel against fwd_kernel / adj_kernel (profile with -k regex:...)."""
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
ap.add_argument("--workload", default="large")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7, initial=configs.make_scene(w))
eng.sample_device(0, 1, w.batch)
eng.step_staged()
eng.run_loop(a.iters, table=None, seed=0, iter0=1, batch=w.batch, tol=0.0)
print(eng.loop_result())
torch.cuda.synchronize()
