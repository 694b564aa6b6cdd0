#!/usr/bin/env python3
"""Where the host time of one spgm_solve goes on a BASELINE workload (persistent-loop path): wall clock of
repeated solves and a cProfile of one.

    python tools/solve_overhead.py --workload medium [--iters 300]
"""
import argparse
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.solver import SolverConfig, spgm_solve  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="medium")
ap.add_argument("--iters", type=int, default=None)
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
iters = a.iters or w.iters
cfg = SolverConfig(eta=1e-3, alpha=1e-7, max_iters=iters, tol=1e-300, dtype=w.dtype, flat_batch=w.batch, rng_seed=0)
spgm_solve(y, scn, cfg)
walls = []
for _ in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    spgm_solve(y, scn, cfg)
    walls.append(time.perf_counter() - t0)
print({"workload": a.workload, "iters": iters, "walls_ms": [round(x * 1e3, 2) for x in walls],
       "us_per_iter_median": round(float(np.median(walls)) / iters * 1e6, 2)})
pr = cProfile.Profile()
pr.enable()
spgm_solve(y, scn, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
