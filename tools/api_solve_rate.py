#!/usr/bin/env python3
"""Iterations/s of the public API (spgm_solve, the reference's entry point) on a BASELINE workload,
with the reference's per-iteration semantics (records, termination check every iteration), against
the engine's device-timed step. One JSON line per sampler.

    python tools/api_solve_rate.py --workload large --iters 100
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.solver import SolverConfig, spgm_solve  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="large")
    ap.add_argument("--iters", type=int, default=100)
    a = ap.parse_args()
    w = configs.WORKLOADS[a.workload]()
    scn = w.scenario
    rng = np.random.default_rng(0)
    y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
    for sampler in ("host", "device"):
        cfg = SolverConfig(eta=1e-2, alpha=1e-6, max_iters=a.iters, tol=1e-300, dtype=w.dtype, flat_batch=w.batch,
                           sampler=sampler)
        spgm_solve(y, scn, SolverConfig(eta=1e-2, alpha=1e-6, max_iters=3, tol=1e-300, dtype=w.dtype,
                                        flat_batch=w.batch, sampler=sampler))  # warm (plan cache)
        t0 = time.perf_counter()
        rep = spgm_solve(y, scn, cfg)
        dt = time.perf_counter() - t0
        print(json.dumps({"workload": a.workload, "sampler": sampler, "iters": rep.iterations, "seconds": dt,
                          "iters_per_s": rep.iterations / dt,
                          "entries_per_s": 2.0 * w.batch * scn.n_voxels * rep.iterations / dt}), flush=True)


if __name__ == "__main__":
    main()
