#!/usr/bin/env python3
"""Minimal SPGM steps on a BASELINE workload for ncu captures (no setup solves).

    python tools/profile_step.py [--workload large] [--steps 3]
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="large")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dtype", default=None)
    a = ap.parse_args()
    w = configs.WORKLOADS[a.workload]()
    scn = w.scenario
    rng = np.random.default_rng(0)
    y = (rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)).astype(np.complex64)
    s0 = configs.make_scene(w)
    plan = DevicePlan(scn, dtype=a.dtype or w.dtype, device="cuda:0", max_batch=w.batch)
    eng = SPGMEngine(plan, y, eta=1e-2, alpha=1e-6, initial=s0)
    for k in range(a.steps):
        eng.sample_device(0, k, w.batch)
        eng.step_staged()
    torch.cuda.synchronize()
    print("ok", plan.info())


if __name__ == "__main__":
    main()
