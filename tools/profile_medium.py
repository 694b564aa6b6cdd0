#!/usr/bin/env python3
"""One per-launch SPGM step on BASELINE Medium (for ncu -k regex:"fwd_kernel|adj_kernel")."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402

w = configs.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "medium"]()
scn = w.scenario
rng = np.random.default_rng(0)
y = rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)
plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
eng = SPGMEngine(plan, y, eta=1e-3, alpha=1e-7, initial=configs.make_scene(w))
for k in range(3):
    eng.sample_device(0, k, w.batch)
    eng.step_staged()
torch.cuda.synchronize()
