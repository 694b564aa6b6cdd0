#!/usr/bin/env python3
"""Time the fused forward and adjoint+prox kernels on a BASELINE workload (CUDA events,
median of reps, steady state). Used for tuning sweeps: NFGPU_LIB selects a library build.

    NFGPU_LIB=tools/variants/libnfgpu_x.so python tools/time_kernels.py --workload large
"""
import argparse
import json
import os
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
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--zslab", type=int, default=0, help="time one rank's slab: the first Z z-planes (0 = all)")
ap.add_argument("--dtype", default=None, help="c64 or c128 (default: the workload's)")
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
rng = np.random.default_rng(0)
y = (rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)).astype(np.complex64)
zr = (0, a.zslab) if a.zslab else None
plan = DevicePlan(scn, dtype=a.dtype or w.dtype, device="cuda:0", max_batch=w.batch, z_range=zr)
s0 = configs.make_scene(w)[plan.vox_offset:plan.vox_offset + plan.n_local]
eng = SPGMEngine(plan, y, eta=1e-2, alpha=1e-6, initial=s0)
st = torch.cuda.current_stream()
f_ms, a_ms = [], []
for i in range(a.reps + 3):
    eng.sample_device(0, i, w.batch)
    yb = eng.ybuf[: w.batch]
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(st)
    plan.forward(eng.s, out=yb)
    e1.record(st)
    plan.adjoint_prox(yb, eng.y, eng.s, eng.s_next, eng.eta / w.batch, eng.alpha, eng.stats)
    e2.record(st)
    eng.s, eng.s_next = eng.s_next, eng.s
    torch.cuda.synchronize()
    if i >= 3:
        f_ms.append(e0.elapsed_time(e1))
        a_ms.append(e1.elapsed_time(e2))
entries = w.batch * plan.n_local
fm, am = float(np.median(f_ms)), float(np.median(a_ms))
print(json.dumps({"lib": os.environ.get("NFGPU_LIB", "default"), "workload": a.workload, "zslab": a.zslab,
                  "fwd_ms": fm, "adj_ms": am,
                  "fwd_Gentry_s": entries / fm / 1e6, "adj_Gentry_s": entries / am / 1e6,
                  "step_Gentry_s": 2 * entries / (fm + am) / 1e6}))
