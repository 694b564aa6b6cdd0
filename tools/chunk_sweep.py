#!/usr/bin/env python3
"""Sweep the flat kernels' work-unit sizes on one workload in one process: for each (forward min chunk,
adjoint min chunk) pair a fresh plan is built (the knobs are read at plan creation) and the forward and
adjoint+prox kernels are timed with CUDA events (median of reps).

    python tools/chunk_sweep.py --workload medium --fwd 64,56,48,40 --adj 128,96,64,56
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
ap.add_argument("--workload", default="medium")
ap.add_argument("--fwd", default="64")
ap.add_argument("--adj", default="128")
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--graph", action="store_true", help="also time whole steps in a CUDA graph")
ap.add_argument("--fit", default="", help="NFGPU_WAVE_FIT values to sweep (default: leave unset)")
a = ap.parse_args()
w = configs.WORKLOADS[a.workload]()
scn = w.scenario
rng = np.random.default_rng(0)
y = (rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)).astype(np.complex64)
st = torch.cuda.current_stream()
import itertools

for fm, am, fit in itertools.product(a.fwd.split(","), a.adj.split(","), a.fit.split(",")):
    if True:
        os.environ["NFGPU_MIN_CHUNK"] = fm
        os.environ["NFGPU_ADJ_MIN_CHUNK"] = am
        if fit:
            os.environ["NFGPU_WAVE_FIT"] = fit
        plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch)
        eng = SPGMEngine(plan, y, eta=1e-2, alpha=1e-6, initial=configs.make_scene(w))
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
        out = {"workload": a.workload, "fwd_min_chunk": int(fm), "adj_min_chunk": int(am), "wave_fit": fit,
               "fwd_ms": float(np.median(f_ms)), "adj_ms": float(np.median(a_ms))}
        if a.graph:
            g = eng.graph(0, w.batch, pairs=4)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(25):
                g.replay()
            e1.record(st)
            torch.cuda.synchronize()
            out["step_ms_graph"] = e0.elapsed_time(e1) / 200
        print(json.dumps(out), flush=True)
        del eng, plan
        torch.cuda.empty_cache()
