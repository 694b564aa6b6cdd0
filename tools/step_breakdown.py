#!/usr/bin/env python3
"""Per-step cost of one rank's slab of Large (the N-GPU per-rank workload on one GPU).

Times K graph-replayed SPGM iterations (device sampler, as bench.py) and the two fused
kernels alone, and prints one JSON line. Under ncu (--metrics gpu__time_duration.sum)
the eager steps it runs first give the per-kernel launch list of a step.

    python tools/step_breakdown.py --zslab 8 [--steps 200] [--eager 2]
"""

from __future__ import annotations

import argparse
import json
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
    ap.add_argument("--zslab", type=int, default=8, help="first Z z-planes (one rank of 64/Z GPUs); 0 = all")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--eager", type=int, default=2, help="eager steps first (for an ncu launch list)")
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    w = configs.WORKLOADS[a.workload]()
    scn = w.scenario
    rng = np.random.default_rng(0)
    y = (rng.standard_normal(scn.n_channels) + 1j * rng.standard_normal(scn.n_channels)).astype(np.complex64)
    zr = (0, a.zslab) if a.zslab else None
    plan = DevicePlan(scn, dtype=w.dtype, device="cuda:0", max_batch=w.batch, z_range=zr)
    s0 = configs.make_scene(w)[plan.vox_offset:plan.vox_offset + plan.n_local]
    eng = SPGMEngine(plan, y, eta=1e-2, alpha=1e-6, initial=s0)
    B = w.batch
    for k in range(a.eager):
        eng.sample_device(0, k, B)
        eng.step_staged()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    g = None if a.no_graph else eng.graph(0, B, pairs=1)

    def run(n):
        if g is not None:
            for _ in range(n // 2):
                g.replay()
        else:
            for _ in range(n):
                eng.sample_device(0, None, B)
                eng.step_staged()

    run(10)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run(a.steps)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    # kernels alone
    f_ms, a_ms = [], []
    for i in range(10):
        eng.sample_device(0, 1000 + i, B)
        yb = eng.ybuf[:B]
        t0, t1, t2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        t0.record(st)
        plan.forward(eng.s, out=yb)
        t1.record(st)
        plan.adjoint_prox(yb, eng.y, eng.s, eng.s_next, eng.eta / B, eng.alpha, eng.stats)
        t2.record(st)
        eng.s, eng.s_next = eng.s_next, eng.s
        torch.cuda.synchronize()
        f_ms.append(t0.elapsed_time(t1))
        a_ms.append(t1.elapsed_time(t2))
    ent = 2.0 * B * plan.n_local
    print(json.dumps({"zslab": a.zslab, "n_local": plan.n_local, "tiles": plan.info()["tiles"], "graph": g is not None,
                      "ms_per_step": ms, "entries_per_s": ent / (ms * 1e-3),
                      "fwd_ms": float(np.median(f_ms)), "adj_ms": float(np.median(a_ms)),
                      "kernels_ms": float(np.median(f_ms) + np.median(a_ms)),
                      "overhead_ms": ms - float(np.median(f_ms) + np.median(a_ms))}), flush=True)


if __name__ == "__main__":
    main()
