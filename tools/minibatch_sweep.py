#!/usr/bin/env python3
"""BASELINE config 3: minibatch sweep on the Large geometry.

|B| in {256, 1024, 4096, 16384, 65536} plus full-batch proximal gradient (ISTA, |B| = M),
fixed seed, 100 iterations each, complex64. Reports iterations/s and entries/s, with
the objective F(s) = (1/2M)||y - A s||^2 + λ||s||_1 against wall time. The objective is
evaluated off the timed path at checkpoints (a full-M forward). Flat minibatches come
from the device sampler. ISTA uses the full channel set every iteration (solver.py:275, 286).

    python tools/minibatch_sweep.py [--iters 100] [--every 10] [--out profiles/r01_minibatch_sweep.csv]
"""

from __future__ import annotations

import argparse
import csv
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_00774_b200 import configs  # noqa: E402
from paper_2509_00774_b200.plan import DevicePlan  # noqa: E402
from paper_2509_00774_b200.sharding import ShardedSetup  # noqa: E402
from paper_2509_00774_b200.solver import SPGMEngine  # noqa: E402


def sweep(scn, y, eta: float, alpha: float, lam: float, iters: int = 100, every: int = 25,
          batches=(256, 1024, 4096, 16384, 65536, "M"), dev=None, dtype: str = "c64"):
    """Run the sweep; returns (summary per batch size, objective-vs-time rows). Flat batches are drawn on
    the device (fixed seed); ISTA (|B| = M) steps on the full channel set (structured kernels). Device time
    (CUDA events around the iterations only); the objective is evaluated between segments, untimed."""
    dev = dev or torch.device("cuda", 0)
    M, N = scn.n_channels, scn.n_voxels
    obj_plan = DevicePlan(scn, dtype=dtype, device=dev)
    obj_plan.prepare_full()
    y_dev = obj_plan._as_dev(y, M, "y")

    def objective(s: torch.Tensor) -> float:
        r = obj_plan.forward(s) - y_dev
        return float(0.5 * (r.abs().double() ** 2).sum().item() / M + lam * s.abs().double().sum().item())

    rows, summary = [], []
    st = torch.cuda.current_stream()
    for bs in batches:
        B = M if bs == "M" else int(bs)
        plan = DevicePlan(scn, dtype=dtype, device=dev, max_batch=B)
        eng = SPGMEngine(plan, y, eta, alpha)
        if B == M:
            eng.stage(np.arange(M))
            eng.step_staged()  # warm-up (kernel attributes), then restart from s = 0
        else:
            eng.sample_device(configs.SEEDS["minibatch"], 0, B)
            eng.step_staged()
        eng.s.zero_()
        torch.cuda.synchronize()
        t_total = 0.0
        f0 = objective(eng.s)
        rows.append({"batch": B, "iter": 0, "elapsed_s": 0.0, "objective": f0})
        for k0 in range(0, iters, every):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for k in range(k0, min(iters, k0 + every)):
                if B < M:
                    eng.sample_device(configs.SEEDS["minibatch"], k, B)
                eng.step_staged()
            e1.record(st)
            torch.cuda.synchronize()
            t_total += e0.elapsed_time(e1) / 1e3
            rows.append({"batch": B, "iter": min(iters, k0 + every), "elapsed_s": t_total,
                         "objective": objective(eng.s)})
        ips = iters / t_total
        summary.append({"batch": B, "iters": iters, "seconds": t_total, "iters_per_s": ips,
                        "entries_per_s": 2.0 * B * N * ips, "structured": plan.staged_structured,
                        "initial_objective": f0, "final_objective": rows[-1]["objective"],
                        "objective_vs_time": [[r["elapsed_s"], r["objective"]] for r in rows if r["batch"] == B]})
        del eng, plan
        torch.cuda.empty_cache()
    del obj_plan
    torch.cuda.empty_cache()
    return summary, rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--batches", default="256,1024,4096,16384,65536,M")
    ap.add_argument("--out", default="gpurun_out/minibatch_sweep.csv")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    w = configs.WORKLOADS["large"]()
    scn = w.scenario
    M = scn.n_channels
    setup = ShardedSetup(scn, dtype="c64", device=dev, z_range=None)
    y = configs.add_noise(setup.forward_full(configs.make_scene(w)), 0.0)
    sigma = configs.noise_sigma(y, w.snr_db)
    y = configs.add_noise(y, sigma)
    L = setup.lipschitz(n_iters=20)
    lam = 1e-3 * setup.max_abs_adjoint(y) / M
    setup.release()
    batches = [b if b == "M" else int(b) for b in a.batches.split(",")]
    summary, rows = sweep(scn, y, 1.0 / L, lam / L, lam, a.iters, a.every, batches, dev)
    for line in summary:
        print(json.dumps({k: v for k, v in line.items() if k != "objective_vs_time"}), flush=True)
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    with open(a.out, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=["batch", "iter", "elapsed_s", "objective"])
        wr.writeheader()
        wr.writerows(rows)


if __name__ == "__main__":
    main()
