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
    M, N = scn.n_channels, scn.n_voxels
    setup = ShardedSetup(scn, dtype="c64", device=dev, z_range=None)
    y = configs.add_noise(setup.forward_full(configs.make_scene(w)), 0.0)
    sigma = configs.noise_sigma(y, w.snr_db)
    y = configs.add_noise(y, sigma)
    L = setup.lipschitz(n_iters=20)
    lam = 1e-3 * setup.max_abs_adjoint(y) / M
    eta, alpha = 1.0 / L, lam / L
    y_dev = setup.plan._as_dev(y, M, "y")

    def objective(s: torch.Tensor) -> float:
        pred = setup.plan.forward(s)
        r = pred - y_dev
        return float(0.5 * (r.abs() ** 2).sum().item() / M + lam * s.abs().sum().item())

    rows = []
    for bs in a.batches.split(","):
        B = M if bs == "M" else int(bs)
        plan = DevicePlan(scn, dtype="c64", device=dev, max_batch=B)
        eng = SPGMEngine(plan, y, eta, alpha)
        if B == M:
            eng.stage(np.arange(M))
        st = torch.cuda.current_stream()
        t_total = 0.0
        rows.append({"batch": B, "iter": 0, "elapsed_s": 0.0, "objective": objective(eng.s)})
        for k0 in range(0, a.iters, a.every):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for k in range(k0, min(a.iters, k0 + a.every)):
                if B < M:
                    eng.sample_device(configs.SEEDS["minibatch"], k, B)
                eng.step_staged()
            e1.record(st)
            torch.cuda.synchronize()
            t_total += e0.elapsed_time(e1) / 1e3
            rows.append({"batch": B, "iter": min(a.iters, k0 + a.every), "elapsed_s": t_total,
                         "objective": objective(eng.s)})
        ips = a.iters / t_total
        print(json.dumps({"batch": B, "iters": a.iters, "seconds": t_total, "iters_per_s": ips,
                          "entries_per_s": 2.0 * B * N * ips, "final_objective": rows[-1]["objective"],
                          "initial_objective": rows[-a.iters // a.every - 1]["objective"]}), flush=True)
        del eng, plan
        torch.cuda.empty_cache()
    Path(a.out).parent.mkdir(parents=True, exist_ok=True)
    with open(a.out, "w", newline="") as f:
        wr = csv.DictWriter(f, fieldnames=["batch", "iter", "elapsed_s", "objective"])
        wr.writeheader()
        wr.writerows(rows)


if __name__ == "__main__":
    main()
