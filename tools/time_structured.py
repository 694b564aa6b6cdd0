#!/usr/bin/env python3
"""Structured (Cartesian) vs flat kernels on BASELINE Large, complex64.

For each composition (n_f, n_tx, n_rx) it times forward and adjoint+prox (CUDA events,
after warm-up) on the separable path and on the flat path over the same channel list,
and prints one JSON line per composition with A-entry evaluations/s.

    python tools/time_structured.py [--comps 4x32x32,16x16x16,128x48x48] [--reps 5] [--zslab 0:64]
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


def timed(fn, reps):
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--comps", default="4x32x32,2x48x48,16x16x16,8x8x8,32x4x4,128x48x48")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--zslab", default=None)
    ap.add_argument("--dtype", default="c64")
    ap.add_argument("--no-flat", action="store_true")
    a = ap.parse_args()
    scn = configs.large_scenario()
    z = None if a.zslab is None else tuple(int(v) for v in a.zslab.split(":"))
    plan = DevicePlan(scn, dtype=a.dtype, z_range=z)
    T, R, F = scn.array.n_tx, scn.array.n_rx, scn.frequencies.count
    rng = np.random.default_rng(0)
    dt = plan.torch_dtype
    s = (torch.randn(plan.n_local, dtype=dt, device=plan.device) * 1e-3)
    s2 = torch.empty_like(s)
    y = torch.randn(plan.M, dtype=dt, device=plan.device)
    stats = torch.zeros(4, dtype=torch.float64, device=plan.device)
    for comp in a.comps.split(","):
        kf, kt, kr = (int(v) for v in comp.split("x"))
        fs = np.sort(rng.choice(F, kf, replace=False))
        ts = np.sort(rng.choice(T, kt, replace=False))
        rs = np.sort(rng.choice(R, kr, replace=False))
        idx = (rs[None, None, :] + R * (ts[None, :, None] + T * fs[:, None, None])).reshape(-1)
        B = idx.size
        yb = torch.empty(B, dtype=dt, device=plan.device)
        out = {"comp": comp, "B": B, "N": plan.n_local}
        for name in ("structured", "flat"):
            if name == "flat" and a.no_flat:
                continue
            if name == "structured":
                plan.prepare_structured(fs, ts, rs)
            else:
                plan.prepare(torch.from_numpy(idx.astype(np.int32)).to(plan.device))
            tf = timed(lambda: plan.forward(s, out=yb), a.reps)
            ta = timed(lambda: plan.adjoint_prox(yb, y, s, s2, 1e-3 / B, 1e-9, stats), a.reps)
            ent = float(B) * plan.n_local
            out[name] = {"fwd_ms": tf * 1e3, "adj_ms": ta * 1e3, "fwd_eps": ent / tf, "adj_eps": ent / ta,
                         "step_eps": 2 * ent / (tf + ta)}
        if "flat" in out:
            out["speedup"] = out["flat"]["fwd_ms"] + out["flat"]["adj_ms"]
            out["speedup"] /= out["structured"]["fwd_ms"] + out["structured"]["adj_ms"]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
